#!/bin/bash
# launch list (cold, serialised) of one C4 step at 1024^3 and at 512^3
O=gpurun_out/c4prof; mkdir -p $O
for n in 1024 512; do
  timeout 900 python tools/prof_c4.py $n 1 > $O/plain_$n.log 2>&1 || { tail -5 $O/plain_$n.log; continue; }
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_$n.csv python tools/prof_c4.py $n 1 > $O/ncu_$n.log 2>&1
  python tools/launch_summary.py $O/launches_c4_$n.csv | tee $O/summary_$n.txt
done
