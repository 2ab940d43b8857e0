#!/bin/bash
# ncu --set full (application replay: no 100+ GB save/restore) of one axis-0 column pass and one
# axis-1 lines pass of a C4 step at 1024^3
O=gpurun_out/c4prof; mkdir -p $O
timeout 2400 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:"col_tmem" -c 1 -o $O/c4_col_full -f python tools/prof_c4.py 1024 1 > $O/ncu_col_full.log 2>&1; tail -2 $O/ncu_col_full.log
timeout 2400 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:"lines_kernel" --launch-skip 7 -c 1 -o $O/c4_lines_full -f python tools/prof_c4.py 1024 1 > $O/ncu_lines_full.log 2>&1; tail -2 $O/ncu_lines_full.log
python tools/ncu_summary.py $O/c4_col_full.ncu-rep | tee $O/ncu_full_c4_col.txt
python tools/ncu_summary.py $O/c4_lines_full.ncu-rep | tee $O/ncu_full_c4_lines.txt
