#!/bin/bash
# ncu --set full (application replay) of the final axis-1 lines kernels of a C4 step at 1024^3
O=gpurun_out/c4prof; mkdir -p $O
timeout 2400 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:"lines_kernel" --launch-skip 7 -c 1 -o $O/c4_lines_full2 -f python tools/prof_c4.py 1024 1 > $O/ncu_lines_full2.log 2>&1; tail -2 $O/ncu_lines_full2.log
python tools/ncu_summary.py $O/c4_lines_full2.ncu-rep | tee $O/ncu_full_c4_lines_final.txt
timeout 2400 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:"lines_kernel" --launch-skip 11 -c 1 -o $O/c4_linesinv_full2 -f python tools/prof_c4.py 1024 1 > $O/ncu_linesinv_full2.log 2>&1
python tools/ncu_summary.py $O/c4_linesinv_full2.ncu-rep | tee $O/ncu_full_c4_linesinv_final.txt
rm -f $O/*.ncu-rep
