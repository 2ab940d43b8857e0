# Round profile capture under gpurun (one GPU): launch lists of the bench
# command (C2 default, C3, C5) and one ncu --set full capture per config of
# one device-resident step (tools/prof_step.py; plan-time kernels excluded).
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
for c in C2 C3 C5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch_$c.log 2>&1
done
K='regex:col_tmem_kernel|row_kernel|impulse_rows|lines_kernel'
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -c 5 -o $OUT/c2_full -f \
  python tools/prof_step.py C2 1 > $OUT/ncu_full_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" --launch-skip 4 -c 5 -o $OUT/c3_full -f \
  python tools/prof_step.py C3 1 > $OUT/ncu_full_c3.log 2>&1
ls -la $OUT
# text summaries on the box (the reports together exceed gpurun's 64 MiB return limit)
python tools/ncu_summary.py $OUT/c2_full.ncu-rep > $OUT/ncu_full_c2.txt 2>&1
python tools/ncu_summary.py $OUT/c3_full.ncu-rep > $OUT/ncu_full_c3.txt 2>&1
ncu -i $OUT/c2_full.ncu-rep --page source --csv --print-kernel-base demangled > $OUT/c2_sass_src.csv 2>/dev/null
ncu -i $OUT/c3_full.ncu-rep --page source --csv --print-kernel-base demangled > $OUT/c3_sass_src.csv 2>/dev/null
gzip -f $OUT/c2_sass_src.csv $OUT/c3_sass_src.csv
rm -f $OUT/c3_full.ncu-rep
