#!/bin/bash
# A/B: library built from HEAD (altv/head) against the working tree, same box; 3-D tests; C4 timings; launch list
O=gpurun_out/abhead; mkdir -p $O gpurun_out/c4prof
rm -f $O/bench.txt
for rep in 1 2; do
for v in head default; do
  echo "== $v" | tee -a $O/bench.txt
  L=""; [ $v != default ] && L=$PWD/altv/$v/libeikfld_b200.so
  EIK_LIB=$L bash tools/quick_bench.sh C2 C3 C5 | tee -a $O/bench.txt
done
done
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_shapes3d.py tests/test_gpu_parity.py tests/test_slab_gpu.py tests/test_gpu_c4_full.py -x -q -m gpu 2>&1 | tail -6 | tee $O/tests.txt
timeout 900 python bench.py --config C4 --steps 2 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4', d['ms_per_step'], d['pass_ms'], d['config']['inside_fraction'])" | tee -a $O/bench.txt
timeout 900 python bench.py --config C4 --c4-size 512 --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4@512', d['ms_per_step'], d['pass_ms'], d['config']['inside_fraction'])" | tee -a $O/bench.txt
O=gpurun_out/c4prof
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_1024_v2.csv python tools/prof_c4.py 1024 1 > $O/ncu_1024_v2.log 2>&1
python tools/launch_summary.py $O/launches_c4_1024_v2.csv | tee $O/summary_1024_v2.txt
