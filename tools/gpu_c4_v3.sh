#!/bin/bash
# E=16 persistent lines kernels + wide 3-D column kernels: 3-D tests, C4 / C3 timing, L2 fetch granularity probe, launch list
O=gpurun_out/c4v3; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_shapes3d.py tests/test_gpu_parity.py tests/test_slab_gpu.py tests/test_gpu_c4_full.py tests/test_slab_ipc_gpu.py -x -q -m gpu 2>&1 | tail -6 | tee $O/tests.txt
P='import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], d["ms_per_step"], d["pass_ms"], d["config"].get("inside_fraction"))'
timeout 900 python bench.py --config C4 --steps 2 --warmup 1 2>/dev/null | python -c "$P" | tee -a $O/bench.txt
timeout 900 python bench.py --config C4 --c4-size 512 --steps 3 --warmup 2 2>/dev/null | python -c "$P" | tee -a $O/bench.txt
bash tools/quick_bench.sh C3 | tee -a $O/bench.txt
for g in 32 128; do
  echo "== L2 fetch granularity $g" | tee -a $O/bench.txt
  timeout 900 python tools/bench_l2g.py $g --config C4 --steps 2 --warmup 1 2>>$O/l2g.err | python -c "$P" | tee -a $O/bench.txt
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_1024_v3.csv python tools/prof_c4.py 1024 1 > $O/ncu_1024_v3.log 2>&1
python tools/launch_summary.py $O/launches_c4_1024_v3.csv | tee $O/summary_1024_v3.txt
