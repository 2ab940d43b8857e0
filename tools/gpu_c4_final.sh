#!/bin/bash
# final C4 evidence: 3-D tests, bench lines (1024^3 and 512^3), launch list of one step
O=gpurun_out/c4final; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_shapes3d.py tests/test_slab_gpu.py tests/test_gpu_c4_full.py tests/test_slab_ipc_gpu.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -4 | tee $O/tests_3d.txt
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 > $O/bench_c4_1024.json 2> $O/bench_c4.err; tail -c 600 $O/bench_c4_1024.json
timeout 900 python bench.py --config C4 --c4-size 512 --steps 5 --warmup 3 > $O/bench_c4_512.json 2>> $O/bench_c4.err; tail -c 300 $O/bench_c4_512.json
bash tools/quick_bench.sh C3 C2 | tee $O/quick.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_1024.csv python tools/prof_c4.py 1024 1 > $O/ncu_1024.log 2>&1
python tools/launch_summary.py $O/launches_c4_1024.csv | tee $O/launches_1024_final.txt
