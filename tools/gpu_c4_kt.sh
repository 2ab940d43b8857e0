#!/bin/bash
# line-major 3-D spectra: 3-D parity tests, then C4 1024^3 / 512^3 / C3 timing (default and LPC=4 variant)
O=gpurun_out/c4kt; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_shapes3d.py tests/test_gpu_parity.py tests/test_slab_gpu.py tests/test_gpu_c4_full.py -x -q -m gpu 2>&1 | tail -6 | tee $O/tests.txt
for v in default lpc4; do
  echo "== $v" | tee -a $O/bench.txt
  L=""; [ $v != default ] && L=$PWD/altv/$v/libeikfld_b200.so
  EIK_LIB=$L timeout 900 python bench.py --config C4 --steps 2 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4', d['ms_per_step'], d['pass_ms'], d['config']['inside_fraction'])" | tee -a $O/bench.txt
  EIK_LIB=$L timeout 900 python bench.py --config C4 --c4-size 512 --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4@512', d['ms_per_step'], d['pass_ms'], d['config']['inside_fraction'])" | tee -a $O/bench.txt
  EIK_LIB=$L bash tools/quick_bench.sh C3 C2 | tee -a $O/bench.txt
done
