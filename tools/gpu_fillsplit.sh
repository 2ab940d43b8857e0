#!/bin/bash
O=gpurun_out/fillsplit; mkdir -p $O; rm -f $O/bench.txt
timeout 1500 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_fill_rule.py tests/test_slab_gpu.py tests/test_gpu_shapes3d.py -x -q -m gpu 2>&1 | tail -3 | tee $O/tests.txt
for e in 1 0 1 0; do
  echo "== EIK_FILL_SPLIT=$e" | tee -a $O/bench.txt
  EIK_FILL_SPLIT=$e bash tools/quick_bench.sh C2 | tee -a $O/bench.txt
done
