#!/bin/bash
# even/odd column kernel: C2 parity, then A/B bench (EIK_EO=1 vs 0)
mkdir -p gpurun_out/eo
timeout 600 python -m pytest tests/test_gpu_configs.py::test_c2_all_nodes_vs_oracle tests/test_gpu_parity.py::test_c2_full_size_unchecked_matches_reference -x -q 2>&1 | tail -15 | tee gpurun_out/eo/tests.txt
for eo in 1 0 1 0; do
  echo "EIK_EO=$eo" | tee -a gpurun_out/eo/bench.txt
  EIK_EO=$eo bash tools/quick_bench.sh C2 2>&1 | tee -a gpurun_out/eo/bench.txt
done
