#!/bin/bash
O=gpurun_out/tm10; mkdir -p $O; rm -f $O/bench.txt
for v in default tm10 default tm10; do
  echo "== $v" | tee -a $O/bench.txt
  L=""; [ $v != default ] && L=$PWD/altv/$v/libeikfld_b200.so
  EIK_LIB=$L bash tools/quick_bench.sh C5 | tee -a $O/bench.txt
done
EIK_LIB=$PWD/altv/tm10/libeikfld_b200.so timeout 600 python -m pytest tests/test_gpu_configs.py::test_c5_eight_items_vs_oracle tests/test_gpu_parity.py::test_c5_item_and_batch_consistency -x -q 2>&1 | tail -3
