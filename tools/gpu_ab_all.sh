#!/bin/bash
# A/B of library variants under altv/: C2 / C5 / C3 quick bench twice, then C4 1024^3
O=gpurun_out/aball; mkdir -p $O; rm -f $O/bench.txt
for rep in 1 2; do
for v in default $(ls altv); do
  echo "== $v" | tee -a $O/bench.txt
  L=""; [ $v != default ] && L=$PWD/altv/$v/libeikfld_b200.so
  EIK_LIB=$L bash tools/quick_bench.sh C2 C5 C3 | tee -a $O/bench.txt
done
done
bash tools/gpu_c4_ab.sh
for v in $(ls altv); do
EIK_LIB=$PWD/altv/$v/libeikfld_b200.so timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_shapes3d.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
done
