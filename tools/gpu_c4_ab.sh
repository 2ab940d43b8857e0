#!/bin/bash
# C4 A/B of library variants under altv/ (1024^3 step and pass times)
O=gpurun_out/c4ab; mkdir -p $O; rm -f $O/bench.txt
P='import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], round(d["ms_per_step"],1), {k: round(v,1) for k,v in d["pass_ms"].items()}, d["config"].get("inside_fraction"))'
for v in default $(ls altv); do
  echo "== $v" | tee -a $O/bench.txt
  L=""; [ $v != default ] && L=$PWD/altv/$v/libeikfld_b200.so
  EIK_LIB=$L timeout 900 python bench.py --config C4 --steps 2 --warmup 1 2>/dev/null | python -c "$P" | tee -a $O/bench.txt
done
