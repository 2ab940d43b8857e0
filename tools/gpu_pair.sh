#!/bin/bash
O=gpurun_out/pair; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_shapes3d.py tests/test_slab_gpu.py tests/test_gpu_c4_full.py -x -q -m gpu 2>&1 | tail -4 | tee $O/tests.txt
P='import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], round(d["ms_per_step"],1), {k: round(v,1) for k,v in d["pass_ms"].items()}, d["config"].get("inside_fraction"))'
for e in 1 0 1; do
  echo "== EIK_STREAM_PAIR=$e" | tee -a $O/bench.txt
  EIK_STREAM_PAIR=$e timeout 900 python bench.py --config C4 --steps 2 --warmup 1 2>/dev/null | python -c "$P" | tee -a $O/bench.txt
done
