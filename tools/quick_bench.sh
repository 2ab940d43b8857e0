#!/bin/bash
# quick per-config bench summary (used under gpurun)
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value']/1e9,3), 'Gpts/s ms', round(d['ms_per_step'],3), d.get('pass_ms'), 'e2e', d.get('e2e') and round(d['e2e']['value']/1e9,3), d.get('roofline') and d['roofline']['frac'], d.get('roofline') and d['roofline'].get('step_frac'))"
done
