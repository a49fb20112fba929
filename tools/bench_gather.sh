#!/bin/bash
# quick per-config timing: prints workload, ms/step and per-stage ms
for c in "$@"; do
  timeout 400 python bench.py --cfg $c --steps 5 --warmup 2 --no-variants --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:40], '| ms/step', round(d['ms_per_step'],3), '| nodes/s %.3g' % d['value'], {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
