#!/bin/bash
T=${1:-c3k}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_round2.py -q -x -k "gather2c" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
B="--cfg 3 --no-variants --no-cpu --no-e2e --no-peaks --steps 20 --warmup 5"
for i in 1 2; do timeout 120 python bench.py $B 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['ms_per_step'],4), round(d['stages_ms']['gather'],4))" >> gpurun_out/${T}_cfg3.txt; done
