#!/bin/bash
T=${1:-c3d}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py -q -x -k "gather2c or reduced or cfg3 or repeat or sorted or bin_sort" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
O=gpurun_out/${T}_cfg3.txt
: > $O
B="--cfg 3 --no-variants --no-cpu --no-e2e --no-peaks --steps 20 --warmup 5"
for th in 64 128 256; do for nb in 2 3 4; do
  echo "## TH=$th NB=$nb" >> $O
  env BNFFT_GATHER2C_THREADS=$th BNFFT_BOX_BUFS=$nb timeout 120 python bench.py $B 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})" >> $O
done; done
