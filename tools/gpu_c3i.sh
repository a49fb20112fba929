#!/bin/bash
T=${1:-c3i}
mkdir -p gpurun_out
O=gpurun_out/${T}_cfg3.txt
: > $O
B="--cfg 3 --no-variants --no-cpu --no-e2e --no-peaks --steps 20 --warmup 5"
for ub in 19 20 21; do for th in 32 64; do for nb in 2 3; do
  echo "## UB=$ub TH=$th NB=$nb" >> $O
  env BNFFT_UB_LOG2=$ub BNFFT_GATHER2C_THREADS=$th BNFFT_BOX_BUFS=$nb timeout 120 python bench.py $B 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})" >> $O
done; done; done
