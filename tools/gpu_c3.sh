#!/bin/bash
# cfg3 knobs: user-block size x CTA size x box ring depth; T=tag
T=${1:-c3}
mkdir -p gpurun_out
O=gpurun_out/${T}_cfg3.txt
: > $O
B="--cfg 3 --no-variants --no-cpu --no-e2e --no-peaks --steps 20 --warmup 5"
for ub in "" 19 20 22 31; do for th in 256 128; do for nb in 3 6; do
  echo "## UB=$ub TH=$th NB=$nb" >> $O
  env ${ub:+BNFFT_UB_LOG2=$ub} BNFFT_GATHERN_THREADS=$th BNFFT_BOX_BUFS=$nb timeout 120 python bench.py $B 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})" >> $O
done; done; done
