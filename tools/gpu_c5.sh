#!/bin/bash
# cfg5 knobs of the batched gatherN: CTA size x box ring depth; T=tag
T=${1:-c5}
mkdir -p gpurun_out
O=gpurun_out/${T}_cfg5.txt
: > $O
B="--cfg 5 --no-variants --no-cpu --no-e2e --no-peaks --steps 2 --warmup 1"
for th in 256 128 64 32; do for nb in 2 3; do
  echo "## TH=$th NB=$nb" >> $O
  env BNFFT_GATHERN_THREADS=$th BNFFT_BOX_BUFS=$nb timeout 200 python bench.py $B 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['ms_per_step'],2), round(d['stages_ms']['gather'],2))" >> $O
done; done
