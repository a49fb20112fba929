#!/bin/bash
# A/B of library builds on the cfg4 bench (on the GPU box's copy of the repo): each variant
# paper_2502_07155_b200/libbnfft_<v>.so is copied over libbnfft.so for its run.  T=tag, args = variants
T=$1; shift
mkdir -p gpurun_out
P=paper_2502_07155_b200
cp $P/libbnfft.so $P/libbnfft_base.so
run() { timeout 300 python bench.py --no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3 > gpurun_out/${T}_$1.json 2>> gpurun_out/${T}.err; }
run base
for v in "$@"; do
  cp $P/libbnfft_$v.so $P/libbnfft.so
  run $v
done
cp $P/libbnfft_base.so $P/libbnfft.so
run base2
