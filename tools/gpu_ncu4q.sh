#!/bin/bash
T=${1:-n4q}
mkdir -p gpurun_out
BNFFT_GATHER3Q=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather3q -s 1 -c 1 -o gpurun_out/${T}_g3q -f python bench.py --steps 1 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu.log 2>&1
