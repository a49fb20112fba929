#!/bin/bash
# cfg4 gather A/B: gather3c vs gather3s bench + ncu --set full of each; T=tag
T=${1:-g3}
mkdir -p gpurun_out
timeout 300 python bench.py --no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3 > gpurun_out/${T}_b3c.json 2> gpurun_out/${T}_b.err
BNFFT_GATHER3S=1 timeout 300 python bench.py --no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3 > gpurun_out/${T}_b3s.json 2>> gpurun_out/${T}_b.err
BNFFT_GATHER3S=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather3s -s 1 -c 1 -o gpurun_out/${T}_g3s -f python bench.py --steps 1 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu3s.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather3c -s 1 -c 1 -o gpurun_out/${T}_g3c -f python bench.py --steps 1 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu3c.log 2>&1
