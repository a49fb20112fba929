#!/bin/bash
T=${1:-s4}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:radix_scatter -s 3 -c 1 -o gpurun_out/${T}_scatter -f python bench.py --steps 1 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu_s.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:keys_kernel -s 1 -c 1 -o gpurun_out/${T}_keys -f python bench.py --steps 1 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu_k.log 2>&1
