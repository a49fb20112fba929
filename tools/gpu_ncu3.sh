#!/bin/bash
T=${1:-n3}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather2c -s 1 -c 1 -o gpurun_out/${T}_g2c -f python bench.py --cfg 3 --steps 1 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu.log 2>&1
