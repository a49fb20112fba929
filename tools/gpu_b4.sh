#!/bin/bash
# quick cfg4 bench (gather3s default) + ncu of the gather; T=tag
T=${1:-x}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_round2.py -q -x -k "sweep3" > gpurun_out/${T}_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_sweep.log
timeout 300 python bench.py --no-variants --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/${T}_bench4.json 2> gpurun_out/${T}_bench4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather3 -s 1 -c 1 -o gpurun_out/${T}_g3s -f python bench.py --steps 1 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu.log 2>&1
