#!/bin/bash
# d = 2 tests, then the cfg3 bench (default gather2c) and all GPU tests; T=tag
T=${1:-c3h}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
B="--cfg 3 --no-variants --no-cpu --no-e2e --no-peaks --steps 20 --warmup 5"
timeout 300 python bench.py $B > gpurun_out/${T}_bench3.json 2> gpurun_out/${T}_bench3.err
