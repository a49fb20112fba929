#!/bin/bash
# fast iteration on the cfg4 path: d=3 GPU tests + cfg4 full-size parity + cfg4 bench line; T=tag
T=${1:-q4}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_round2.py tests/test_gpu_fullsize.py -q -x -k "sweep3 or ysweep or slab or repeat or sorted or cfg4" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 300 python bench.py --no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3 > gpurun_out/${T}_bench4.json 2> gpurun_out/${T}_bench4.err
