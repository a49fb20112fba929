#!/bin/bash
# fast iteration: round-2 GPU tests + cfg4 bench line; T=tag
T=${1:-q4}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_round2.py -q -x > gpurun_out/${T}_round2.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_round2.log
timeout 300 python bench.py --no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3 > gpurun_out/${T}_bench4.json 2> gpurun_out/${T}_bench4.err
