#!/bin/bash
# gather3q A/B: round-2 tests, then the cfg4 bench with the default gather and with BNFFT_GATHER3Q; T=tag
T=${1:-q1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_round2.py -q -x -k "sweep3" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
B="--no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3"
timeout 300 python bench.py $B > gpurun_out/${T}_bench4_y.json 2> gpurun_out/${T}_bench4_y.err
BNFFT_GATHER3Q=1 timeout 300 python bench.py $B > gpurun_out/${T}_bench4_q.json 2> gpurun_out/${T}_bench4_q.err
