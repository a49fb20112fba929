#!/bin/bash
# gather2c: d = 2 tests, then cfg3 bench with gather2c and with gatherN; T=tag
T=${1:-c3b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_round2.py -q -x -k "not slab and not nccl" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
B="--cfg 3 --no-variants --no-cpu --no-e2e --no-peaks --steps 20 --warmup 5"
timeout 300 python bench.py $B > gpurun_out/${T}_bench3.json 2> gpurun_out/${T}_bench3.err
BNFFT_GATHER2N=1 timeout 300 python bench.py $B > gpurun_out/${T}_bench3_n.json 2> gpurun_out/${T}_bench3_n.err
