#!/bin/bash
# one-call transform: its test, then the cfg4 bench with and without the overlap; T=tag
T=${1:-t1}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "transform" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
B="--no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3"
timeout 300 python bench.py $B > gpurun_out/${T}_bench4.json 2> gpurun_out/${T}_bench4.err
timeout 300 python bench.py $B --three-calls > gpurun_out/${T}_bench4_3c.json 2> gpurun_out/${T}_bench4_3c.err
timeout 300 python bench.py $B --cfg 2 > gpurun_out/${T}_bench2.json 2> gpurun_out/${T}_bench2.err
timeout 300 python bench.py $B --cfg 2 --three-calls > gpurun_out/${T}_bench2_3c.json 2> gpurun_out/${T}_bench2_3c.err
