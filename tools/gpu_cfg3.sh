#!/bin/bash
# cfg3/cfg5 iteration: gatherN parity tests + cfg3/cfg5 bench lines (+ ring-depth A/B); T=tag
T=${1:-c3}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_binned.py tests/test_gpu_round2.py -q -x > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 300 python bench.py --cfg 3 --no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3 > gpurun_out/${T}_bench3.json 2> gpurun_out/${T}_bench3.err
BNFFT_GATHERN_THREADS=256 timeout 300 python bench.py --cfg 3 --no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3 > gpurun_out/${T}_bench3_b3.json 2>> gpurun_out/${T}_bench3.err
timeout 600 python bench.py --cfg 5 --no-variants --no-cpu --no-e2e --no-peaks --steps 3 --warmup 1 > gpurun_out/${T}_bench5.json 2>> gpurun_out/${T}_bench3.err
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gatherN -s 1 -c 1 -o gpurun_out/${T}_gather_cfg3 -f python bench.py --cfg 3 --steps 1 --warmup 2 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu_g3.log 2>&1
