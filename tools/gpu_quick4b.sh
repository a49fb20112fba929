#!/bin/bash
# fast iteration: d=3 parity tests + round-2 tests + cfg4 bench + launch list; T=tag
T=${1:-q4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/${T}_round2.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_round2.log
timeout 300 python bench.py --no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3 > gpurun_out/${T}_bench4.json 2> gpurun_out/${T}_bench4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/${T}_launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu_l4.log 2>&1
