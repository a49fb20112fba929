#!/bin/bash
# y-sweep gather bring-up: round-2 tests, all GPU tests, cfg4 bench, launch list, ncu of gather3y; T=tag
T=${1:-y1}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_round2.py -q -x > gpurun_out/${T}_round2.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_round2.log
timeout 300 python bench.py --no-variants --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/${T}_bench4.json 2> gpurun_out/${T}_bench4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/${T}_launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu_l4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather3y -s 1 -c 1 -o gpurun_out/${T}_g3y -f python bench.py --steps 1 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${T}_ncu.log 2>&1
timeout 900 python -m pytest tests/ -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
