#!/bin/bash
# Round-2 capture on one GPU: tests, the default bench line (cfg4 headline + variants + CPU oracle +
# e2e), the reference arm, launch lists (cfg4, cfg2), ncu --set full of the top kernels.
# Usage: bash tools/r2_capture.sh <tag>
TAG=${1:-r2x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>> gpurun_out/${TAG}_bench.err
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none -c 80 --csv --log-file gpurun_out/${TAG}_launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${TAG}_ncu_l4.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -c 80 --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv python bench.py --cfg 2 --steps 2 --warmup 1 --no-variants --no-cpu --no-e2e --no-peaks > gpurun_out/${TAG}_ncu_l2.log 2>&1
NO="--no-variants --no-cpu --no-e2e --no-peaks"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather3y -s 1 -c 1 -o gpurun_out/${TAG}_gather_cfg4 -f python bench.py --steps 1 --warmup 1 $NO > gpurun_out/${TAG}_ncu_g4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:radix_scatter -s 2 -c 1 -o gpurun_out/${TAG}_sort_cfg4 -f python bench.py --steps 1 --warmup 1 $NO > gpurun_out/${TAG}_ncu_s4.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gather1b -s 2 -c 1 -o gpurun_out/${TAG}_gather_cfg2 -f python bench.py --cfg 2 --steps 1 --warmup 3 $NO > gpurun_out/${TAG}_ncu_g2.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gather2c -s 1 -c 1 -o gpurun_out/${TAG}_gather_cfg3 -f python bench.py --cfg 3 --steps 1 --warmup 2 $NO > gpurun_out/${TAG}_ncu_g3.log 2>&1
