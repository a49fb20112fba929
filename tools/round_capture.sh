TAG=${1:-rX}
set -x
timeout 900 python -m pytest tests/ -q -m gpu > gpurun_out/${TAG}_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
for c in 3 4 5; do timeout 600 python bench.py --cfg $c --no-cpu > gpurun_out/${TAG}_bench_cfg$c.json 2>> gpurun_out/${TAG}_bench.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2>> gpurun_out/${TAG}_bench.err
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-variants --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_l.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gather1b -s 2 -c 1 -o gpurun_out/${TAG}_gather_cfg2 -f python bench.py --steps 1 --warmup 3 --no-variants --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_g2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather3c -s 1 -c 1 -o gpurun_out/${TAG}_gather_cfg4 -f python bench.py --cfg 4 --steps 1 --warmup 3 --no-variants --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_g4.log 2>&1
