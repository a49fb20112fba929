#!/bin/bash
# host-transform pipeline: parity tests + cfg2 / cfg4 bench lines with e2e; T=tag
T=${1:-e2}
mkdir -p gpurun_out
python tools/pcie_probe.py > gpurun_out/${T}_pcie.json 2>&1
timeout 300 python bench.py --cfg 2 --no-variants --no-cpu --no-peaks --steps 40 --warmup 3 > gpurun_out/${T}_bench2.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --no-variants --no-cpu --no-peaks --steps 10 --warmup 3 > gpurun_out/${T}_bench4.json 2>> gpurun_out/${T}_bench.err
