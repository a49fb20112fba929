#!/bin/bash
# experiment: L2 fetch granularity and the sequential-record ablation on the cfg4 bench
T=${1:-e1}
mkdir -p gpurun_out
P=paper_2502_07155_b200
B="--no-variants --no-cpu --no-e2e --no-peaks --steps 10 --warmup 3"
run() { timeout 300 python -c "
import ctypes, sys, torch
torch.cuda.init(); torch.zeros(1, device='cuda')
g = int('$2')
if g:
    rt = ctypes.CDLL('libcudart.so.12'); print('setlimit', rt.cudaDeviceSetLimit(5, g), file=sys.stderr)
    v = ctypes.c_size_t(0); rt.cudaDeviceGetLimit(ctypes.byref(v), 5); print('limit', v.value, file=sys.stderr)
sys.argv = ['bench.py'] + '$B'.split()
import bench; bench.main()
" > gpurun_out/${T}_$1.json 2>> gpurun_out/${T}.err; }
cp $P/libbnfft.so $P/libbnfft_base.so
run base 0
run g32 32
run g64 64
run g128 128
cp $P/libbnfft_seq.so $P/libbnfft.so
run seq 0
cp $P/libbnfft_base.so $P/libbnfft.so
