#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/k2tma_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k2tma_tests.log
for B in 25 128; do
 timeout 300 python bench_kernels.py --iters 20 --batch $B --ctx 4608,16384 --only verify >> gpurun_out/k2tma_kb.log 2>&1
 SD_K2_TMA=0 timeout 300 python bench_kernels.py --iters 20 --batch $B --ctx 4608 --only verify 2>&1 | sed 's/^/cpasync /' >> gpurun_out/k2tma_kb.log
done
SD_ATTN_TRACE=1 timeout 120 python tools/trace_umma.py 4608 25 5 0 > gpurun_out/k2tma_trace.log 2>&1
for C in 2 3 4 5 6 8; do SD_ATTN_C=$C timeout 120 python bench_kernels.py --iters 20 --batch 25 --ctx 4608 --only verify 2>&1 | sed "s/^/C=$C /" >> gpurun_out/k2tma_csweep.log; done
