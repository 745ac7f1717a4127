#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/k1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k1_tests.log
timeout 300 python bench_kernels.py --iters 20 --batch 128 --ctx 4096,16384,65536 --sparsity 0.01,0.05 --only draft > gpurun_out/k1_kb.log 2>&1
timeout 300 python bench_kernels.py --iters 20 --batch 103 --ctx 4608 --sparsity 0.05 --only draft >> gpurun_out/k1_kb.log 2>&1
SD_ATTN_TRACE=1 timeout 120 python tools/trace_umma.py 4608 103 0 231 > gpurun_out/k1_trace.log 2>&1
