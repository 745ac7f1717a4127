#!/bin/bash
mkdir -p gpurun_out
SD_ATTN_PLAN_LOG=1 SD_ATTN_TRACE=1 timeout 120 python tools/trace_umma.py 4608 25 5 0 > gpurun_out/trace_k2_bench.log 2>&1
SD_ATTN_PLAN_LOG=1 SD_ATTN_TRACE=1 timeout 120 python tools/trace_umma.py 4096 128 5 0 > gpurun_out/trace_k2_128.log 2>&1
SD_ATTN_TRACE=1 timeout 120 python tools/trace_umma.py 4608 103 0 231 > gpurun_out/trace_k1_bench.log 2>&1
timeout 600 python bench_kernels.py --iters 20 --ctx 4096,16384,65536 --sparsity 0.01,0.05 > gpurun_out/kb.log 2>&1
