#!/bin/bash
# Quick check of the tcgen05 attention kernels: kernel parity tests + microbench + phase trace.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/umma_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/umma_pytest.log
timeout 600 python bench_kernels.py --sparsity 0.05 --iters 20 --only verify > gpurun_out/umma_kb.log 2>&1
timeout 600 python bench_kernels.py --sparsity 0.05 --iters 20 --only verify --G 8 --ctx 4096,8192,32768 >> gpurun_out/umma_kb.log 2>&1
SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py 4096 128 5 > gpurun_out/trace.log 2>&1
