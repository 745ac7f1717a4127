#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/pk_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pk_pytest.log
SD_ATTN_TRACE=1 timeout 300 python tools/trace_pk.py 4096 128 > gpurun_out/trace_pk.log 2>&1
timeout 300 python bench_kernels.py --iters 20 --only verify > gpurun_out/pk_kb.log 2>&1; echo "rc=$?" >> gpurun_out/pk_kb.log
timeout 300 python bench_kernels.py --iters 20 --only verify --G 8 --ctx 4096,8192,32768 >> gpurun_out/pk_kb.log 2>&1
