#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/dense_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/dense_pytest.log
timeout 600 python bench_kernels.py --iters 20 --only verify > gpurun_out/dense_kb.log 2>&1
timeout 600 python bench_kernels.py --iters 20 --only verify --G 8 --ctx 4096,8192,32768 >> gpurun_out/dense_kb.log 2>&1
