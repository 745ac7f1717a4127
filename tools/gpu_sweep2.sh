#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/s2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s2_pytest.log
timeout 600 python bench_kernels.py --iters 20 --only draft --sparsity 0.05,0.1 > gpurun_out/s2_kb.log 2>&1
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/s2_bench.log 2>&1
