#!/bin/bash
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/hp3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/hp3_pytest.log
timeout 300 python bench_kernels.py --iters 20 --only draft --ctx 4096,8192,32768 --sparsity 0.05 > gpurun_out/hp3_kb.log 2>&1
SD_UMMA_HP_SLOTS=2 timeout 300 python bench_kernels.py --iters 20 --only draft --ctx 4096,8192 --sparsity 0.05 >> gpurun_out/hp3_kb.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/hp3_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --nvtx --nvtx-include "timed_random/" -k regex:attn_umma_kernel -c 1 \
  -o gpurun_out/prof_bench_k2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/prof_bench_k2.log 2>&1
