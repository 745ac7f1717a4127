#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/umma_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/umma_pytest.log
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
for c in 2 4 6 8; do SD_ATTN_C=$c SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py 4096 128 5 > gpurun_out/trace_c$c.log 2>&1; done
