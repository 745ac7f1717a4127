#!/bin/bash
mkdir -p gpurun_out
SD_UMMA_OPT=2 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/ab_pytest.log 2>&1
for o in 0 2; do echo "opt=$o $(SD_UMMA_OPT=$o SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py 4096 128 5 2>&1 | head -5 | tr '\n' ' ')"; done > gpurun_out/ab.log 2>&1
