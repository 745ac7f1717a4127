#!/bin/bash
mkdir -p gpurun_out
SD_UMMA_PF=2 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/pf_pytest.log 2>&1
for n in 4096 8192 32768; do for pf in 0 1 2 3; do echo "n=$n pf=$pf $(SD_UMMA_PF=$pf SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py $n 128 5 2>&1 | head -5 | tr '\n' ' ')"; done; done > gpurun_out/pf.log 2>&1
