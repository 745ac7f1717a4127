#!/bin/bash
mkdir -p gpurun_out
SD_ATTN_FUSED=1 timeout 900 python -m pytest tests/test_api_gpu.py -x -q -k native > gpurun_out/fused_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fused_pytest.log
for f in 0 1; do echo "fused=$f $(SD_ATTN_FUSED=$f timeout 600 python tools/gpu_only_step.py 2>&1 | tail -1)"; done > gpurun_out/fused_gonly.log 2>&1
