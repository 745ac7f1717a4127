#!/bin/bash
mkdir -p gpurun_out
for mb in 0 64; do echo "ws=$mb $(SD_CUBLAS_WS_MB=$mb timeout 600 python tools/gpu_only_step.py 2>&1 | tail -1)"; done > gpurun_out/ws.log 2>&1
