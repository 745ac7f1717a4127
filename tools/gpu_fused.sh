#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fused_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fused_pytest.log
timeout 600 python tools/gpu_only_step.py > gpurun_out/fused_gonly.log 2>&1
SD_ATTN_FUSED=0 timeout 600 python tools/gpu_only_step.py > gpurun_out/fused_gonly0.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/fused_bench.log 2>&1
