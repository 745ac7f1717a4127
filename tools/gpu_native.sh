#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/gpu_only_step.py > gpurun_out/native_gonly.log 2>&1
SD_BENCH_NO_CLOCKS=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/native_bench.log 2>&1
