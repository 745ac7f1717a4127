#!/bin/bash
mkdir -p gpurun_out
for c in 0 5 6 10 11; do echo "C=$c n=8192 $(SD_ATTN_C=$c SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py 8192 128 5 2>&1 | head -1)"; done > gpurun_out/csweep.log 2>&1
for c in 0 3 5; do echo "C=$c n=4096 $(SD_ATTN_C=$c SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py 4096 128 5 2>&1 | head -1)"; done >> gpurun_out/csweep.log 2>&1
echo "C=auto e2e-shape $(SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py 4613 26 5 2>&1 | head -1)" >> gpurun_out/csweep.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/bench_new.log 2>&1
