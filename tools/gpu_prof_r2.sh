#!/bin/bash
# round-2 profiling pass: K1 phase traces, ncu --set full of bench.py's own K2 and K1 launches
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
SD_ATTN_TRACE=1 timeout 120 python tools/trace_umma.py 4096 128 0 41 > gpurun_out/trace_k1_s1.log 2>&1
SD_ATTN_TRACE=1 timeout 120 python tools/trace_umma.py 4096 128 0 205 > gpurun_out/trace_k1_s5.log 2>&1
SD_ATTN_TRACE=1 timeout 120 python tools/trace_umma.py 4608 103 0 231 > gpurun_out/trace_k1_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_random/" \
  -k regex:attn_umma_kernel -c 1 -o gpurun_out/prof_k2_bench -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/prof_k2_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_random/" \
  -k regex:attn_umma_hp -c 1 -o gpurun_out/prof_k1_bench -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/prof_k1_bench.log 2>&1
