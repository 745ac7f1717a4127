#!/bin/bash
# ncu evidence: full capture of the K2 verify and K1 draft launches (microbench shape
# configs[1]-like: batch 128, ctx 4096, GQA 4), and the per-launch list of bench.py's
# timed region.
set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:attn -s 3 -c 1 \
  -o gpurun_out/prof_k2 -f python bench_kernels.py --ctx 4096 --only verify --iters 2 --warmup 3 > gpurun_out/prof_k2.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:attn -s 3 -c 1 \
  -o gpurun_out/prof_k1 -f python bench_kernels.py --ctx 8192 --sparsity 0.05 --only draft --iters 2 --warmup 3 > gpurun_out/prof_k1.log 2>&1
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_random/" \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/launches.log 2>&1
