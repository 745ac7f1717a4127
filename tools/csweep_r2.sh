#!/bin/bash
# K2 cluster-size sweep at bench.py's four window contexts (25 verify items) vs the planner's pick
mkdir -p gpurun_out
for ctx in 1536 3584 5632 7680; do
  SD_ATTN_PLAN_LOG=1 timeout 60 python bench_kernels.py --iters 20 --batch 25 --ctx $ctx --only verify 2>&1 | grep -E "sd plan|K2" | head -2 | sed "s/^/planner ctx=$ctx /"
  for C in 1 2 3 4 5 6 8; do
    SD_ATTN_C=$C timeout 60 python bench_kernels.py --iters 20 --batch 25 --ctx $ctx --only verify 2>/dev/null | sed "s/^/C=$C ctx=$ctx /"
  done
done
