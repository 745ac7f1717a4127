#!/bin/bash
# One gpurun call: GPU tests per attention impl, microbench per impl, short bench, launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
for impl in tm ws mma; do
  SD_ATTN_IMPL=$impl timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$impl.log 2>&1
  SD_ATTN_IMPL=$impl timeout 600 python bench_kernels.py --ctx 4096,8192,32768 --sparsity 0.05 --iters 20 > gpurun_out/kb_$impl.log 2>&1
done
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
