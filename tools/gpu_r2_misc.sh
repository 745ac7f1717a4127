#!/bin/bash
# round-2: configs[4] microbench grid (k x G x ctx, drafts s x G x ctx), configs[3] variant timing,
# compute-sanitizer on the tiny K2/K1 case
mkdir -p gpurun_out
rm -f gpurun_out/kb_grid.jsonl
for G in 4 8; do
  for k in 2 4 8; do
    timeout 300 python bench_kernels.py --iters 10 --G $G --k $k --ctx 4096,16384,65536 --only verify >> gpurun_out/kb_grid.jsonl 2>gpurun_out/kb_grid.err
  done
  timeout 300 python bench_kernels.py --iters 10 --G $G --ctx 4096,16384,65536 --sparsity 0.01,0.05,0.10 --only draft >> gpurun_out/kb_grid.jsonl 2>>gpurun_out/kb_grid.err
done
( time timeout 900 python bench.py --variants c3 --no-cpu-baseline --steps 6 ) > gpurun_out/c3.log 2> gpurun_out/c3_err.log
bash tools/gpu_sanitize.sh
