#!/bin/bash
mkdir -p gpurun_out
for n in 4096 8192; do for pf in 0 2 4; do echo "n=$n pf=$pf $(SD_UMMA_PF=$pf SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py $n 128 5 2>&1 | head -5 | tr '\n' ' ')"; done; done > gpurun_out/pf.log 2>&1
for pf in 0 3; do SD_UMMA_PF=$pf timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/bench_pf$pf.log 2>&1; done
