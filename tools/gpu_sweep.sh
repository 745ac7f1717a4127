#!/bin/bash
mkdir -p gpurun_out
for n in 4096 8192; do
for c in 1 2 3; do echo "narrow n=$n C=$c $(SD_ATTN_C=$c SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py $n 128 5 2>&1 | head -1)"; done
for c in 1 2 3 4; do echo "wide n=$n C=$c $(SD_UMMA_WIDE=1 SD_ATTN_C=$c SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py $n 128 5 2>&1 | head -1)"; done
echo "wide n=$n auto $(SD_UMMA_WIDE=1 SD_ATTN_TRACE=1 timeout 300 python tools/trace_umma.py $n 128 5 2>&1 | head -1)"
done > gpurun_out/sweep.log 2>&1
