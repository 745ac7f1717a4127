#!/bin/bash
# compute-sanitizer on a tiny K2 (2-CTA cluster) + K1 launch (tools/race_small.py)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  SD_ATTN_C=2 timeout 1200 $CS --tool $tool --target-processes all python tools/race_small.py \
    > gpurun_out/san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san_$tool.log
done
