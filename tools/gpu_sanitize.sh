#!/bin/bash
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $CS --tool racecheck --racecheck-report analysis --target-processes all python -m pytest tests/test_kernels_gpu.py -q -x -k "(test_verify_attention_matches_oracle and False-128) or test_batched_items_mixed_lengths_bf16" > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
