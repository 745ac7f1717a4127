#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_api_gpu.py -x -q -k native > gpurun_out/c3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c3_pytest.log
timeout 1500 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --variants planted,c3 > gpurun_out/c3_bench.log 2>&1
