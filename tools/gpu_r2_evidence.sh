#!/bin/bash
# round-2 evidence: GPU tests, smoke, default bench line, launch list of the timed region,
# ncu --set full of bench.py's own K2, K1 and largest GEMM launches
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
( time timeout 1500 python bench.py ) > gpurun_out/bench.log 2> gpurun_out/bench_err.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_random/" \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/launches.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_random/" \
  -k regex:attn_umma_kernel -c 1 -o gpurun_out/prof_k2_bench -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/prof_k2_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_random/" \
  -k regex:attn_umma_hp -c 1 -o gpurun_out/prof_k1_bench -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/prof_k1_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --nvtx --nvtx-include "timed_random/" \
  -k regex:nvjet -c 4 -o gpurun_out/prof_gemm_bench -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/prof_gemm_bench.log 2>&1
