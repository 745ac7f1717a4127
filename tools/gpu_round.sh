#!/bin/bash
# Round evidence: GPU tests, smoke, bench line (+ reference arm), per-launch list of the
# timed region, and one full ncu capture of the K2 verify and K1 draft launches.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
( time timeout 1500 python bench.py ) > gpurun_out/bench.log 2> gpurun_out/bench_time.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 python bench_kernels.py --iters 20 > gpurun_out/kb_all.log 2>&1
timeout 600 python bench_kernels.py --iters 20 --G 8 --ctx 4096,8192,32768 --sparsity 0.05 > gpurun_out/kb_g8.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:attn_umma_kernel -s 3 -c 1 \
  -o gpurun_out/prof_k2 -f python bench_kernels.py --ctx 4096 --only verify --iters 2 --warmup 3 > gpurun_out/prof_k2.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:attn_umma_hp -s 3 -c 1 \
  -o gpurun_out/prof_k1 -f python bench_kernels.py --ctx 8192 --sparsity 0.05 --only draft --iters 2 --warmup 3 > gpurun_out/prof_k1.log 2>&1
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed_random/" \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --variants none > gpurun_out/launches.log 2>&1
