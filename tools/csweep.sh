mkdir -p gpurun_out
for c in 2 3 4 5 6 8; do echo "C=$c"; SD_ATTN_C=$c timeout 120 python bench_kernels.py --iters 20 --only verify --batch 25 --ctx 4608; done > gpurun_out/csweep_b25.log 2>&1
for c in 4 6 8 10 12 13 16; do echo "C=$c"; SD_ATTN_C=$c timeout 120 python bench_kernels.py --iters 10 --only verify --ctx 16384; done > gpurun_out/csweep_16k.log 2>&1
for c in 2 3 4 6 8; do echo "C=$c"; SD_ATTN_C=$c timeout 120 python bench_kernels.py --iters 10 --only verify --ctx 4096; done > gpurun_out/csweep_4k.log 2>&1
