// Streaming probe for the paged KV layout (diagnostics, not product code).
//
// Measures the HBM read bandwidth a CTA can pull for one kv head of one
// request, i.e. 256-byte rows at a 2 KB stride (token-major pages, Hkv = 8),
// with several load strategies:
//   0  all threads: LDG.128 into registers (sum, no smem)
//   1  all threads: cp.async 16 B, 4-stage ring, __syncthreads per tile
//   2  1 producer warp: cp.async 16 B + mbarrier (noinc arrive), 5-slot ring
//   3  1 producer warp: cp.async.bulk 256 B per row + mbarrier expect_tx
//   4  all threads: LDG.128, rows contiguous (dense 256 B stride) for reference
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe tools/stream_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int TK = 64;      // rows per tile
constexpr int ROWB = 256;   // bytes per row
constexpr int STRIDE = 2048;  // bytes between consecutive tokens of one head

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// mode 0/4: plain loads
__global__ void k_ldg(const uint4* base, int tiles, long long stride_u4, float* out) {
  const int unit = blockIdx.x;
  const uint4* p = base + (long long)unit * tiles * TK * stride_u4;
  float acc = 0.f;
  for (int t = 0; t < tiles; ++t) {
    uint4 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = threadIdx.x + i * 256;  // 1024 chunks of 16 B per tile
      const int row = c >> 4, part = c & 15;
      v[i] = __ldg(p + ((long long)(t * TK + row)) * stride_u4 + part);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) acc += __int_as_float(v[i].x ^ v[i].y ^ v[i].z ^ v[i].w);
  }
  if (acc == 1.2345f) out[0] = acc;
}

// mode 1: cp.async ring, all threads
__global__ void k_cpasync(const uint4* base, int tiles, long long stride_u4, float* out) {
  extern __shared__ uint4 sm[];
  constexpr int ST = 4;
  const int unit = blockIdx.x;
  const uint4* p = base + (long long)unit * tiles * TK * stride_u4;
  auto load = [&](int t, int s) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = threadIdx.x + i * 256, row = c >> 4, part = c & 15;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(sm + s * 1024 + c)),
                   "l"(p + ((long long)(t * TK + row)) * stride_u4 + part));
    }
  };
  for (int s = 0; s < ST - 1; ++s) { if (s < tiles) load(s, s); asm volatile("cp.async.commit_group;\n"); }
  float acc = 0.f;
  for (int t = 0; t < tiles; ++t) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(ST - 2));
    __syncthreads();
    if (t + ST - 1 < tiles) load(t + ST - 1, (t + ST - 1) % ST);
    asm volatile("cp.async.commit_group;\n");
    uint4 v = sm[(t % ST) * 1024 + threadIdx.x];
    acc += __int_as_float(v.x);
  }
  if (acc == 1.2345f) out[0] = acc;
}

// mode 2/3: producer warp + mbarrier ring
template <int MODE, int NS = 5, int NPROD = 1>
__global__ void k_ws(const uint4* base, int tiles, long long stride_u4, float* out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + NS;
  uint4* ring = reinterpret_cast<uint4*>(smraw + 128);
  const int unit = blockIdx.x;
  const uint4* p = base + (long long)unit * tiles * TK * stride_u4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < NS) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(full + threadIdx.x)), "r"(MODE == 2 ? 32 * NPROD : 1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(empty + threadIdx.x)), "r"(8));
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n");
  __syncthreads();
  auto wait = [&](uint64_t* b, unsigned par) {
    asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par));
  };
  if (warp >= 8) {
    const int pw = warp - 8;
    for (int t = 0; t < tiles; ++t) {
      const int s = t % NS;
      if (t >= NS) wait(empty + s, ((t / NS) - 1) & 1);
      uint4* dst = ring + s * 1024;
      if (MODE == 2) {
#pragma unroll 8
        for (int c = lane + 32 * pw; c < 1024; c += 32 * NPROD) {
          const int row = c >> 4, part = c & 15;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(dst + c)),
                       "l"(p + ((long long)(t * TK + row)) * stride_u4 + part));
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(su32(full + s)));
      } else if (pw == 0) {
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(full + s)), "r"(TK * ROWB));
        __syncwarp();
        for (int row = lane; row < TK; row += 32)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
                           "r"(su32(dst + row * 16)), "l"(p + ((long long)(t * TK + row)) * stride_u4), "r"(ROWB),
                       "r"(su32(full + s)));
      }
    }
    return;
  }
  float acc = 0.f;
  for (int t = 0; t < tiles; ++t) {
    const int s = t % NS;
    wait(full + s, (t / NS) & 1);
    acc += __int_as_float(ring[s * 1024 + threadIdx.x].x);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(empty + s)));
  }
  if (acc == 1.2345f) out[0] = acc;
}

// mode 5/6: two passes like the attention kernel: pass 1 streams K (tiles
// 0..T-1), pass 2 streams K again (L2) and V; mode 6 adds a cluster barrier of
// C CTAs between the passes.  Producer warp + cp.async + mbarrier, 5 slots.
template <bool CLUSTER>
__global__ void k_2pass(const uint4* kbase, const uint4* vbase, int tiles, long long stride_u4, float* out,
                        int evict) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int NS = 5;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + NS;
  uint4* ring = reinterpret_cast<uint4*>(smraw + 128);
  const int unit = blockIdx.x;
  const uint4* pk = kbase + (long long)unit * tiles * TK * stride_u4;
  const uint4* pv = vbase + (long long)unit * tiles * TK * stride_u4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < NS) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(full + threadIdx.x)), "r"(32));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(empty + threadIdx.x)), "r"(8));
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n");
  __syncthreads();
  auto wait = [&](uint64_t* b, unsigned par) {
    asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par));
  };
  uint64_t keep, drop;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(keep));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(drop));
  const int total = 3 * tiles;
  if (warp == 8) {
    for (int f = 0; f < total; ++f) {
      const int s = f % NS;
      if (f >= NS) wait(empty + s, ((f / NS) - 1) & 1);
      int t;
      const uint4* p;
      uint64_t pol;
      if (f < tiles) { t = f; p = pk; pol = keep; }
      else { t = (f - tiles) >> 1; p = ((f - tiles) & 1) ? pv : pk; pol = drop; }
      uint4* dst = ring + s * 1024;
#pragma unroll 8
      for (int c = lane; c < 1024; c += 32) {
        const int row = c >> 4, part = c & 15;
        if (evict)
          asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(su32(dst + c)),
                       "l"(p + ((long long)(t * TK + row)) * stride_u4 + part), "l"(pol));
        else
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(dst + c)),
                       "l"(p + ((long long)(t * TK + row)) * stride_u4 + part));
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(su32(full + s)));
      if (CLUSTER && f == tiles - 1) asm volatile("barrier.cluster.arrive.release.aligned;\n");
    }
    if (CLUSTER) asm volatile("barrier.cluster.wait.acquire.aligned;\n");
    return;
  }
  float acc = 0.f;
  for (int f = 0; f < total; ++f) {
    if (CLUSTER && f == tiles) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n");
    }
    const int s = f % NS;
    wait(full + s, (f / NS) & 1);
    acc += __int_as_float(ring[s * 1024 + threadIdx.x].x);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(empty + s)));
  }
  if (CLUSTER && tiles == 0) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n");
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main(int argc, char** argv) {
  if (argc > 3) {  // two-pass probe: units tiles cluster evict
    const int units = atoi(argv[1]), tiles = atoi(argv[2]), C = atoi(argv[3]), evict = argc > 4 ? atoi(argv[4]) : 1;
    const size_t per_unit = (size_t)tiles * TK * STRIDE;
    void *kb, *vb;
    float* out;
    CK(cudaMalloc(&kb, per_unit * units + 4096));
    CK(cudaMalloc(&vb, per_unit * units + 4096));
    CK(cudaMalloc(&out, 64));
    cudaMemset(kb, 1, per_unit * units);
    cudaMemset(vb, 1, per_unit * units);
    const int smem = 128 + 5 * 16384;
    cudaFuncSetAttribute(k_2pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_2pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_2pass<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    auto run = [&]() {
      if (C <= 0) {
        k_2pass<false><<<units, 288, smem>>>((const uint4*)kb, (const uint4*)vb, tiles, STRIDE / 16, out, evict);
      } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(units);
        cfg.blockDim = dim3(288);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, k_2pass<true>, (const uint4*)kb, (const uint4*)vb, tiles, (long long)(STRIDE / 16), out, evict));
      }
    };
    run();
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) run();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    const double hbm = 2.0 * units * tiles * TK * ROWB;
    printf("2pass units %d tiles %d C %d evict %d: %.1f us  %.0f GB/s (K+V once)\n", units, tiles, C, evict, ms * 1e3,
           hbm / ms / 1e6);
    return 0;
  }
  const int units = argc > 1 ? atoi(argv[1]) : 2048;   // CTAs (one head-stream each)
  const int tiles = argc > 2 ? atoi(argv[2]) : 16;     // 64-row tiles per CTA
  const size_t per_unit = (size_t)tiles * TK * STRIDE;
  const size_t bytes = per_unit * units;
  void* buf;
  CK(cudaMalloc(&buf, bytes + 4096));
  CK(cudaMemset(buf, 1, bytes));
  float* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double useful = (double)units * tiles * TK * ROWB;
  for (int mode = 0; mode <= 8; ++mode) {
    if (mode == 5 || mode == 6) continue;
    long long stride_u4 = (mode == 4) ? ROWB / 16 : STRIDE / 16;
    auto run = [&]() {
      if (mode == 0 || mode == 4) k_ldg<<<units, 256>>>((const uint4*)buf, tiles, stride_u4, out);
      if (mode == 1) { cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384);
                       k_cpasync<<<units, 256, 4 * 16384>>>((const uint4*)buf, tiles, stride_u4, out); }
      if (mode == 2) { cudaFuncSetAttribute(k_ws<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + 5 * 16384);
                       k_ws<2><<<units, 288, 128 + 5 * 16384>>>((const uint4*)buf, tiles, stride_u4, out); }
      if (mode == 3) { cudaFuncSetAttribute(k_ws<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + 5 * 16384);
                       k_ws<3><<<units, 288, 128 + 5 * 16384>>>((const uint4*)buf, tiles, stride_u4, out); }
      if (mode == 5 || mode == 6) return;  // (two-pass modes use the other entry)
      if (mode == 7) { auto k = k_ws<2, 10, 1>; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + 12 * 16384);
                       k<<<units, 288, 128 + 12 * 16384>>>((const uint4*)buf, tiles, stride_u4, out); }
      if (mode == 8) { auto k = k_ws<2, 10, 2>; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + 12 * 16384);
                       k<<<units, 320, 128 + 12 * 16384>>>((const uint4*)buf, tiles, stride_u4, out); }
    };
    run();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) run();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("mode %d units %d tiles %d: %.1f us  %.0f GB/s useful\n", mode, units, tiles, ms * 1e3, useful / ms / 1e6);
  }
  return 0;
}
