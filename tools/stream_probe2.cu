// Streaming-rate probe (diagnostics, not product code): how fast can one CTA pull 32 KB
// paged K tiles (128 keys x 256-byte rows at a 2 KB slot stride, 16-key pages in random
// order) into a shared-memory ring, by producer mechanism?  A consumer warp only waits for
// each tile and releases its slot, so the rate is the load path's alone.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/stream_probe2 tools/stream_probe2.cu -lcuda
//   tools/stream_probe2 <mode> <slots> <ctas_per_sm>
//   mode 0: cp.async, 1 warp   1: cp.async, 2 warps   2: cp.async, 4 warps
//        3: TMA 16-key boxes, 1 lane issues 16       4: TMA, 8 lanes issue 2 each
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

constexpr int TK = 128, D = 128, HKV = 8, TILE = TK * D * 2;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mwait(uint64_t* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void marrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void marrive_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void cpa16(uint32_t d, const void* s) { asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(s) : "memory"); }
__device__ __forceinline__ void cpa_arrive(uint64_t* b) { asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void tma3(uint32_t d, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(d), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(b)) : "memory");
}

struct Prm {
  CUtensorMap map;
  const __nv_bfloat16* k;
  const int* pages;  // [units][tiles*8] page ids
  int tiles;         // tiles per unit
  int units;
  int mode, slots, pwarps;
};

__global__ void __launch_bounds__(192) probe(const __grid_constant__ Prm p) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* ring = sm;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + p.slots * TILE);
  uint64_t* empty = full + 8;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int nprod = p.pwarps;
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.slots; ++i) minit(full + i, p.mode >= 3 ? 1 : nprod), minit(empty + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int h = blockIdx.x % HKV;
  for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
    const int* pg = p.pages + (size_t)u * p.tiles * 8;
    const int base_f = ((u - blockIdx.x) / gridDim.x) * p.tiles;
    if (warp < nprod) {
      for (int t = 0; t < p.tiles; ++t) {
        const int f = base_f + t, s = f % p.slots;
        if (f >= p.slots) mwait(empty + s, ((f / p.slots) - 1) & 1);
        const uint32_t dst = su32(ring + s * TILE);
        if (p.mode >= 3) {
          if (warp == 0) {
            const int nl = p.mode == 3 ? 1 : 8;
            if (lane == 0) marrive_tx(full + s, TILE);
            if (lane < nl) {
              for (int b = lane; b < 8; b += nl) {
                const int slot0 = pg[t * 8 + b] * 16;
                tma3(dst + b * 2048, &p.map, 0, h, slot0, full + s);
                tma3(dst + TK * 128 + b * 2048, &p.map, 64, h, slot0, full + s);
              }
            }
          }
        } else {
          const int rows = TK / nprod, r0 = warp * rows;
          const int sub = lane >> 4, c = lane & 15;
          for (int kk = 0; kk < rows / 2; ++kk) {
            const int i = r0 + 2 * kk + sub;
            const int slot = pg[t * 8 + i / 16] * 16 + (i & 15);
            cpa16(dst + (c >> 3) * (TK * 128) + i * 128 + (((c & 7) ^ (i & 7)) << 4),
                  p.k + ((size_t)slot * HKV + h) * D + c * 8);
          }
          cpa_arrive(full + s);
          __syncwarp();
          if (lane == 0) marrive(full + s);
        }
      }
    } else if (warp == 5 && lane == 0) {
      for (int t = 0; t < p.tiles; ++t) {
        const int f = base_f + t, s = f % p.slots;
        mwait(full + s, (f / p.slots) & 1);
        marrive(empty + s);
      }
    }
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int slots = argc > 2 ? atoi(argv[2]) : 4;
  const int per_sm = argc > 3 ? atoi(argv[3]) : 1;
  const int pwarps = mode == 0 ? 1 : mode == 1 ? 2 : mode == 2 ? 4 : 1;
  const int tiles = 36, units = 148 * per_sm * 8;
  const size_t n_pages = (size_t)units * tiles * 8 / HKV + 64;  // 8 heads share a page
  const size_t slots_total = n_pages * 16;
  __nv_bfloat16* k;
  cudaMalloc(&k, slots_total * HKV * D * 2);
  cudaMemset(k, 0, slots_total * HKV * D * 2);
  std::vector<int> pages((size_t)units * tiles * 8);
  std::vector<int> perm(n_pages);
  for (size_t i = 0; i < n_pages; ++i) perm[i] = (int)i;
  std::mt19937 rng(1);
  std::shuffle(perm.begin(), perm.end(), rng);
  for (int u = 0; u < units; ++u)
    for (int j = 0; j < tiles * 8; ++j) pages[(size_t)u * tiles * 8 + j] = perm[((size_t)(u / HKV) * tiles * 8 + j) % n_pages];
  int* dpages;
  cudaMalloc(&dpages, pages.size() * 4);
  cudaMemcpy(dpages, pages.data(), pages.size() * 4, cudaMemcpyHostToDevice);
  Prm p{};
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  cuuint64_t dims[3] = {D, HKV, slots_total};
  cuuint64_t str[2] = {D * 2, HKV * D * 2};
  cuuint32_t box[3] = {64, 1, 16}, es[3] = {1, 1, 1};
  ((Enc)fn)(&p.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, k, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  p.k = k, p.pages = dpages, p.tiles = tiles, p.units = units, p.mode = mode, p.slots = slots, p.pwarps = pwarps;
  const int smem = slots * TILE + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  const int grid = 148 * per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) probe<<<grid, 192, smem>>>(p);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int it = 0; it < reps; ++it) probe<<<grid, 192, smem>>>(p);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)units * tiles * TILE * reps;
  printf("mode %d slots %d ctas/SM %d: %.1f GB/s (%s)\n", mode, slots, per_sm, bytes / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
