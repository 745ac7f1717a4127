// cuBLASLt exhaustive algorithm search (diagnostics): for the configs[1] linear-layer shapes at
// R rows, time every (algo id, tile, split-K, reduction scheme) cublasLt accepts against the
// best of the heuristic's top 8 (what csrc/forward.cu's lt_tune picks from).
//   nvcc -O2 -std=c++17 -o tools/lt_search tools/lt_search.cu -lcublasLt
//   tools/lt_search [R]
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 240;
  struct Shape { const char* name; int N, K; bool f32out; float beta; };
  Shape shapes[] = {{"qkv", 6144, 4096, false, 0.f}, {"wo", 4096, 4096, true, 1.f}, {"mlp_in", 8192, 4096, false, 0.f},
                    {"mlp_out", 4096, 8192, true, 1.f}};
  cublasLtHandle_t lt;
  cublasLtCreate(&lt);
  size_t wsz = 64 << 20;
  void* ws;
  cudaMalloc(&ws, wsz);
  void* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (const Shape& sh : shapes) {
    const int N = sh.N, K = sh.K;
    void *A, *W, *C;
    cudaMalloc(&A, (size_t)R * K * 2);
    cudaMalloc(&W, (size_t)N * K * 2);
    cudaMalloc(&C, (size_t)R * N * 4);
    cudaMemset(A, 0, (size_t)R * K * 2);
    cudaMemset(W, 0, (size_t)N * K * 2);
    cudaMemset(C, 0, (size_t)R * N * 4);
    const float alpha = 1.f, beta = sh.beta;
    const cudaDataType ct = sh.f32out ? CUDA_R_32F : CUDA_R_16BF;
    cublasLtMatmulDesc_t op;
    cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
    cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
    cublasLtMatrixLayout_t la, lb, lc;
    cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, K, N, K);
    cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, K, R, K);
    cublasLtMatrixLayoutCreate(&lc, ct, N, R, N);
    auto time_algo = [&](const cublasLtMatmulAlgo_t& algo) -> float {
      cublasLtMatmulHeuristicResult_t chk;
      if (cublasLtMatmulAlgoCheck(lt, op, la, lb, lc, lc, &algo, &chk) != CUBLAS_STATUS_SUCCESS) return -1.f;
      if (chk.workspaceSize > wsz) return -1.f;
      for (int i = 0; i < 2; ++i)
        if (cublasLtMatmul(lt, op, &alpha, W, la, A, lb, &beta, C, lc, C, lc, &algo, ws, wsz, 0) != CUBLAS_STATUS_SUCCESS)
          return -1.f;
      float tot = 0.f;
      for (int i = 0; i < 6; ++i) {
        cudaMemsetAsync(flush, i, 256 << 20);
        cudaEventRecord(e0);
        cublasLtMatmul(lt, op, &alpha, W, la, A, lb, &beta, C, lc, C, lc, &algo, ws, wsz, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      cudaGetLastError();
      return tot / 6 * 1000.f;
    };
    // heuristic top 8
    cublasLtMatmulPreference_t pref;
    cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz));
    cublasLtMatmulHeuristicResult_t res[8];
    int n = 0;
    cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 8, res, &n);
    float hbest = 1e9;
    for (int i = 0; i < n; ++i)
      if (res[i].state == CUBLAS_STATUS_SUCCESS) {
        const float us = time_algo(res[i].algo);
        if (us > 0 && us < hbest) hbest = us;
      }
    // exhaustive
    int ids[256];
    int nids = 0;
    cublasLtMatmulAlgoGetIds(lt, CUBLAS_COMPUTE_32F, CUDA_R_32F, CUDA_R_16BF, CUDA_R_16BF, ct, ct, 256, ids, &nids);
    float best = 1e9;
    int tried = 0, bid = -1, btile = -1, bsk = -1;
    for (int ii = 0; ii < nids; ++ii) {
      cublasLtMatmulAlgo_t algo;
      if (cublasLtMatmulAlgoInit(lt, CUBLAS_COMPUTE_32F, CUDA_R_32F, CUDA_R_16BF, CUDA_R_16BF, ct, ct, ids[ii], &algo) !=
          CUBLAS_STATUS_SUCCESS)
        continue;
      size_t sz = 0;
      cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_TILE_IDS, nullptr, 0, &sz);
      std::vector<int> tiles(sz / sizeof(int));
      if (!tiles.empty()) cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_TILE_IDS, tiles.data(), sz, &sz);
      if (tiles.empty()) tiles.push_back(CUBLASLT_MATMUL_TILE_UNDEFINED);
      int splitk_ok = 0;
      cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_SPLITK_SUPPORT, &splitk_ok, sizeof(splitk_ok), &sz);
      for (int tile : tiles) {
        for (int sk : {1, 2, 3, 4, 6, 8}) {
          if (sk > 1 && !splitk_ok) continue;
          cublasLtMatmulAlgo_t a2 = algo;
          cublasLtMatmulAlgoConfigSetAttribute(&a2, CUBLASLT_ALGO_CONFIG_TILE_ID, &tile, sizeof(tile));
          cublasLtMatmulAlgoConfigSetAttribute(&a2, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &sk, sizeof(sk));
          uint32_t red = sk > 1 ? CUBLASLT_REDUCTION_SCHEME_COMPUTE_TYPE : CUBLASLT_REDUCTION_SCHEME_NONE;
          cublasLtMatmulAlgoConfigSetAttribute(&a2, CUBLASLT_ALGO_CONFIG_REDUCTION_SCHEME, &red, sizeof(red));
          const float us = time_algo(a2);
          if (us <= 0) continue;
          ++tried;
          if (us < best) best = us, bid = ids[ii], btile = tile, bsk = sk;
        }
      }
    }
    printf("%-8s R=%d N=%d K=%d  heuristic-best %.1f us  exhaustive-best %.1f us (algo %d tile %d splitk %d; %d configs, %d ids) "
           "weights %.1f MB -> %.0f GB/s\n",
           sh.name, R, N, K, hbest, best, bid, btile, bsk, tried, nids, N * (double)K * 2 / 1e6,
           N * (double)K * 2 / (best < hbest ? best : hbest) / 1e3);
    fflush(stdout);
    cudaFree(A), cudaFree(W), cudaFree(C);
  }
  return 0;
}
