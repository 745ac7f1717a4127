// cuBLASLt algorithm probe (diagnostics): for the configs[1] linear-layer shapes at R rows,
// time every heuristic candidate cublasLt offers against the default cublasGemmEx choice.
//   nvcc -O2 -std=c++17 -o tools/lt_probe tools/lt_probe.cu -lcublasLt -lcublas
//   tools/lt_probe [R]
#include <cublasLt.h>
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 228;
  struct Shape { const char* name; int N, K; bool f32out; float beta; };
  Shape shapes[] = {{"qkv", 6144, 4096, false, 0.f}, {"wo", 4096, 4096, true, 1.f}, {"mlp_in", 8192, 4096, false, 0.f},
                    {"mlp_out", 4096, 8192, true, 1.f}, {"lm_head", 151936, 4096, true, 0.f}};
  cublasLtHandle_t lt;
  cublasLtCreate(&lt);
  cublasHandle_t hb;
  cublasCreate(&hb);
  size_t wsz = 64 << 20;
  void* ws;
  cudaMalloc(&ws, wsz);
  cublasSetWorkspace(hb, ws, wsz);
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
    auto time_it = [&](auto fn) {
      for (int i = 0; i < 3; ++i) fn();
      float tot = 0.f;
      for (int i = 0; i < 10; ++i) {
        cudaMemsetAsync(flush, i, 256 << 20);
        cudaEventRecord(e0);
        fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      return tot / 10 * 1000.f;
    };
    const float us_def = time_it([&] {
      cublasGemmEx(hb, CUBLAS_OP_T, CUBLAS_OP_N, N, R, K, &alpha, W, CUDA_R_16BF, K, A, CUDA_R_16BF, K, &beta, C, ct, N,
                   CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    });
    cublasLtMatmulDesc_t op;
    cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
    cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
    cublasLtMatrixLayout_t la, lb, lc;
    cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, K, N, K);
    cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, K, R, K);
    cublasLtMatrixLayoutCreate(&lc, ct, N, R, N);
    cublasLtMatmulPreference_t pref;
    cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz));
    cublasLtMatmulHeuristicResult_t res[32];
    int n = 0;
    cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 32, res, &n);
    float best = 1e9;
    int besti = -1;
    for (int i = 0; i < n; ++i) {
      if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
      const float us = time_it([&] {
        cublasLtMatmul(lt, op, &alpha, W, la, A, lb, &beta, C, lc, C, lc, &res[i].algo, ws, wsz, 0);
      });
      if (us < best) best = us, besti = i;
    }
    printf("%-8s R=%d N=%d K=%d  default %.1f us  lt-best %.1f us (candidate %d of %d; weights %.1f MB -> %.0f GB/s)\n",
           sh.name, R, N, K, us_def, best, besti, n, N * (double)K * 2 / 1e6, N * (double)K * 2 / best / 1e3);
    cudaFree(A), cudaFree(W), cudaFree(C);
  }
  return 0;
}
