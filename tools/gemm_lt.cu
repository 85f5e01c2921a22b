// cuBLASLt algorithm sweep for the prefill / batched projections (M > 32):
// Y[M][N] = X[M][K] . W[N][K]^T with the heuristic's candidate algorithms, each
// timed on the stream over rotating weight copies (> L2), against the
// cublasGemmEx default the forward uses.  Measurement-only export
// (tools/bench_lt.py); the forward picks its algorithm in runtime.cu.
#include "deltaserve_b200.h"

#include <cublasLt.h>
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

extern "C" int ds_debug_lt_sweep(const void* X, const void* const* Ws, int n_w, void* Y, int M,
                                 int N, int K, int y_f32, int reps, ds_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cublasLtHandle_t lt = nullptr;
  if (cublasLtCreate(&lt) != CUBLAS_STATUS_SUCCESS) return 1001;
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
  const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
  const cudaDataType_t yt = y_f32 ? CUDA_R_32F : CUDA_R_16BF;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, K, N, K);
  cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, K, M, K);
  cublasLtMatrixLayoutCreate(&lc, yt, N, M, N);
  const size_t ws_bytes = 32u << 20;
  void* ws = nullptr;
  cudaMalloc(&ws, ws_bytes);
  cublasLtMatmulPreference_t pref = nullptr;
  cublasLtMatmulPreferenceCreate(&pref);
  cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes,
                                       sizeof(ws_bytes));
  std::vector<cublasLtMatmulHeuristicResult_t> res(32);
  int n_res = 0;
  cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 32, res.data(), &n_res);
  const float alpha = 1.f, beta = 0.f;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time_it = [&](auto&& fn) {
    for (int i = 0; i < 3; ++i) fn(i);
    cudaEventRecord(e0, s);
    for (int i = 0; i < reps; ++i) fn(i);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return 1000.f * ms / reps;
  };
  cublasHandle_t h = nullptr;
  cublasCreate(&h);
  cublasSetStream(h, s);
  cublasSetWorkspace(h, ws, ws_bytes);
  const float t_def = time_it([&](int i) {
    cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, &alpha, Ws[i % n_w], CUDA_R_16BF, K, X,
                 CUDA_R_16BF, K, &beta, Y, yt, N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  });
  fprintf(stderr, "M=%d N=%d K=%d gemmEx default %.2f us; %d heuristic candidates\n", M, N, K,
          t_def, n_res);
  for (int a = 0; a < n_res; ++a) {
    const float t = time_it([&](int i) {
      cublasLtMatmul(lt, op, &alpha, Ws[i % n_w], la, X, lb, &beta, Y, lc, Y, lc, &res[a].algo,
                     ws, ws_bytes, s);
    });
    int tile = 0, stages = 0, splitk = 0, cluster = 0;
    size_t w = 0;
    cublasLtMatmulAlgoConfigGetAttribute(&res[a].algo, CUBLASLT_ALGO_CONFIG_TILE_ID, &tile,
                                         sizeof(tile), &w);
    cublasLtMatmulAlgoConfigGetAttribute(&res[a].algo, CUBLASLT_ALGO_CONFIG_STAGES_ID, &stages,
                                         sizeof(stages), &w);
    cublasLtMatmulAlgoConfigGetAttribute(&res[a].algo, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &splitk,
                                         sizeof(splitk), &w);
    cublasLtMatmulAlgoConfigGetAttribute(&res[a].algo, CUBLASLT_ALGO_CONFIG_CLUSTER_SHAPE_ID,
                                         &cluster, sizeof(cluster), &w);
    fprintf(stderr, "  algo %2d: %8.2f us  tile %d stages %d splitk %d cluster %d ws %zu\n", a, t,
            tile, stages, splitk, cluster, res[a].workspaceSize);
  }
  cudaStreamSynchronize(s);
  cublasDestroy(h);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cublasLtMatmulPreferenceDestroy(pref);
  cublasLtMatrixLayoutDestroy(la);
  cublasLtMatrixLayoutDestroy(lb);
  cublasLtMatrixLayoutDestroy(lc);
  cublasLtMatmulDescDestroy(op);
  cublasLtDestroy(lt);
  cudaFree(ws);
  return static_cast<int>(cudaGetLastError());
}
