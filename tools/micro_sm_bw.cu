// Micro: HBM streaming rate vs the number of streaming CTAs (one per SM) and
// the bytes each keeps in flight (TMA bulk copies into an mbarrier ring), with
// an optional second stream of L2-resident "token" bytes re-read by every CTA
// at a given ratio to the streamed "weight" bytes.  Decides whether a GEMM
// with fewer weight tiles than SMs can stream the weights without split-K.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/msb tools/micro_sm_bw.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(n)
               : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          su32(d)),
      "l"(s), "r"(n), "r"(su32(b))
      : "memory");
}

__device__ __forceinline__ void tma3(void* d, const CUtensorMap* m, int c0, int c1, int c2,
                                     uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(su32(d)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(b))
      : "memory");
}
// tensor variant: W viewed as [rows][4096] bf16 = (64, rows, 64 slabs); CTA c
// owns rows [c*rpc, (c+1)*rpc) in 128-row tiles (all slabs), box (64, box_rows,
// box_slabs); n_prod producer warps split the stages round-robin.
__global__ void tensor_kernel(const __grid_constant__ CUtensorMap tm, int rpc, int box_rows,
                              int box_slabs, int n_stages, int n_prod) {
  extern __shared__ __align__(1024) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 32;
  char* ring = sm + 1024;
  const int stage = box_rows * box_slabs * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();
  const int per_row_tile = 64 / box_slabs;
  const int n_it = (rpc / box_rows) * per_row_tile;
  const int warp = threadIdx.x / 32;
  if (warp < n_prod && (threadIdx.x & 31) == 0) {
    for (int it = warp; it < n_it; it += n_prod) {
      const int s = it % n_stages;
      if (it >= n_stages) wait(&empty[s], ((it / n_stages) - 1) & 1);
      expect_tx(&full[s], stage);
      const int rt = it / per_row_tile, sl = (it % per_row_tile) * box_slabs;
      tma3(ring + s * stage, &tm, 0, blockIdx.x * rpc + rt * box_rows, sl, &full[s]);
    }
  } else if (threadIdx.x == 32 * n_prod) {
    for (int it = 0; it < n_it; ++it) {
      const int s = it % n_stages;
      wait(&full[s], (it / n_stages) & 1);
      arrive(&empty[s]);
    }
  }
}

// CTA c streams bytes [c*per, (c+1)*per) of W in `stage` chunks through
// n_stages stages; each stage also pulls `tok` bytes of X (L2-resident).
__global__ void stream_kernel(const char* W, int64_t per, const char* X, int64_t xbytes, int stage,
                              int tok, int n_stages) {
  extern __shared__ __align__(1024) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 32;
  char* ring = sm + 1024;
  if (threadIdx.x == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();
  const int64_t n_it = per / stage;
  const char* w = W + blockIdx.x * per;
  if (threadIdx.x == 0) {
    for (int64_t it = 0; it < n_it; ++it) {
      const int s = it % n_stages;
      if (it >= n_stages) wait(&empty[s], ((it / n_stages) - 1) & 1);
      expect_tx(&full[s], stage + tok);
      char* d = ring + s * (stage + tok);
      g2s(d, w + it * stage, stage, &full[s]);
      if (tok) g2s(d + stage, X + (it * tok) % xbytes, tok, &full[s]);
    }
  } else if (threadIdx.x == 32) {
    for (int64_t it = 0; it < n_it; ++it) {
      const int s = it % n_stages;
      wait(&full[s], (it / n_stages) & 1);
      arrive(&empty[s]);
    }
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int64_t total = 1ll << 30;  // 1 GB of "weights"
  char *W, *X;
  cudaMalloc(&W, total + (64 << 20));
  cudaMalloc(&X, 4 << 20);
  cudaMemset(W, 1, total);
  cudaMemset(X, 1, 4 << 20);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Cfg {
    int stage, tok, ns;
  };
  std::vector<Cfg> cfgs = {{16384, 0, 8}, {32768, 0, 6}, {65536, 0, 3}, {98304, 0, 2},
                           {4096, 0, 32}};
  for (auto c : cfgs) {
    for (int ctas : {32, 64, 148}) {
      if (ctas == 296 && (c.stage + c.tok) * c.ns > 110 * 1024) continue;
      int64_t per = (total / ctas) / c.stage * c.stage;
      int smem = 1024 + (c.stage + c.tok) * c.ns;
      if (smem > 227 * 1024) continue;
      for (int r = 0; r < 2; ++r)
        stream_kernel<<<ctas, 64, smem>>>(W, per, X, 1 << 20, c.stage, c.tok, c.ns);
      cudaEventRecord(a);
      const int reps = 5;
      for (int r = 0; r < reps; ++r)
        stream_kernel<<<ctas, 64, smem>>>(W, per, X, 1 << 20, c.stage, c.tok, c.ns);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double s = ms / 1e3 / reps;
      printf("stage %6d tok %6d stages %2d inflight %6d KB ctas %3d: HBM %7.1f GB/s (%6.1f per CTA)  L2 tok %7.1f GB/s\n",
             c.stage, c.tok, c.ns, (c.stage + c.tok) * c.ns / 1024, ctas, per * ctas / s / 1e9,
             per / s / 1e9, (double)per / c.stage * c.tok * ctas / s / 1e9);
    }
  }
  // tensor maps
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int64_t rows = total / 8192;  // [rows][4096] bf16
  cudaFuncSetAttribute(tensor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct TC { int box_rows, box_slabs, ns, np; };
  std::vector<TC> tcs = {{128, 1, 8, 1}, {128, 1, 12, 1}, {128, 2, 6, 1}, {128, 4, 3, 1},
                         {256, 1, 6, 1}, {128, 1, 12, 2}, {128, 1, 12, 4}, {128, 2, 6, 2}};
  for (auto c : tcs) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, 64};
    cuuint64_t strides[2] = {8192, 128};
    cuuint32_t box[3] = {64, (cuuint32_t)c.box_rows, (cuuint32_t)c.box_slabs};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, W, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); continue; }
    const int stage = c.box_rows * c.box_slabs * 128;
    for (int ctas : {32, 48, 64, 96, 148}) {
      int rpc = (int)(rows / ctas) / 256 * 256;
      int smem = 1024 + stage * c.ns;
      if (smem > 227 * 1024) continue;
      for (int r2 = 0; r2 < 2; ++r2)
        tensor_kernel<<<ctas, 32 * (c.np + 1), smem>>>(tm, rpc, c.box_rows, c.box_slabs, c.ns, c.np);
      cudaEventRecord(a);
      const int reps = 5;
      for (int r2 = 0; r2 < reps; ++r2)
        tensor_kernel<<<ctas, 32 * (c.np + 1), smem>>>(tm, rpc, c.box_rows, c.box_slabs, c.ns, c.np);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double s = ms / 1e3 / reps;
      double by = (double)rpc * 8192 * ctas;
      printf("tensor box %3dx%d (%6d B) stages %2d prod %d ctas %3d: HBM %7.1f GB/s (%6.1f per CTA)\n",
             c.box_rows, c.box_slabs, stage, c.ns, c.np, ctas, by / s / 1e9, by / ctas / s / 1e9);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
}
