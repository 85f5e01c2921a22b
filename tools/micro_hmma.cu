// legacy mma.sync m16n8k16 bf16 throughput: every warp of every SM issues
// independent MMAs back to back
#include <cstdio>
#include <cstdint>
__global__ void k(float* out, int iters) {
  float acc[8][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 1.f) out[0] = s;
}
// one dependent chain per warp: latency of an accumulating mma.sync
__global__ void chain(float* out, int iters, long long* cyc) {
  float acc[4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  const float s = acc[0] + acc[1] + acc[2] + acc[3];
  const long long t1 = clock64();
  if (s == 1.f) out[0] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* o; cudaMalloc(&o, 4);
  long long* cyc; cudaMalloc(&cyc, 8);
  for (int w : {1, 8}) {
    chain<<<1, 32 * w>>>(o, 4096, cyc);
    long long h; cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent mma.sync chain, %d warp(s): %.1f cycles per MMA\n", w, h / 4096.0);
  }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096;
    k<<<148, warps * 32>>>(o, iters);
    cudaEventRecord(a);
    k<<<148, warps * 32>>>(o, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flop = 148.0 * warps * iters * 8 * 4096.0;
    printf("warps/SM %2d: %.1f TFLOP/s (mma.sync m16n8k16 bf16)\n", warps, flop / ms / 1e9);
  }
}
