// Skinny GEMM for decode / verify: Y[M][N] (+)= X[M][K] . W[N][K]^T, M <= 32.
//
// At M = 1..17 rows (decode, verify k+1) every weight byte is used M times, so
// the projection is HBM-bound on the weight stream (the whole 8B forward is
// ~16 GB of weights).  "Swap AB" on mma.sync m16n8k16: A = 16 weight rows,
// B = X^T (8 tokens), D = 16 features x 8 tokens.  Weights are streamed
// straight from HBM into registers with 128-bit L1-bypassing loads (no smem
// round trip): lane (g, t) loads 8 consecutive k of rows g and g+8, and the
// k order inside each 32-wide chunk is permuted identically for A and B (a dot
// product is order free), so one 16-byte X load supplies both k16 steps.
// A CTA owns 16 output features; its 8 warps split K and reduce through smem.
#include "../../include/deltaserve_b200.h"
#include "common.cuh"

namespace ds {

constexpr int kGemvWarps = 8;

DS_DEVICE uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int MT, int U>
__global__ void __launch_bounds__(kGemvWarps * 32) gemm_skinny_kernel(
    const __nv_bfloat16* __restrict__ X, const __nv_bfloat16* __restrict__ W, void* __restrict__ Y,
    int M, int N, int K, int y_f32, int accumulate) {
  __shared__ float red[kGemvWarps][MT][4][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n0 = blockIdx.x * 16;
  const int kslice = K / kGemvWarps;
  const int kbeg = warp * kslice;
  const __nv_bfloat16* w0 = W + static_cast<int64_t>(n0 + g) * K + kbeg + 8 * t;
  const __nv_bfloat16* w1 = w0 + static_cast<int64_t>(8) * K;
  const __nv_bfloat16* xr[MT];
  bool xv[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int m = mt * 8 + g;
    xv[mt] = m < M;
    xr[mt] = X + static_cast<int64_t>(xv[mt] ? m : 0) * K + kbeg + 8 * t;
  }
  float acc[MT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;

  uint4 a[U][2], b[U][MT];
  // weights do not depend on the previous kernel: stream the first chunk
  // before waiting on the activations (programmatic dependent launch)
#pragma unroll
  for (int u = 0; u < U; ++u) {
    a[u][0] = ldg_stream(w0 + 32 * u);
    a[u][1] = ldg_stream(w1 + 32 * u);
  }
  pdl_wait();
  pdl_trigger();
  for (int kc = 0; kc < kslice; kc += 32 * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kc) {
        a[u][0] = ldg_stream(w0 + kc + 32 * u);
        a[u][1] = ldg_stream(w1 + kc + 32 * u);
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
        b[u][mt] = xv[mt] ? __ldg(reinterpret_cast<const uint4*>(xr[mt] + kc + 32 * u))
                          : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t s0[4] = {a[u][0].x, a[u][1].x, a[u][0].y, a[u][1].y};
      const uint32_t s1[4] = {a[u][0].z, a[u][1].z, a[u][0].w, a[u][1].w};
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        mma_bf16_16816(acc[mt], s0, b[u][mt].x, b[u][mt].y);
        mma_bf16_16816(acc[mt], s1, b[u][mt].z, b[u][mt].w);
      }
    }
  }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int q = 0; q < 4; ++q) red[warp][mt][q][lane] = acc[mt][q];
  __syncthreads();
  // thread -> (mt, q, lane) output element; sum the 8 warps' partials
  for (int idx = threadIdx.x; idx < MT * 4 * 32; idx += kGemvWarps * 32) {
    const int mt = idx / 128, q = (idx / 32) & 3, ln = idx & 31;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kGemvWarps; ++w) s += red[w][mt][q][ln];
    // c0,c1: (feature g, tokens 2t, 2t+1); c2,c3: (feature g+8, same tokens)
    const int feat = n0 + (ln >> 2) + ((q & 2) ? 8 : 0);
    const int m = mt * 8 + 2 * (ln & 3) + (q & 1);
    if (m >= M) continue;
    const int64_t o = static_cast<int64_t>(m) * N + feat;
    if (y_f32) {
      float* y = static_cast<float*>(Y) + o;
      *y = accumulate ? *y + s : s;
    } else {
      __nv_bfloat16* y = static_cast<__nv_bfloat16*>(Y) + o;
      *y = __float2bfloat16_rn(accumulate ? __bfloat162float(*y) + s : s);
    }
  }
}

template <int MT, int U>
static void launch(const void* X, const void* W, void* Y, int M, int N, int K, int y_f32, int acc,
                   cudaStream_t s) {
  launch_pdl(gemm_skinny_kernel<MT, U>, dim3(N / 16), dim3(kGemvWarps * 32), 0, s,
             static_cast<const __nv_bfloat16*>(X), static_cast<const __nv_bfloat16*>(W), Y, M, N,
             K, y_f32, acc);
}

}  // namespace ds

extern "C" int ds_gemm_skinny(const void* X, const void* W, void* Y, int M, int N, int K,
                              int y_f32, int accumulate, ds_stream_t stream) {
  if (M <= 0 || M > 32 || N % 16 || K % (32 * ds::kGemvWarps)) return DS_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const int kslice = K / ds::kGemvWarps;
  if (M <= 8) {
    if (kslice % (32 * 8) == 0) ds::launch<1, 8>(X, W, Y, M, N, K, y_f32, accumulate, s);
    else if (kslice % (32 * 4) == 0) ds::launch<1, 4>(X, W, Y, M, N, K, y_f32, accumulate, s);
    else ds::launch<1, 1>(X, W, Y, M, N, K, y_f32, accumulate, s);
  } else if (M <= 16) {
    if (kslice % (32 * 4) == 0) ds::launch<2, 4>(X, W, Y, M, N, K, y_f32, accumulate, s);
    else ds::launch<2, 1>(X, W, Y, M, N, K, y_f32, accumulate, s);
  } else {
    if (kslice % (32 * 2) == 0) ds::launch<4, 2>(X, W, Y, M, N, K, y_f32, accumulate, s);
    else ds::launch<4, 1>(X, W, Y, M, N, K, y_f32, accumulate, s);
  }
  return (int)cudaGetLastError();
}
