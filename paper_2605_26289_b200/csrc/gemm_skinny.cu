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
// The activation operand (L2-resident) is software-pipelined one chunk ahead
// in registers so its latency never serialises the MMAs; rows >= M are
// predicated off (no load).
//
// The epilogue absorbs the layer's elementwise kernels (ds_skinny_epi):
//  * residual producer (wo, down; Y fp32 accumulate): also writes
//    h = bf16(y * h_w) - the next RMSNorm's weight multiply - and this CTA's
//    per-row partial sum of y^2 over its 16 features, added into the row sums
//    in 2^-24 fixed point (integer atomics: bit-identical whatever the CTA
//    order); it also clears the other ss buffer (consumed upstream);
//  * norm consumer (wqkv, gate_up): scales row m of the product by
//    rsqrt(row sum / K + eps) - RMSNorm is a per-row scalar, so it commutes
//    with the projection.  The row sum is loaded before the main loop and
//    only consumed in the epilogue (no exposed latency);
//  * SwiGLU (gate_up with 8-row interleaved weights): feature rows g / g+8 of
//    the CTA are gate / up of the same FFN unit, so the thread holding both
//    writes act = bf16(silu(g) * u) directly (half the output bytes, no
//    separate kernel);
//  * RoPE + KV store (wqkv with RoPE-pair interleaved q/k rows): rows g / g+8
//    are dims i / i+64 of one head, so the thread holding both rotates them;
//    q goes to Y, k and v straight into the paged pools (the K5 kernel).
#include "../../include/deltaserve_b200.h"
#include "common.cuh"

namespace ds {

constexpr int kGemvWarps = 8;
constexpr float kSsScale = 16777216.f;  // 2^24 fixed point for the row sums of squares

DS_DEVICE uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// predicated 16-byte activation load (zeros when off), no branch
DS_DEVICE uint4 ldg_pred(const void* p, bool on) {
  uint4 r = make_uint4(0, 0, 0, 0);
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n"
      " @q ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n}\n"
      : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
      : "l"(p), "r"(static_cast<int>(on)));
  return r;
}

DS_DEVICE float bf16r(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

// RoPE + KV store epilogue (head_dim 128; see the header comment)
template <int MT>
DS_DEVICE void rope_epilogue(const float (*red)[MT][4][32], const float* s_inv, const int* s_pos,
                             const int64_t* s_cell, const ds_skinny_epi& epi, void* Y, int M,
                             int N, int n0) {
  constexpr int kHd = 128, kHalf = 64;
  const int qk_width = (epi.n_heads + epi.n_kv_heads) * kHd;
  __nv_bfloat16* kp = static_cast<__nv_bfloat16*>(epi.k_pool_l);
  __nv_bfloat16* vp = static_cast<__nv_bfloat16*>(epi.v_pool_l);
  if (n0 < qk_width) {
    const int head = n0 / kHd, t = (n0 % kHd) / 16;
    for (int idx = threadIdx.x; idx < MT * 2 * 32; idx += kGemvWarps * 32) {
      const int mt = idx / 64, q = (idx / 32) & 1, ln = idx & 31;
      const int m = mt * 8 + 2 * (ln & 3) + q;
      if (m >= M) continue;
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int w = 0; w < kGemvWarps; ++w) {
        s1 += red[w][mt][q][ln];
        s2 += red[w][mt][q + 2][ln];
      }
      if (epi.row_ss) {
        s1 *= s_inv[m];
        s2 *= s_inv[m];
      }
      const float x1 = bf16r(s1), x2 = bf16r(s2);  // the unfused path stores qkv in bf16
      const int i = 8 * t + (ln >> 2);
      const int64_t tp = static_cast<int64_t>(s_pos[m]) * kHalf + i;
      const float c = __ldg(epi.rope_cos + tp), sn = __ldg(epi.rope_sin + tp);
      const __nv_bfloat16 y1 = __float2bfloat16_rn(x1 * c - x2 * sn);
      const __nv_bfloat16 y2 = __float2bfloat16_rn(x2 * c + x1 * sn);
      __nv_bfloat16* dst;
      if (head < epi.n_heads)
        dst = static_cast<__nv_bfloat16*>(Y) + static_cast<int64_t>(m) * N + head * kHd;
      else
        dst = kp + ((head - epi.n_heads) * epi.kv_head_stride + s_cell[m]) * kHd;
      dst[i] = y1;
      dst[i + kHalf] = y2;
    }
  } else {
    for (int idx = threadIdx.x; idx < MT * 4 * 32; idx += kGemvWarps * 32) {
      const int mt = idx / 128, q = (idx / 32) & 3, ln = idx & 31;
      const int m = mt * 8 + 2 * (ln & 3) + (q & 1);
      if (m >= M) continue;
      const int f = n0 - qk_width + (ln >> 2) + ((q & 2) ? 8 : 0);
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kGemvWarps; ++w) s += red[w][mt][q][ln];
      if (epi.row_ss) s *= s_inv[m];
      vp[((f / kHd) * epi.kv_head_stride + s_cell[m]) * kHd + f % kHd] = __float2bfloat16_rn(s);
    }
  }
}

template <int MT, int U>
__global__ void __launch_bounds__(kGemvWarps * 32) gemm_skinny_kernel(
    const __nv_bfloat16* __restrict__ X, const __nv_bfloat16* __restrict__ W, void* __restrict__ Y,
    int M, int N, int K, int y_f32, int accumulate, ds_skinny_epi epi) {
  __shared__ float red[kGemvWarps][MT][4][32];
  __shared__ float s_inv[32];
  __shared__ float s_sq[32][17];
  __shared__ int s_pos[32];
  __shared__ int64_t s_cell[32];
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

  uint4 a[U][2], bn[U][MT];
  // weights do not depend on the previous kernel: stream the first chunk
  // before waiting on the activations (programmatic dependent launch)
#pragma unroll
  for (int u = 0; u < U; ++u) {
    a[u][0] = ldg_stream(w0 + 32 * u);
    a[u][1] = ldg_stream(w1 + 32 * u);
  }
  pdl_wait();
  pdl_trigger();
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) bn[u][mt] = ldg_pred(xr[mt] + 32 * u, xv[mt]);
  if (epi.ss_zero && blockIdx.x == 0 && threadIdx.x < 32) epi.ss_zero[threadIdx.x] = 0;
  // norm consumer: the producer's row sum of squares, needed only in the epilogue
  const unsigned long long row_sum =
      epi.row_ss && threadIdx.x < M ? __ldcg(reinterpret_cast<const unsigned long long*>(epi.row_ss) + threadIdx.x) : 0ull;
  // RoPE/KV store: row positions and sequences (the cell lookup waits for the epilogue)
  int r_pos = 0, r_seq = 0;
  if (epi.rope && threadIdx.x < M) {
    r_pos = __ldg(epi.row_pos + threadIdx.x);
    r_seq = __ldg(epi.row_seq + threadIdx.x);
  }

  for (int kc = 0; kc < kslice; kc += 32 * U) {
    if (kc) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u][0] = ldg_stream(w0 + kc + 32 * u);
        a[u][1] = ldg_stream(w1 + kc + 32 * u);
      }
    }
    uint4 b[U][MT];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) b[u][mt] = bn[u][mt];
    // next chunk (the last iteration re-reads its own chunk: harmless, branch-free)
    const int kn = kc + 32 * U < kslice ? kc + 32 * U : kc;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) bn[u][mt] = ldg_pred(xr[mt] + kn + 32 * u, xv[mt]);
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
  if (epi.row_ss && threadIdx.x < M)
    s_inv[threadIdx.x] =
        rsqrtf(__ull2float_rn(row_sum) / (kSsScale * static_cast<float>(K)) + epi.eps);
  if (epi.rope && threadIdx.x < M) {
    s_pos[threadIdx.x] = r_pos;
    s_cell[threadIdx.x] = __ldg(epi.pos2cell + static_cast<int64_t>(r_seq) * epi.pos_stride + r_pos);
  }
  __syncthreads();
  if (epi.rope) {
    rope_epilogue<MT>(red, s_inv, s_pos, s_cell, epi, Y, M, N, n0);
    return;
  }
  // accumulator element (mt, q, ln): c0,c1 = (feature g, tokens 2t, 2t+1);
  // c2,c3 = (feature g+8, same tokens)
  if (epi.swiglu) {
    // (q, q+2) hold gate / up of FFN unit n0/2 + g for the same token
    for (int idx = threadIdx.x; idx < MT * 2 * 32; idx += kGemvWarps * 32) {
      const int mt = idx / 64, q = (idx / 32) & 1, ln = idx & 31;
      const int m = mt * 8 + 2 * (ln & 3) + q;
      if (m >= M) continue;
      float sg = 0.f, su = 0.f;
#pragma unroll
      for (int w = 0; w < kGemvWarps; ++w) {
        sg += red[w][mt][q][ln];
        su += red[w][mt][q + 2][ln];
      }
      if (epi.row_ss) {
        sg *= s_inv[m];
        su *= s_inv[m];
      }
      const float gg = bf16r(sg), uu = bf16r(su);  // the unfused path stores gate|up in bf16
      static_cast<__nv_bfloat16*>(Y)[static_cast<int64_t>(m) * (N / 2) + n0 / 2 + (ln >> 2)] =
          __float2bfloat16_rn(gg / (1.f + expf(-gg)) * uu);
    }
    return;
  }
  for (int idx = threadIdx.x; idx < MT * 4 * 32; idx += kGemvWarps * 32) {
    const int mt = idx / 128, q = (idx / 32) & 3, ln = idx & 31;
    const int fl = (ln >> 2) + ((q & 2) ? 8 : 0);  // feature within the CTA
    const int feat = n0 + fl;
    const int m = mt * 8 + 2 * (ln & 3) + (q & 1);
    if (m >= M) continue;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kGemvWarps; ++w) s += red[w][mt][q][ln];
    if (epi.row_ss) s *= s_inv[m];
    const int64_t o = static_cast<int64_t>(m) * N + feat;
    float y;
    if (y_f32) {
      float* yp = static_cast<float*>(Y) + o;
      y = accumulate ? *yp + s : s;
      *yp = y;
    } else {
      __nv_bfloat16* yp = static_cast<__nv_bfloat16*>(Y) + o;
      const __nv_bfloat16 yb = __float2bfloat16_rn(accumulate ? __bfloat162float(*yp) + s : s);
      *yp = yb;
      y = __bfloat162float(yb);
    }
    if (epi.ss_out) {  // residual producer: the next RMSNorm's weight multiply + partial sums
      if (epi.h_out)
        static_cast<__nv_bfloat16*>(epi.h_out)[o] =
            __float2bfloat16_rn(y * __bfloat162float(static_cast<const __nv_bfloat16*>(epi.h_w)[feat]));
      s_sq[m][fl] = y * y;
    }
  }
  if (epi.ss_out) {
    __syncthreads();
    if (threadIdx.x < M) {
      float v = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) v += s_sq[threadIdx.x][j];
      atomicAdd(reinterpret_cast<unsigned long long*>(epi.ss_out) + threadIdx.x,
                static_cast<unsigned long long>(__float2ll_rn(v * kSsScale)));
    }
  }
}

template <int MT, int U>
static void launch(const void* X, const void* W, void* Y, int M, int N, int K, int y_f32, int acc,
                   const ds_skinny_epi& epi, cudaStream_t s) {
  const int kslice = K / kGemvWarps;
  if constexpr (U > 1) {
    if (kslice % (32 * U)) {
      launch<MT, U / 2>(X, W, Y, M, N, K, y_f32, acc, epi, s);
      return;
    }
  }
  launch_pdl(gemm_skinny_kernel<MT, U>, dim3(N / 16), dim3(kGemvWarps * 32), 0, s,
             static_cast<const __nv_bfloat16*>(X), static_cast<const __nv_bfloat16*>(W), Y, M, N,
             K, y_f32, acc, epi);
}

static int run(const void* X, const void* W, void* Y, int M, int N, int K, int y_f32, int acc,
               const ds_skinny_epi& epi, cudaStream_t s) {
  if (M <= 8) launch<1, 8>(X, W, Y, M, N, K, y_f32, acc, epi, s);
  else if (M <= 16) launch<2, 4>(X, W, Y, M, N, K, y_f32, acc, epi, s);
  else launch<4, 2>(X, W, Y, M, N, K, y_f32, acc, epi, s);
  return (int)cudaGetLastError();
}

}  // namespace ds

extern "C" int ds_gemm_skinny(const void* X, const void* W, void* Y, int M, int N, int K,
                              int y_f32, int accumulate, ds_stream_t stream) {
  if (M <= 0 || M > 32 || N % 16 || K % (32 * ds::kGemvWarps)) return DS_EINVAL;
  const ds_skinny_epi none{};
  return ds::run(X, W, Y, M, N, K, y_f32, accumulate, none, (cudaStream_t)stream);
}

extern "C" int ds_gemm_skinny_ex(const void* X, const void* W, void* Y, int M, int N, int K,
                                 int y_f32, int accumulate, const ds_skinny_epi* epi,
                                 ds_stream_t stream) {
  if (M <= 0 || M > 32 || N % 16 || K % (32 * ds::kGemvWarps) || !epi) return DS_EINVAL;
  if (epi->swiglu && (y_f32 || accumulate || epi->ss_out)) return DS_EINVAL;
  if (epi->rope && (y_f32 || accumulate || epi->ss_out || epi->swiglu || epi->n_kv_heads <= 0 ||
                    N != (epi->n_heads + 2 * epi->n_kv_heads) * 128 || !epi->row_seq ||
                    !epi->row_pos || !epi->pos2cell || !epi->rope_cos || !epi->rope_sin ||
                    !epi->k_pool_l || !epi->v_pool_l))
    return DS_EINVAL;
  if (epi->ss_out && !y_f32) return DS_EINVAL;
  if (epi->h_out && (!epi->ss_out || !epi->h_w)) return DS_EINVAL;
  return ds::run(X, W, Y, M, N, K, y_f32, accumulate, *epi, (cudaStream_t)stream);
}
