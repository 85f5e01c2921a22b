// Skinny GEMM for decode / verify: Y[M][N] (+)= X[M][K] . W[N][K]^T, M <= 32.
//
// At M = 1..17 rows (decode, verify k+1) every weight byte is used M times, so
// the projection is HBM-bound on the weight stream (the whole 8B forward is
// ~16 GB of weights).  Work unit = 16 output features x all of K.
//
// Data movement (TMA): persistent CTAs, two per SM (112 KB of shared memory
// each), walk the units round-robin.  One producer thread streams, per stage,
// ONE TMA box of the unit's 16 weight rows x KC columns and ONE box of the M
// activation rows (3D tensor maps over 128-byte column slabs, SWIZZLE_128B)
// into a ring of mbarrier-tracked stages; the weight boxes of the ring's first
// round are issued before the programmatic-dependency wait (weights do not
// depend on the previous kernel), so each projection's ring fills while its
// predecessor drains.  Keeping the bytes in flight in shared memory (not in
// L1 as register-streaming loads do) makes the kernel independent of the SM's
// L1/shared carveout, which the decode attention (~200 KB of shared memory)
// otherwise leaves behind - measured: the register-streaming version ran the
// forward up to 1.5x slower after a non-cluster attention launch.
//
// Math: "swap AB" mma.sync m16n8k16, A = 16 weight rows, B = X^T (8 tokens per
// n-tile), D = 16 features x 8 tokens.  Lane (g, t) reads 16 bytes at columns
// [8t, 8t+8) of a k32 step for weight rows g, g+8 and token row g (the k order
// inside a 32-column step is permuted identically for A and B - a dot product
// is order free - so one 16-byte read feeds both k16 MMAs); the swizzle makes
// those reads bank-conflict free.  8 math warps split each stage's k32 steps
// and reduce through shared memory per unit.
//
// The epilogue absorbs the layer's elementwise kernels (ds_skinny_epi):
//  * residual producer (wo, down; Y fp32 accumulate): also writes
//    h = bf16(y * h_w) - the next RMSNorm's weight multiply - and this unit's
//    per-row partial sum of y^2 over its 16 features, added into the row sums
//    in 2^-24 fixed point (integer atomics: bit-identical whatever the CTA
//    order); it also clears the other ss buffer (consumed upstream);
//  * norm consumer (wqkv, gate_up): scales row m of the product by
//    rsqrt(row sum / K + eps) - RMSNorm is a per-row scalar, so it commutes
//    with the projection;
//  * SwiGLU (gate_up with 8-row interleaved weights): feature rows g / g+8 of
//    the unit are gate / up of the same FFN unit, so the thread holding both
//    writes act = bf16(silu(g) * u) directly (half the output bytes, no
//    separate kernel);
//  * RoPE + KV store (wqkv with RoPE-pair interleaved q/k rows): rows g / g+8
//    are dims i / i+64 of one head, so the thread holding both rotates them;
//    q goes to Y, k and v straight into the paged pools (the K5 kernel).
#include "../../include/deltaserve_b200.h"
#include "attn_plan.h"
#include "common.cuh"
#include "tma.h"

namespace ds {

constexpr int kGemvWarps = 8;
constexpr float kSsScale = 16777216.f;  // 2^24 fixed point for the row sums of squares

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

// The unit epilogue: reduce the 8 warps' partial accumulators (red) of the
// 16 output features starting at n0 and apply the fused elementwise work.  Run
// by the kGemvWarps*32 math threads (threadIdx.x < 256), after a barrier that
// makes red visible; uses named barrier 1 over those threads.
template <int MT>
DS_DEVICE void unit_epilogue(const float (*red)[MT][4][32], const float* s_inv, const int* s_pos,
                             const int64_t* s_cell, float (*s_sq)[17],
                             unsigned long long* s_amax, const ds_skinny_epi& epi, void* Y, int M,
                             int N, int n0, int y_f32, int accumulate) {
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
    if (epi.argmax_out) {  // LM head: running per-row best of this CTA
      if (Y) static_cast<float*>(Y)[o] = s;
      atomicMax(&s_amax[m], argmax_key(s, feat));
      continue;
    }
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
    named_bar_sync(1, kGemvWarps * 32);
    if (threadIdx.x < M) {
      float v = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) v += s_sq[threadIdx.x][j];
      atomicAdd(reinterpret_cast<unsigned long long*>(epi.ss_out) + threadIdx.x,
                static_cast<unsigned long long>(__float2ll_rn(v * kSsScale)));
    }
  }
}

constexpr int kRingSmemBudget = 112 * 1024;  // two CTAs (two kernels) per SM

DS_DEVICE uint4 lds128(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(addr));
  return r;
}

template <int MT, int NS>  // NS = k32 steps per math warp per stage (KC = 256*NS)
__global__ void __launch_bounds__((kGemvWarps + 1) * 32, 2) gemm_ring_kernel(
    void* __restrict__ Y, int M, int N, int K, int y_f32, int accumulate, int n_stages,
    const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx,
    ds_skinny_epi epi) {
  constexpr int KC = 256 * NS;  // columns per stage = KC/64 slabs of 128 B
  constexpr int kSlabs = KC / 64;
  const int wbytes = 16 * KC * 2, xbytes = M * KC * 2;
  const int SB = (wbytes + xbytes + 1023) & ~1023;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // SW128 atoms
  float(*red)[MT][4][32] = reinterpret_cast<float(*)[MT][4][32]>(smem + n_stages * SB);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + n_stages * SB + kGemvWarps * MT * 4 * 32 * 4);
  uint64_t* empty = full + n_stages;
  __shared__ float s_inv[32];
  __shared__ float s_sq[32][17];
  __shared__ int s_pos[32];
  __shared__ int64_t s_cell[32];
  __shared__ unsigned long long s_amax[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int units = N / 16, nst = K / KC;
  if (threadIdx.x < 32) s_amax[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n_stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kGemvWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kGemvWarps) {
    // ---- producer (one thread): per stage one TMA box of 16 weight rows and
    // one of the M activation rows.  Weights do not depend on the previous
    // kernel: the ring's first round of weight boxes is issued before the
    // dependency wait, those stages' activation boxes after it ----
    if (lane == 0) {
      tma_prefetch_desc(&tw);
      tma_prefetch_desc(&tx);
      const int my_units = static_cast<int>(blockIdx.x) < units
                               ? (units - 1 - static_cast<int>(blockIdx.x)) / gridDim.x + 1 : 0;
      const int total = my_units * nst;
      const int pre = total < n_stages ? total : n_stages;
      auto unit_of = [&](int it) { return static_cast<int>(blockIdx.x) + (it / nst) * gridDim.x; };
      for (int it = 0; it < pre; ++it) {
        mbar_expect_tx(&full[it], wbytes + xbytes);
        tma_load_3d(smem + it * SB, &tw, 0, unit_of(it) * 16, (it % nst) * kSlabs, &full[it]);
      }
      if (epi.l2_pre) {  // this CTA's share of a later kernel's weights, while waiting
        const L2Hint h{{static_cast<const char*>(epi.l2_pre), nullptr}, {epi.l2_pre_bytes, 0}};
        l2_prefetch_share(h, blockIdx.x, gridDim.x);
      }
      pdl_wait();
      for (int it = 0; it < pre; ++it)
        tma_load_3d(smem + it * SB + wbytes, &tx, 0, 0, (it % nst) * kSlabs, &full[it]);
      for (int it = pre; it < total; ++it) {
        const int slot = it % n_stages, round = it / n_stages;
        mbar_wait(&empty[slot], (round - 1) & 1);
        uint8_t* st = smem + slot * SB;
        mbar_expect_tx(&full[slot], wbytes + xbytes);
        tma_load_3d(st, &tw, 0, unit_of(it) * 16, (it % nst) * kSlabs, &full[slot]);
        tma_load_3d(st + wbytes, &tx, 0, 0, (it % nst) * kSlabs, &full[slot]);
      }
      // prefetch the next kernel's first weights into L2 (optional)
      if (epi.l2_next) {
        const char* base = static_cast<const char*>(epi.l2_next);
        const int64_t share = ((epi.l2_next_bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ll;
        const int64_t lim = epi.l2_next_bytes & ~15ll;
        const int64_t beg = share * blockIdx.x;
        const int64_t end = beg + share < lim ? beg + share : lim;
        for (int64_t off = beg; off < end; off += 32768) {
          const uint32_t n = static_cast<uint32_t>(end - off < 32768 ? end - off : 32768);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(base + off), "r"(n)
                       : "memory");
        }
      }
    }
    return;
  }

  // ---- math warps ----
  const int g = lane >> 2, t = lane & 3;
  pdl_wait();  // the row scalars come from the previous kernel too
  pdl_trigger();
  if (epi.ss_zero && blockIdx.x == 0 && threadIdx.x < 32) epi.ss_zero[threadIdx.x] = 0;
  if (threadIdx.x < M) {
    if (epi.row_ss) {
      const unsigned long long rs =
          __ldcg(reinterpret_cast<const unsigned long long*>(epi.row_ss) + threadIdx.x);
      s_inv[threadIdx.x] =
          rsqrtf(__ull2float_rn(rs) / (kSsScale * static_cast<float>(K)) + epi.eps);
    }
    if (epi.rope) {
      const int r_pos = __ldg(epi.row_pos + threadIdx.x);
      const int r_seq = __ldg(epi.row_seq + threadIdx.x);
      s_pos[threadIdx.x] = r_pos;
      s_cell[threadIdx.x] =
          __ldg(epi.pos2cell + static_cast<int64_t>(r_seq) * epi.pos_stride + r_pos);
    }
  }
  // k32 step j = warp + 8i of a stage lives in slab j/2, 16-byte chunks
  // 4*(j&1) + t; smem row R holds chunk c at c ^ (R & 7) (SWIZZLE_128B)
  const uint32_t ring = smem_u32(smem);
  uint32_t a_off[NS], x_off[NS][MT];
  bool xv[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) xv[mt] = mt * 8 + g < M;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    const int j = warp + 8 * i, slab = j >> 1, c = 4 * (j & 1) + t;
    a_off[i] = slab * 2048 + g * 128 + ((c ^ g) << 4);  // row g; row g+8 is +1024
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int R = slab * M + (xv[mt] ? mt * 8 + g : 0);
      x_off[i][mt] = wbytes + R * 128 + ((c ^ (R & 7)) << 4);
    }
  }
  int it = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    float acc[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
    for (int s = 0; s < nst; ++s, ++it) {
      const int slot = it % n_stages, round = it / n_stages;
      mbar_wait(&full[slot], round & 1);
      const uint32_t st = ring + slot * SB;
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        const uint4 a0 = lds128(st + a_off[i]), a1 = lds128(st + a_off[i] + 1024);
        uint4 bx[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          bx[mt] = xv[mt] ? lds128(st + x_off[i][mt]) : make_uint4(0, 0, 0, 0);
        const uint32_t s0[4] = {a0.x, a1.x, a0.y, a1.y};
        const uint32_t s1[4] = {a0.z, a1.z, a0.w, a1.w};
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          mma_bf16_16816(acc[mt], s0, bx[mt].x, bx[mt].y);
          mma_bf16_16816(acc[mt], s1, bx[mt].z, bx[mt].w);
        }
      }
      // the reads above (generic proxy) complete before the TMA (async proxy)
      // may overwrite the slot
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[warp][mt][q][lane] = acc[mt][q];
    named_bar_sync(1, kGemvWarps * 32);
    unit_epilogue<MT>(red, s_inv, s_pos, s_cell, s_sq, s_amax, epi, Y, M, N, u * 16, y_f32,
                      accumulate);
    named_bar_sync(1, kGemvWarps * 32);  // red / s_sq reused by the next unit
  }
  // one global max per row and CTA (not per unit: 8k units on M addresses
  // would serialise in L2)
  if (epi.argmax_out && threadIdx.x < M && s_amax[threadIdx.x])
    atomicMax(reinterpret_cast<unsigned long long*>(epi.argmax_out) + threadIdx.x,
              s_amax[threadIdx.x]);
}

template <int MT, int NS>
static int launch_ring(const void* X, const void* W, void* Y, int M, int N, int K, int y_f32,
                       int acc, const ds_skinny_epi& epi, cudaStream_t s) {
  // DS_RING_KB / DS_RING_CTAS: smem budget per CTA and CTAs per SM (A/B knobs)
  static const int budget =
      getenv("DS_RING_KB") ? atoi(getenv("DS_RING_KB")) * 1024 : kRingSmemBudget;
  static const int per_sm = getenv("DS_RING_CTAS") ? atoi(getenv("DS_RING_CTAS")) : 2;
  constexpr int KC = 256 * NS;
  const int SB = ((16 + M) * KC * 2 + 1023) & ~1023;
  const int red_bytes = kGemvWarps * MT * 4 * 32 * 4;
  const int fixed = red_bytes + 4096 /* static smem */ + 1024 /* reserved */ + 1024 /* align */;
  int n_stages = (budget - fixed) / (SB + 16);
  n_stages = n_stages < 2 ? 2 : n_stages > 12 ? 12 : n_stages;
  const int smem = 1024 + n_stages * SB + red_bytes + 2 * n_stages * 8;
  const CUtensorMap* tw = slab_tensor_map(W, N, K, 16, KC / 64);
  const CUtensorMap* tx = slab_tensor_map(X, M, K, M, KC / 64);
  if (!tw || !tx) return DS_EUNSUPPORTED;
  static int attr_smem = 0;
  if (smem > attr_smem) {
    cudaFuncSetAttribute(gemm_ring_kernel<MT, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    cudaFuncSetAttribute(gemm_ring_kernel<MT, NS>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr_smem = smem;
  }
  const int units = N / 16;
  int grid = units < per_sm * kNumSMs ? units : per_sm * kNumSMs;
  // verify rows (M > 1): the fewest CTAs that keep the most-loaded CTA's unit
  // count, so every CTA walks the same number of units and none streams a
  // last unit alone (gate_up: 1,792 units on 256 CTAs x 7 instead of 296 with
  // 16 taking a 7th; qkv 192 x 2; the LM head 287 x 28).  Measured per
  // forward: q=5 at m=1k 2.821 -> 2.792 ms, 8k 3.089 -> 3.051, 32k 3.608 ->
  // 3.591; decode (M = 1) lost 2% with fewer CTAs (fewer bytes in flight) and
  // keeps the full grid.  DS_RING_BALANCE: 0 off, 2 also M = 1
  static const int balance = getenv("DS_RING_BALANCE") ? atoi(getenv("DS_RING_BALANCE")) : 1;
  if (balance && (M > 1 || balance == 2) && grid > 0 && units % grid) {
    const int upc = (units + grid - 1) / grid;
    grid = (units + upc - 1) / upc;
  }
  launch_pdl(gemm_ring_kernel<MT, NS>, dim3(grid), dim3((kGemvWarps + 1) * 32), smem, s, Y, M, N,
             K, y_f32, acc, n_stages, *tw, *tx, epi);
  return (int)cudaGetLastError();
}

template <int MT>
static int run_ring(const void* X, const void* W, void* Y, int M, int N, int K, int y_f32, int acc,
                    const ds_skinny_epi& epi, cudaStream_t s) {
  // stage width: 512 columns (measured best at M <= 16), 1024 at M > 16
  static const int ns = getenv("DS_RING_NS") ? atoi(getenv("DS_RING_NS")) : (MT == 4 ? 4 : 2);
  if (ns == 4 && K % 1024 == 0) return launch_ring<MT, 4>(X, W, Y, M, N, K, y_f32, acc, epi, s);
  if (ns == 1) return launch_ring<MT, 1>(X, W, Y, M, N, K, y_f32, acc, epi, s);
  if (MT == 4 && K % 1024 == 0) return launch_ring<MT, 4>(X, W, Y, M, N, K, y_f32, acc, epi, s);
  if (K % 512 == 0) return launch_ring<MT, 2>(X, W, Y, M, N, K, y_f32, acc, epi, s);
  return launch_ring<MT, 1>(X, W, Y, M, N, K, y_f32, acc, epi, s);
}

static int run(const void* X, const void* W, void* Y, int M, int N, int K, int y_f32, int acc,
               const ds_skinny_epi& epi, cudaStream_t s) {
  if (M <= 8) return run_ring<1>(X, W, Y, M, N, K, y_f32, acc, epi, s);
  if (M <= 16) return run_ring<2>(X, W, Y, M, N, K, y_f32, acc, epi, s);
  return run_ring<4>(X, W, Y, M, N, K, y_f32, acc, epi, s);
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
  if (epi->argmax_out && (!y_f32 || accumulate || epi->ss_out || epi->swiglu || epi->rope ||
                          epi->row_ss))
    return DS_EINVAL;
  if (!Y && !epi->argmax_out) return DS_EINVAL;
  return ds::run(X, W, Y, M, N, K, y_f32, accumulate, *epi, (cudaStream_t)stream);
}
