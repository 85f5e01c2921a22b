// K6: delta-prefill attention on the 5th-generation tensor cores (tcgen05).
//
// Delta new query tokens attend causally over an m-token prefix that lives in
// the paged (head-major) cell pool.  Work unit = (128 packed query rows, KV
// head, key split): GQA packing puts the G query heads of 128/G consecutive
// positions in the M=128 rows, so every K/V tile is loaded once for all G
// heads.  Two CTAs share an SM (256 TMEM columns and ~112 KB smem each), so
// one CTA's softmax overlaps the other's tensor-core work.  Warp roles:
//   warp 0  TMA producer: per 64-key tile, two 2D TMA boxes each for K and
//           V (128-byte column halves, SWIZZLE_128B) when the tile's cells
//           form one run, else a cell-by-cell cp.async gather into the same
//           layout.  K and V have their own rings (3 and 2 stages): a K stage
//           frees as soon as its S = QK^T MMA completes, so K loads run three
//           tiles ahead of the MMAs and V loads two - the load latency no
//           longer gates the tensor pipe (with one shared 2-stage K|V ring the
//           softmax warps sat ~45% of the time waiting for S).
//   warp 1  MMA issuer (one elected thread): S_j = Q.K_j^T (M=128, N=64, K=128;
//           8 x tcgen05.mma kind::f16, K-major SW128 descriptors) into a
//           double-buffered TMEM S; O += P_j.V_j with P read straight from
//           TMEM (the "TS" form; B = V MN-major) into a TMEM-resident O;
//           completion through tcgen05.commit.  S_{j+1} is issued before PV_j.
//   warps 2-5 softmax (thread = TMEM lane = query row): batched tcgen05.ld of
//           the S row, online softmax in the log2 domain (scale folded into one
//           FFMA per element), causal masking only on diagonal tiles, P (bf16)
//           written back over its own S columns with one tcgen05.st - no smem
//           round trip and no wait on the previous PV.  The running max is
//           raised only when it grows by more than 2^8, so the O rescale in
//           TMEM is rare.
// Long contexts are split over keys so the grid fills whole waves of
// 2 x 148 CTAs; attn_prefill_combine merges the (O, lse) partials.
#include "../../include/deltaserve_b200.h"
#include "common.cuh"
#include "tc.cuh"
#include "tma.h"

#include <cstdio>
#include <cstdlib>

namespace ds {

namespace {
constexpr int kD = 128;
constexpr int kBM = 128;                    // packed query rows per CTA
constexpr int kBN = 64;                     // keys per tile
constexpr int kQHalf = kBM * 128;           // Q: 64-column half of [128 rows][128 d] (16 KB)
constexpr int kKHalf = kBN * 128;           // K/V: 64-column half of [64 keys][128 d] (8 KB)
constexpr int kKStages = 3, kVStages = 2;
constexpr int kThreads = 6 * 32;
constexpr int kSmemQ = 0;                             // 32 KB
constexpr int kSmemK = 2 * kQHalf;                    // K ring: 3 x 16 KB
constexpr int kSmemV = kSmemK + kKStages * 2 * kKHalf;  // V ring: 2 x 16 KB
constexpr int kSmemBar = kSmemV + kVStages * 2 * kKHalf;  // 112 KB: two CTAs per SM
constexpr int kSmemBytes = kSmemBar + 128;
constexpr int kTmemCols = 256;  // S0/P0 [0,64) S1/P1 [64,128) O [128,256)
constexpr int kMaxSplits = 64;
#ifndef DS_K6_POLY
#define DS_K6_POLY 0
#endif
#ifndef DS_K6_F32X2  // packed FFMA2 / FADD2 in the softmax (0: scalar, the poly A/B path)
#define DS_K6_F32X2 (DS_K6_POLY == 0)
#endif
#if DS_K6_F32X2 && DS_K6_POLY
#error "DS_K6_POLY (FMA-pipe exponentials) is implemented on the scalar softmax: set DS_K6_F32X2=0"
#endif
constexpr int kPolyPeriod = DS_K6_POLY;  // see the softmax loop
constexpr int kMaxPartialCtas = 8 * 148;  // bounds the split-partial workspace

// 16-byte chunk c (0..15 over d) of row r in a tile of `rows` rows, SW128
DS_DEVICE int sw128(int rows, int row, int chunk16) {
  return (chunk16 >> 3) * rows * 128 + row * 128 + (((chunk16 & 7) ^ (row & 7)) << 4);
}
}  // namespace

// partial output slot of (entry e, split s, q-block qb, kv head kh): 128 rows
DS_DEVICE int64_t prefill_slot(int e, int s, int qb, int kh, int splits, int max_qb, int nkv) {
  return ((static_cast<int64_t>(e) * splits + s) * max_qb + qb) * nkv + kh;
}

__global__ void __launch_bounds__(kThreads, 2) attn_prefill_kernel(
    const __nv_bfloat16* __restrict__ qkv, int qkv_stride, const ds_entry* __restrict__ entries,
    const __nv_bfloat16* __restrict__ kpool, const __nv_bfloat16* __restrict__ vpool,
    int64_t head_stride, const int32_t* __restrict__ pos2cell, int64_t pos_stride, int nh,
    int nkv, float scale_log2, __nv_bfloat16* __restrict__ out, int splits, int max_qb,
    float* __restrict__ part_o, float* __restrict__ part_lse,
    const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
  uint64_t* k_full = bars;        // [3]
  uint64_t* k_empty = bars + 3;   // [3]
  uint64_t* v_full = bars + 6;    // [2]
  uint64_t* v_empty = bars + 8;   // [2]
  uint64_t* s_full = bars + 10;   // [2]
  uint64_t* pv_done = bars + 12;  // PV_j complete: P_j's TMEM columns free, O stable
  uint64_t* p_full = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  uint64_t* q_ready = bars + 15;  // the softmax warps' Q rows are in smem
  if (smem_u32(smem) & 1023) __trap();  // SW128 tiles need 1 KB alignment
  // programmatic dependent launch: only q and this chunk's own K/V rows come
  // from the preceding kernels (projection, RoPE/KV store) - the prologue and
  // the tiles of older keys run before the dependency wait (producer: before
  // the first tile holding new keys; softmax warps: before loading q)
  pdl_trigger();

  const int e = blockIdx.z / splits;
  const int split = blockIdx.z - e * splits;
  const ds_entry en = entries[e];
  const int G = nh / nkv;
  const int ppb = kBM / G;  // positions per block
  const int qb = blockIdx.x;
  const int t0 = qb * ppb;
  if (t0 >= en.q_len) return;
  const int kh = blockIdx.y;
  const int t_last = min(en.q_len, t0 + ppb) - 1;
  const int kv_len = en.past + en.q_len;
  const int kv_hi = en.past + t_last + 1;  // keys any row of this block can see
  const int ntiles_all = (kv_hi + kBN - 1) / kBN;
  const int per = (ntiles_all + splits - 1) / splits;
  const int j0 = split * per;
  const int j1 = min(ntiles_all, j0 + per);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntiles = j0 >= j1 ? 0 : j1 - j0;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
    mbar_init(pv_done, 1);
    mbar_init(p_full, 4);
    mbar_init(q_ready, 128);
    mbar_fence_init();
  }
  if (warp == 1) tc::alloc(tmem_slot, kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const int32_t* p2c = pos2cell + static_cast<int64_t>(en.seq) * pos_stride;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      tma_prefetch_desc(&tmk);
      tma_prefetch_desc(&tmv);
    }
    const int64_t hrow = kh * head_stride;
    // tile cells: one contiguous run -> TMA boxes, else a cp.async gather
    struct Cells {
      int lo, hi, c0;
      bool run;
    };
    auto cells = [&](int jj) {
      const int kt = (j0 + jj) * kBN;
      const int nvalid = min(kBN, kv_hi - kt);
      Cells c;
      c.lo = lane < nvalid ? __ldg(p2c + kt + lane) : -1;
      c.hi = lane + 32 < nvalid ? __ldg(p2c + kt + 32 + lane) : -1;
      c.c0 = __shfl_sync(0xffffffffu, c.lo, 0);
      c.run = __all_sync(0xffffffffu, (c.lo < 0 || c.lo == c.c0 + lane) &&
                                          (c.hi < 0 || c.hi == c.c0 + 32 + lane));
      return c;
    };
    auto load = [&](const Cells& c, const CUtensorMap* map, const __nv_bfloat16* pool,
                    uint8_t* dst, uint64_t* full) {
      if (c.run) {
        if (lane == 0) {
          mbar_expect_tx(full, 2 * kKHalf);
          const int row = static_cast<int>(hrow + c.c0);
          tma_load_2d(dst, map, 0, row, full);
          tma_load_2d(dst + kKHalf, map, 64, row, full);
        }
      } else {
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          const int r = lane + 32 * h;
          const int cv = h ? c.hi : c.lo;
          const int64_t off = (hrow + (cv >= 0 ? cv : c.c0)) * kD;
#pragma unroll
          for (int q = 0; q < 16; ++q) cp_async16(dst + sw128(kBN, r, q), pool + off + q * 8);
        }
        cp_async_commit();
        cp_async_wait<0>();
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(full);
      }
    };
    auto load_v = [&](int jj, const Cells& c) {
      const int st = jj % kVStages;
      if (jj >= kVStages) mbar_wait(&v_empty[st], ((jj / kVStages) - 1) & 1);
      load(c, &tmv, vpool, smem + kSmemV + st * 2 * kKHalf, &v_full[st]);
    };
    // K_jj, then V_{jj-1}: V lags one tile (it is consumed a softmax later)
    bool waited = false;
    auto wait_if_new = [&](int jj) {  // before the first tile holding this chunk's K/V
      if (!waited && min((j0 + jj + 1) * kBN, kv_hi) > en.past) {
        pdl_wait();
        waited = true;
      }
    };
    Cells prev{};
    for (int jj = 0; jj < ntiles; ++jj) {
      const Cells c = cells(jj);
      const int st = jj % kKStages;
      if (jj >= kKStages) mbar_wait(&k_empty[st], ((jj / kKStages) - 1) & 1);
      wait_if_new(jj);
      load(c, &tmk, kpool, smem + kSmemK + st * 2 * kKHalf, &k_full[st]);
      if (jj > 0) load_v(jj - 1, prev);
      prev = c;
    }
    if (ntiles > 0) load_v(ntiles - 1, prev);
  } else if (warp == 1) {
    // ======================= MMA issuer =======================
    if (lane == 0 && ntiles > 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16(kBM, kBN, false);
      constexpr uint32_t idesc_pv = tc::idesc_bf16(kBM, kD, true);
      const uint32_t q_base = smem_u32(smem + kSmemQ);
      const uint32_t k_base = smem_u32(smem + kSmemK);
      const uint32_t v_base = smem_u32(smem + kSmemV);
      auto issue_s = [&](int jj) {
        const int st = jj % kKStages, sb = jj & 1;
        mbar_wait(&k_full[st], (jj / kKStages) & 1);
        // S/P buffer sb was last read by PV_{jj-2}, issued (in order) before us
        tc::fence_after();
        const uint32_t kb = k_base + st * 2 * kKHalf;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          tc::mma(tmem + sb * kBN,
                  tc::smem_desc(q_base + (kk >> 2) * kQHalf + (kk & 3) * 32, 16, 1024),
                  tc::smem_desc(kb + (kk >> 2) * kKHalf + (kk & 3) * 32, 16, 1024), idesc_s,
                  kk > 0);
        }
        tc::commit(&s_full[sb]);
        tc::commit(&k_empty[st]);  // K stage free once S_jj's MMAs complete
      };
      mbar_wait(q_ready, 0);  // the Q tile is in smem
      tc::fence_after();
      issue_s(0);
      for (int jj = 0; jj < ntiles; ++jj) {
        if (jj + 1 < ntiles) issue_s(jj + 1);
        const int st = jj % kVStages;
        mbar_wait(p_full, jj & 1);
        mbar_wait(&v_full[st], (jj / kVStages) & 1);
        tc::fence_after();
        const uint32_t vb = v_base + st * 2 * kKHalf;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          tc::mma_ts(tmem + 2 * kBN, tmem + (jj & 1) * kBN + kk * 8,
                     tc::smem_desc(vb + kk * 2048, kKHalf, 1024), idesc_pv, (jj | kk) > 0);
        }
        tc::commit(pv_done);
        tc::commit(&v_empty[st]);
      }
    }
  } else {
    // ================ softmax / epilogue ================
    {  // Q rows (packed r = t*G + g) -> smem, UMMA A layout; after the CTA
       // barrier, so the producer streams the older keys' tiles meanwhile
      pdl_wait();
      const int r = tid - 64;
      const int t = t0 + r / G, g = r - (r / G) * G;
      const bool ok = t < en.q_len;
      const uint4* src = reinterpret_cast<const uint4*>(
          qkv + static_cast<int64_t>(en.q_start + (ok ? t : 0)) * qkv_stride + (kh * G + g) * kD);
      uint4 qv[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) qv[c] = ok ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < 16; ++c) *reinterpret_cast<uint4*>(smem + kSmemQ + sw128(kBM, r, c)) = qv[c];
      tc::fence_proxy_async();  // generic smem writes -> visible to the tensor core
      mbar_arrive(q_ready);
    }
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int r = quad * 32 + lane;
    const int t = t0 + r / G, g = r - (r / G) * G;
    const int pos = en.past + t;  // absolute position of this row (causal bound)
    const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    const uint32_t tO = trow + 2 * kBN;
    const int blk_pos_min = en.past + t0;
    float m_ref = -INFINITY, l_run = 0.f;
    uint32_t sv[kD];
    for (int jj = 0; jj < ntiles; ++jj) {
      const int sb = jj & 1;
      const int kt = (j0 + jj) * kBN;
      mbar_wait(&s_full[sb], (jj >> 1) & 1);
      tc::fence_after();
      tc::ld32_issue(trow + sb * kBN, sv);
      tc::ld32_issue(trow + sb * kBN + 32, sv + 32);
      tc::wait_ld();
      const bool need_mask = (kt + kBN - 1 > blk_pos_min) || (kt + kBN > kv_len);
      if (need_mask) {
#pragma unroll
        for (int i = 0; i < kBN; ++i)
          if (!(kt + i <= pos && kt + i < kv_len)) sv[i] = __float_as_uint(-INFINITY);
      }
      // max of raw scores (scale > 0 commutes with max); 8 independent chains
      // instead of one 64-long dependent FMNMX chain
      float mpart[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) mpart[c] = __uint_as_float(sv[c]);
#pragma unroll
      for (int i = 8; i < kBN; ++i) mpart[i & 7] = fmaxf(mpart[i & 7], __uint_as_float(sv[i]));
      const float mraw = fmaxf(fmaxf(fmaxf(mpart[0], mpart[1]), fmaxf(mpart[2], mpart[3])),
                               fmaxf(fmaxf(mpart[4], mpart[5]), fmaxf(mpart[6], mpart[7])));
      const float mx = mraw * scale_log2;
      const float new_ref = (mx > m_ref + 8.f) ? mx : m_ref;
      const float scale_old = (m_ref == -INFINITY) ? 0.f : fast_exp2(m_ref - new_ref);
      const float mref = new_ref == -INFINITY ? 0.f : new_ref;
      float spart[4] = {0.f, 0.f, 0.f, 0.f};  // independent partial sums
      uint32_t pk[kBN / 2];
      // every kPolyPeriod-th pair of exponentials on the FMA pipe (0 = all on
      // the MUFU, the default: offloading 1/8, 1/4, 1/2 measured 2.4%, 6%,
      // 15% slower at delta=881 over 31.5k keys - the MUFU is not the limit,
      // the per-tile softmax dependency chain is)
#if DS_K6_F32X2
      // packed FFMA2 / FADD2 (sm_100): the scale-subtract and the row sums two
      // columns per instruction - 5 instead of 7 per column pair; K6 at
      // delta=881 over 31.5k keys 459 -> 447 us (1.00 -> 1.03 PFLOP/s)
      uint64_t acc2[2] = {0ull, 0ull};
      uint64_t sc2, mr2;
      asm("mov.b64 %0, {%1, %1};" : "=l"(sc2) : "f"(scale_log2));
      asm("mov.b64 %0, {%1, %1};" : "=l"(mr2) : "f"(-mref));
#pragma unroll
      for (int i = 0; i < kBN; i += 2) {
        uint64_t sx, x2;
        asm("mov.b64 %0, {%1, %2};" : "=l"(sx) : "r"(sv[i]), "r"(sv[i + 1]));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(x2) : "l"(sx), "l"(sc2), "l"(mr2));
        float x0, x1;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(x0), "=f"(x1) : "l"(x2));
        const float p0 = fast_exp2(x0), p1 = fast_exp2(x1);
        uint64_t pp;
        asm("mov.b64 %0, {%1, %2};" : "=l"(pp) : "f"(p0), "f"(p1));
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc2[(i / 2) & 1]) : "l"(pp));
        pk[i / 2] = pack_bf16(p0, p1);
      }
      float a0, a1, a2, a3;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc2[0]));
      asm("mov.b64 {%0, %1}, %2;" : "=f"(a2), "=f"(a3) : "l"(acc2[1]));
      (void)spart;
      const float sum = (a0 + a1) + (a2 + a3);
#else
#pragma unroll
      for (int i = 0; i < kBN; i += 2) {
        const bool poly = kPolyPeriod > 0 && (i / 2) % (kPolyPeriod > 0 ? kPolyPeriod : 1) ==
                                                 (kPolyPeriod > 0 ? kPolyPeriod - 1 : 0);
        const float x0 = fmaf(__uint_as_float(sv[i]), scale_log2, -mref);
        const float x1 = fmaf(__uint_as_float(sv[i + 1]), scale_log2, -mref);
        const float p0 = poly ? poly_exp2(x0) : fast_exp2(x0);
        const float p1 = poly ? poly_exp2(x1) : fast_exp2(x1);
        spart[(i / 2) & 3] += p0 + p1;
        pk[i / 2] = pack_bf16(p0, p1);
      }
      const float sum = (spart[0] + spart[1]) + (spart[2] + spart[3]);
#endif
      tc::st32(trow + sb * kBN, pk);  // P_j over its own S columns
      // PV_{j-1} done (O stable) before an O correction and before PV_j is issued
      if (jj > 0) {
        mbar_wait(pv_done, (jj - 1) & 1);
        tc::fence_after();
      }
      if (jj > 0 && __any_sync(0xffffffffu, new_ref != m_ref)) {  // rare O correction
        uint32_t ov[32];
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
          tc::ld32_issue(tO + cc * 32, ov);
          tc::wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * scale_old);
          tc::st32(tO + cc * 32, ov);
        }
      }
      tc::wait_st();
      l_run = l_run * scale_old + sum;
      m_ref = new_ref;
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    if (ntiles > 0) {
      mbar_wait(pv_done, (ntiles - 1) & 1);
      tc::fence_after();
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) tc::ld32_issue(tO + cc * 32, sv + cc * 32);
      tc::wait_ld();
    }
    const float* o = reinterpret_cast<const float*>(sv);
    if (splits == 1) {
      if (t < en.q_len) {
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        uint4* dst = reinterpret_cast<uint4*>(
            out + static_cast<int64_t>(en.q_start + t) * nh * kD + (kh * G + g) * kD);
#pragma unroll
        for (int q = 0; q < 16; ++q)
          dst[q] = make_uint4(pack_bf16(o[8 * q] * inv, o[8 * q + 1] * inv),
                              pack_bf16(o[8 * q + 2] * inv, o[8 * q + 3] * inv),
                              pack_bf16(o[8 * q + 4] * inv, o[8 * q + 5] * inv),
                              pack_bf16(o[8 * q + 6] * inv, o[8 * q + 7] * inv));
      }
    } else {
      const int64_t slot = prefill_slot(e, split, qb, kh, splits, max_qb, nkv) * kBM + r;
      const bool any = ntiles > 0 && l_run > 0.f;
      const float inv = any ? 1.f / l_run : 0.f;
      float4* dst = reinterpret_cast<float4*>(part_o + slot * kD);
#pragma unroll
      for (int q = 0; q < 32; ++q)
        dst[q] = make_float4(any ? o[4 * q] * inv : 0.f, any ? o[4 * q + 1] * inv : 0.f,
                             any ? o[4 * q + 2] * inv : 0.f, any ? o[4 * q + 3] * inv : 0.f);
      part_lse[slot] = any ? m_ref + __log2f(l_run) : -INFINITY;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::dealloc(tmem, kTmemCols);
  }
}

// merge key-split partials: out = sum_s 2^(lse_s - max) O_s / sum_s 2^(lse_s - max).
// One warp per packed row (lane = 4 head-dim columns); split loops unrolled so
// the L2 loads of different splits overlap.
__global__ void __launch_bounds__(256) attn_prefill_combine(
    const ds_entry* __restrict__ entries, int splits, int max_qb, int nh, int nkv,
    const float* __restrict__ part_o, const float* __restrict__ part_lse,
    __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int e = blockIdx.z, kh = blockIdx.y;
  const int qb = blockIdx.x >> 4;                          // 16 blocks x 8 rows per q-block
  const int r = ((blockIdx.x & 15) << 3) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const ds_entry en = entries[e];
  const int G = nh / nkv;
  const int t = qb * (kBM / G) + r / G, g = r - (r / G) * G;
  if (t >= en.q_len) return;
  const int64_t s0 = prefill_slot(e, 0, qb, kh, splits, max_qb, nkv) * kBM + r;
  const int64_t ss = static_cast<int64_t>(max_qb) * nkv * kBM;  // slot stride between splits
  float mx = -INFINITY;
#pragma unroll 8
  for (int s = 0; s < splits; ++s) mx = fmaxf(mx, __ldcg(part_lse + s0 + s * ss));
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float wsum = 0.f;
#pragma unroll 8
  for (int s = 0; s < splits; ++s) {
    const int64_t slot = s0 + s * ss;
    const float lse = __ldcg(part_lse + slot);
    const float w = lse == -INFINITY ? 0.f : exp2f(lse - mx);
    const float4 v = __ldcg(reinterpret_cast<const float4*>(part_o + slot * kD) + lane);
    wsum += w;
    acc.x += w * v.x; acc.y += w * v.y; acc.z += w * v.z; acc.w += w * v.w;
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  uint2* dst = reinterpret_cast<uint2*>(out + static_cast<int64_t>(en.q_start + t) * nh * kD +
                                        (kh * G + g) * kD) + lane;
  *dst = make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
}

// key splits (>= 8 tiles each).  A single wave of 2 CTAs per SM that is
// >= 85% full wins outright: short query blocks (delta ~150) are latency
// bound, and a second wave or more splits (more combine traffic) cost more
// than the idle slots (measured at delta=150: 7 splits 6.89 ms per forward
// at m=32k, 22 splits 8.03, 14 splits 7.44); otherwise the split count that
// best fills whole waves.
static int prefill_splits(int ctas, int max_tiles) {
  const long slots = 2L * 148;
  int one = 0;
  for (int s = 1; s <= kMaxSplits && static_cast<long>(ctas) * s <= slots; ++s)
    if (s == 1 || max_tiles / s >= 8) one = s;
  // ... as long as a split's key range of every head stays L2-resident while
  // all query blocks stream it (<= 96 tiles: 8 heads x 6k keys x 512 B =
  // 25 MB): one split over a 32k prefix has every CTA stream the whole 134 MB
  // from HBM (C4 prefill 22 -> 38 ms per chunk when delta >= 1009 took it)
  if (one > 0 && static_cast<double>(ctas) * one >= 0.85 * slots &&
      (max_tiles + one - 1) / one <= 96)
    return one;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= kMaxSplits; ++s) {
    if (s > 1 && (max_tiles / s < 8 || ctas * s > kMaxPartialCtas)) break;
    const long total = static_cast<long>(ctas) * s;
    const long waves = (total + slots - 1) / slots;
    const double eff = static_cast<double>(total) / static_cast<double>(waves * slots);
    if (eff > best_eff + 1e-3) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

int launch_attn_prefill_sm100(const void* qkv, const ds_entry* entries_host,
                              const ds_entry* entries_dev, int n_entries, const void* k_pool,
                              const void* v_pool, int64_t head_stride, const int32_t* pos2cell,
                              int64_t pos_stride, int nh, int nkv, int hd, float scale, void* out,
                              void* workspace, size_t ws_bytes, cudaStream_t stream) {
  if (hd != kD || nh % nkv || kBM % (nh / nkv)) return DS_EUNSUPPORTED;
  const CUtensorMap* tk = kv_tensor_map(k_pool, static_cast<int64_t>(nkv) * head_stride, kBN);
  const CUtensorMap* tv = kv_tensor_map(v_pool, static_cast<int64_t>(nkv) * head_stride, kBN);
  if (!tk || !tv) return DS_EUNSUPPORTED;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmemBytes);
    attr = true;
  }
  const int ppb = kBM / (nh / nkv);
  int max_qb = 0, qb_total = 0, max_tiles = 0;
  for (int e = 0; e < n_entries; ++e) {
    const ds_entry& en = entries_host[e];
    const int qb = (en.q_len + ppb - 1) / ppb;
    max_qb = qb > max_qb ? qb : max_qb;
    qb_total += qb;
    const int tiles = (en.past + en.q_len + kBN - 1) / kBN;
    max_tiles = tiles > max_tiles ? tiles : max_tiles;
  }
  constexpr size_t kCounterBytes = 64 << 10;  // reserved for the decode split counters
  workspace = static_cast<uint8_t*>(workspace) + kCounterBytes;
  ws_bytes = ws_bytes > kCounterBytes ? ws_bytes - kCounterBytes : 0;
  static const int splits_env = getenv("DS_K6_SPLITS") ? atoi(getenv("DS_K6_SPLITS")) : 0;
  int splits = splits_env > 0 ? splits_env : prefill_splits(qb_total * nkv, max_tiles);
  if (getenv("DS_K6_VERBOSE"))
    fprintf(stderr, "K6 ctas=%d max_tiles=%d splits=%d\n", qb_total * nkv, max_tiles, splits);
  const size_t need = static_cast<size_t>(n_entries) * splits * max_qb * nkv * kBM *
                      (kD + 1) * sizeof(float);
  if (splits > 1 && need > ws_bytes) splits = 1;
  float* part_o = static_cast<float*>(workspace);
  float* part_lse =
      part_o + static_cast<size_t>(n_entries) * splits * max_qb * nkv * kBM * kD;
  dim3 grid(max_qb, nkv, n_entries * splits);
  cudaError_t err = launch_pdl(
      attn_prefill_kernel, grid, dim3(kThreads), kSmemBytes, stream,
      static_cast<const __nv_bfloat16*>(qkv), (nh + 2 * nkv) * kD, entries_dev,
      static_cast<const __nv_bfloat16*>(k_pool), static_cast<const __nv_bfloat16*>(v_pool),
      head_stride, pos2cell, pos_stride, nh, nkv, scale * 1.4426950408889634f,
      static_cast<__nv_bfloat16*>(out), splits, max_qb, part_o, part_lse, *tk, *tv);
  if (err != cudaSuccess) return static_cast<int>(err);
  if (splits > 1) {
    err = launch_pdl(attn_prefill_combine, dim3(max_qb * 16, nkv, n_entries), dim3(256), 0, stream,
                     entries_dev, splits, max_qb, nh, nkv, (const float*)part_o,
                     (const float*)part_lse, static_cast<__nv_bfloat16*>(out));
    if (err != cudaSuccess) return static_cast<int>(err);
  }
  return (int)cudaGetLastError();
}

size_t prefill_partial_bytes_bound() {
  return static_cast<size_t>(kMaxPartialCtas) * kBM * (kD + 1) * sizeof(float);
}

}  // namespace ds
