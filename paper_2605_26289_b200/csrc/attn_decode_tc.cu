// K7-tc: decode / speculative verify on the 5th-generation tensor cores, for
// 8 < R <= 24 packed query rows (q = 3..6 with G = 4) over long prefixes.
//
// At R = 20 the mma.sync K7 keeps the legacy HMMA pipe ~66% busy and reaches
// only ~58% of HBM at m = 32k; tcgen05 has ~15x that tensor throughput, so
// here the rows are padded to M = 128 and the kernel stays HBM-bound:
//   warp 0  softmax + epilogue: TMEM lanes 0-31 = packed rows 0-31 (one
//           thread per row; the padding rows' P is never read back)
//   warp 1  TMA producer: per 128-key tile two boxes for K and two for V
//           (SWIZZLE_128B) when the cells form one run, else a cp.async
//           gather; K ring 3 x 32 KB (a stage frees when its QK^T completes),
//           V ring 2 x 32 KB; tiles of older keys are streamed before the PDL
//           wait (only this batch's own K/V rows come from the projection)
//   warp 2  MMA issuer: S_j = Q.K_j^T (M=128, N=128, K=128) into a
//           double-buffered TMEM S; P_j (bf16) is written back over S_j and
//           O += P_j.V_j runs as the TS-form MMA (A from TMEM) into a
//           TMEM-resident O; S_{j+1} is issued before PV_j.
// Same split plan, partial layout and in-cluster DSMEM merge as K7.
#include "../../include/deltaserve_b200.h"
#include "attn_decode_merge.cuh"
#include "attn_plan.h"
#include "common.cuh"
#include "tc.cuh"
#include "tma.h"

#include <cstdio>
#include <cstdlib>

namespace ds {

#ifdef DS_K7_TRACE
// debug build only: per-CTA globaltimer stamps (tools/k7tc_trace.py)
__device__ unsigned long long g_k7tc_trace[1024][8];
DS_DEVICE unsigned long long gtime_tc() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TC_STAMP(i)                                                                        \
  if (threadIdx.x == 0)                                                                    \
  g_k7tc_trace[(blockIdx.z * gridDim.y + blockIdx.y) & 1023][i] = gtime_tc()
#else
#define TC_STAMP(i)
#endif

namespace {
constexpr int kD = 128;
constexpr int kBM = 128;                       // MMA rows (R <= 24 real, rest padding)
constexpr int kBN = 128;                       // keys per tile
constexpr int kHalf = kBN * 128;               // 64-column half of a [128][128] bf16 tile
constexpr int kTileBytes = 2 * kHalf;          // 32 KB
#ifndef DS_K7TC_KST  // K / V ring depths (A/B); K + V <= 6 stages of 32 KB
#define DS_K7TC_KST 3
#endif
#ifndef DS_K7TC_VST
#define DS_K7TC_VST 3
#endif
constexpr int kKStages = DS_K7TC_KST, kVStages = DS_K7TC_VST;
static_assert(kKStages + kVStages <= 6 && kKStages >= 2 && kVStages >= 2, "K7-tc ring");
constexpr int kSmemQ = 0;  // 32 KB
// shared-memory layout of a KS-stage K ring and a VS-stage V ring (one CTA per
// SM; a one-stage variant beside the next projection's CTA, as K7's, measured
// no faster: C2 26.66 vs 26.69 turns/s)
template <int KS, int VS>
struct TcLayout {
  static constexpr int kK = kSmemQ + kTileBytes;
  static constexpr int kV = kK + KS * kTileBytes;
  static constexpr int kBar = kV + VS * kTileBytes;
  static constexpr int kBytes = kBar + 256 + 1024;  // + barriers, + 1 KB alignment slack
};
constexpr int kSmemBytes = TcLayout<kKStages, kVStages>::kBytes;
constexpr int kThreads = 4 * 32;  // softmax, K producer, MMA, V producer
constexpr int kTmemCols = 512;  // S0 [0,128) S1 [128,256) O [256,384)
constexpr int kMaxRows = kDecodeMaxRows;

DS_DEVICE int sw128(int rows, int row, int chunk16) {
  return (chunk16 >> 3) * rows * 128 + row * 128 + (((chunk16 & 7) ^ (row & 7)) << 4);
}
}  // namespace

int decode_tc_smem_bytes() { return kSmemBytes; }

template <int KS, int VS>
__global__ void __launch_bounds__(kThreads, 1) attn_decode_tc_kernel(
    const __nv_bfloat16* __restrict__ qkv, int qkv_stride, const ds_entry* __restrict__ entries,
    int n_entries, int max_splits, const __nv_bfloat16* __restrict__ kpool,
    const __nv_bfloat16* __restrict__ vpool, const int32_t* __restrict__ pos2cell,
    int64_t pos_stride, int nh, int nkv, float scale_log2, __nv_bfloat16* __restrict__ out,
    float* __restrict__ part_o, float* __restrict__ part_lse, int64_t head_stride,
    const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
    const L2Hint l2, int cluster) {
  using Lay = TcLayout<KS, VS>;
  TC_STAMP(6);
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // SW128 alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::kBar);
  uint64_t* k_full = bars;  // [KS]
  uint64_t* k_empty = k_full + KS;
  uint64_t* v_full = k_empty + KS;
  uint64_t* v_empty = v_full + VS;
  uint64_t* s_full = v_empty + VS;  // [2]
  uint64_t* pv_done = s_full + 2;
  uint64_t* p_full = pv_done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_full + 1);
  // split-merge buffers over the K ring (free once the last PV completed)
  float* cval = reinterpret_cast<float*>(smem + Lay::kK);  // [R][128]
  float* clse = cval + kMaxRows * kD;                     // [R]
  float* cw = clse + kMaxRows;                            // [R][kDecodeMaxCluster]

  const int e = blockIdx.z / max_splits;
  const int split = blockIdx.z - e * max_splits;
  const ds_entry en = entries[e];
  const int G = nh / nkv;
  const int R = en.q_len * G;
  const int kv_len = en.past + en.q_len;
  const AttnSplitPlan plan = attn_split_plan(1, kv_len, nkv, n_entries, 1, R);
  const bool active = split < plan.n_splits;  // idle CTAs still join the cluster merge
  const bool cluster_merge = cluster > 0;  // launched with clusters of `cluster` splits
  const int kh = blockIdx.y;
  const int k_begin = split * plan.split_len;
  const int k_end = min(k_begin + plan.split_len, kv_len);
  const int ntiles = active ? (k_end - k_begin + kBN - 1) / kBN : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 1 && lane == 0) {
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
    mbar_init(pv_done, 1);
    mbar_init(p_full, 1);
    mbar_fence_init();
  }
  if (warp == 2) tc::alloc(tmem_slot, kTmemCols);
  // padding q rows [32, 128) are zero (their S/P rows are never read, but the
  // MMA reads the whole tile)
  for (int c = tid; c < (kBM - 32) * 16; c += kThreads) {
    const int r = 32 + (c >> 4), ch = c & 15;
    *reinterpret_cast<uint4*>(smem + kSmemQ + sw128(kBM, r, ch)) = make_uint4(0, 0, 0, 0);
  }
  tc::fence_proxy_async();  // generic smem writes -> visible to the tensor core
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const int32_t* p2c = pos2cell + static_cast<int64_t>(en.seq) * pos_stride;

  if (!active) {
  } else if (warp == 1 || warp == 3) {
    // =========== TMA producers: K tiles (warp 1), V tiles (warp 3) ===========
    // separate issuing threads: a V load waits only for its own ring (the PV
    // that frees it), never behind a K load waiting for the K ring
    const bool is_v = warp == 3;
    if (lane == 0) tma_prefetch_desc(is_v ? &tmv : &tmk);
    const int64_t hrow = kh * head_stride;
    struct Cells {
      int c[4], c0;
      bool run;
    };
    // page-table entries of a tile: loaded two tiles ahead (raw), resolved
    // (run detection) when the tile is issued - their latency would otherwise
    // serialise every TMA issue (ncu: the producer's top stall)
    auto cells_load = [&](int jj, int (&c)[4]) {
      const int kt = k_begin + jj * kBN;
      const int nvalid = jj < ntiles ? min(kBN, k_end - kt) : 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i] = lane + 32 * i < nvalid ? __ldg(p2c + kt + lane + 32 * i) : -1;
    };
    auto cells_resolve = [&](const int (&c)[4]) {
      Cells cc;
      bool mine = true;
#pragma unroll
      for (int i = 0; i < 4; ++i) cc.c[i] = c[i];
      cc.c0 = __shfl_sync(0xffffffffu, cc.c[0], 0);
#pragma unroll
      for (int i = 0; i < 4; ++i) mine &= cc.c[i] < 0 || cc.c[i] == cc.c0 + lane + 32 * i;
      cc.run = __all_sync(0xffffffffu, mine);
      return cc;
    };
    auto load = [&](const Cells& cc, const CUtensorMap* map, const __nv_bfloat16* pool,
                    uint8_t* dst, uint64_t* full) {
      if (cc.run) {
        if (lane == 0) {
          mbar_expect_tx(full, kTileBytes);
          const int row = static_cast<int>(hrow + cc.c0);
          tma_load_2d(dst, map, 0, row, full);
          tma_load_2d(dst + kHalf, map, 64, row, full);
        }
      } else {
#pragma unroll 1
        for (int i = 0; i < 4; ++i) {
          const int r = lane + 32 * i;
          const int64_t off = (hrow + (cc.c[i] >= 0 ? cc.c[i] : cc.c0)) * kD;
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
    bool waited = false;
    const int n_st = is_v ? VS : KS;
    uint64_t* fulls = is_v ? v_full : k_full;
    uint64_t* empties = is_v ? v_empty : k_empty;
    uint8_t* ring = smem + (is_v ? Lay::kV : Lay::kK);
    int raw0[4], raw1[4], raw2[4];
    cells_load(0, raw0);
    cells_load(1, raw1);
    for (int jj = 0; jj < ntiles; ++jj) {
      cells_load(jj + 2, raw2);
      const Cells cc = cells_resolve(raw0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        raw0[i] = raw1[i];
        raw1[i] = raw2[i];
      }
      const int st = jj % n_st;
      if (jj >= n_st) mbar_wait(&empties[st], ((jj / n_st) - 1) & 1);
      const int kt = k_begin + jj * kBN;
      if (!waited && min(kt + kBN, k_end) > en.past) {  // this batch's own K/V rows
        pdl_wait();
        waited = true;
      }
      load(cc, is_v ? &tmv : &tmk, is_v ? vpool : kpool, ring + st * kTileBytes, &fulls[st]);
    }
    if (!waited) pdl_wait();
    if (!is_v) {
      if (!cluster_merge) pdl_trigger();
      if (lane == 0)  // this CTA's share of the next projections' weights -> L2
        l2_prefetch_share(l2, blockIdx.z * gridDim.y + blockIdx.y,
                          static_cast<int64_t>(gridDim.y) * gridDim.z);
    }
  } else if (warp == 2) {
    // ======================= MMA issuer =======================
    if (lane == 0 && ntiles > 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16(kBM, kBN, false);
      constexpr uint32_t idesc_pv = tc::idesc_bf16(kBM, kD, true);
      const uint32_t q_base = smem_u32(smem + kSmemQ);
      const uint32_t k_base = smem_u32(smem + Lay::kK);
      const uint32_t v_base = smem_u32(smem + Lay::kV);
      mbar_wait(p_full, 0);  // q staged (the softmax warp's first p_full phase)
      tc::fence_after();
      auto issue_s = [&](int jj) {
        const int st = jj % KS, sb = jj & 1;
        mbar_wait(&k_full[st], (jj / KS) & 1);
        tc::fence_after();
        const uint32_t kb = k_base + st * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          tc::mma(tmem + sb * kBN,
                  tc::smem_desc(q_base + (kk >> 2) * (kBM * 128) + (kk & 3) * 32, 16, 1024),
                  tc::smem_desc(kb + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024), idesc_s,
                  kk > 0);
        tc::commit(&s_full[sb]);
        tc::commit(&k_empty[st]);  // K stage free once S_jj's MMAs complete
      };
      issue_s(0);
      for (int jj = 0; jj < ntiles; ++jj) {
        if (jj + 1 < ntiles) issue_s(jj + 1);
        const int st = jj % VS;
        mbar_wait(p_full, (jj + 1) & 1);  // P_jj (completion jj + 1)
        mbar_wait(&v_full[st], (jj / VS) & 1);
        tc::fence_after();
        const uint32_t vb = v_base + st * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          tc::mma_ts(tmem + 2 * kBN, tmem + (jj & 1) * kBN + kk * 8,
                     tc::smem_desc(vb + kk * 2048, kHalf, 1024), idesc_pv, (jj | kk) > 0);
        tc::commit(pv_done);
        tc::commit(&v_empty[st]);
      }
    }
  } else {
    // ================ softmax / epilogue (warp 0: rows 0-31) ================
    TC_STAMP(0);
    pdl_wait();  // q comes from the preceding projection
    TC_STAMP(1);
    if (!cluster_merge) pdl_trigger();
    const int r = lane;
    const bool real = r < R;
    {  // q row r -> smem (UMMA A layout); rows >= R zero
      const uint4* src = reinterpret_cast<const uint4*>(
          qkv + static_cast<int64_t>(en.q_start + (real ? r / G : 0)) * qkv_stride +
          (kh * G + (real ? r % G : 0)) * kD);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const uint4 v = real ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(smem + kSmemQ + sw128(kBM, r, c)) = v;
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);  // phase 0: q staged
    }
    const int pos = real ? en.past + r / G : -1;  // causal bound of this row
    const uint32_t trow = tmem;                    // lanes 0-31
    const uint32_t tO = trow + 2 * kBN;
    float m_ref = -INFINITY, l_run = 0.f;
    uint32_t sv[kBN];
    for (int jj = 0; jj < ntiles; ++jj) {
      const int sb = jj & 1;
      const int kt = k_begin + jj * kBN;
      mbar_wait(&s_full[sb], (jj >> 1) & 1);
      if (jj == 0) TC_STAMP(2);
      tc::fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) tc::ld32_issue(trow + sb * kBN + 32 * c, sv + 32 * c);
      tc::wait_ld();
      const bool need_mask = (kt + kBN - 1 > en.past) || (kt + kBN > k_end);
      if (need_mask) {
#pragma unroll
        for (int i = 0; i < kBN; ++i)
          if (!(kt + i <= pos && kt + i < k_end)) sv[i] = __float_as_uint(-INFINITY);
      }
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
      float spart[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < kBN; i += 2) {
        const float p0 = fast_exp2(fmaf(__uint_as_float(sv[i]), scale_log2, -mref));
        const float p1 = fast_exp2(fmaf(__uint_as_float(sv[i + 1]), scale_log2, -mref));
        spart[(i / 2) & 3] += p0 + p1;
        sv[i / 2] = pack_bf16(p0, p1);  // P (bf16 pairs) reuses the low registers
      }
      const float sum = (spart[0] + spart[1]) + (spart[2] + spart[3]);
      tc::st32(trow + sb * kBN, sv);        // P_j over its own S columns
      tc::st32(trow + sb * kBN + 32, sv + 32);
      if (jj > 0) {  // PV_{j-1} done (O stable) before a correction / PV_j
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
    TC_STAMP(3);
    mbar_wait(pv_done, (ntiles - 1) & 1);
    tc::fence_after();
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) tc::ld32_issue(tO + cc * 32, sv + 32 * cc);
    tc::wait_ld();
    const float* o = reinterpret_cast<const float*>(sv);
    const bool any = l_run > 0.f;
    const float inv = any ? 1.f / l_run : 0.f;
    if (real) {
      if (plan.n_splits == 1) {
        const int ti = r / G, gi = r - ti * G;
        uint4* dst = reinterpret_cast<uint4*>(
            out + static_cast<int64_t>(en.q_start + ti) * nh * kD + (kh * G + gi) * kD);
#pragma unroll
        for (int q = 0; q < 16; ++q)
          dst[q] = make_uint4(pack_bf16(o[8 * q] * inv, o[8 * q + 1] * inv),
                              pack_bf16(o[8 * q + 2] * inv, o[8 * q + 3] * inv),
                              pack_bf16(o[8 * q + 4] * inv, o[8 * q + 5] * inv),
                              pack_bf16(o[8 * q + 6] * inv, o[8 * q + 7] * inv));
      } else {
        const float lse = any ? m_ref + __log2f(l_run) : -INFINITY;
        float* dst;
        if (cluster_merge) {
          dst = cval + r * kD;
          clse[r] = lse;
        } else {
          const int64_t base = attn_partial_base(entries, e, n_entries, nh, nkv, 1);
          const int64_t slot = (base + static_cast<int64_t>(split) * R + r) * nkv + kh;
          dst = part_o + slot * kD;
          part_lse[slot] = lse;
        }
#pragma unroll
        for (int q = 0; q < 32; ++q)
          reinterpret_cast<float4*>(dst)[q] =
              make_float4(o[4 * q] * inv, o[4 * q + 1] * inv, o[4 * q + 2] * inv,
                          o[4 * q + 3] * inv);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after();
    tc::dealloc(tmem, kTmemCols);
  }
  if (cluster_merge && plan.n_splits > 1) {
    cluster_sync_all();  // every split's rows are in its cluster buffer
    decode_cluster_merge<kDecodeTcMaxCluster>(cval, clse, cw, R, plan.n_splits, cluster, tid,
                                              kThreads, 1, en, nh, kh, G, out);
    cluster_sync_all();  // peers keep their smem until every read is done
  }
  // PDL: see K7 (triggers only as the grid retires; more splits than a
  // cluster are merged by attn_combine_kernel, R > 8 here)
  TC_STAMP(5);
  pdl_trigger();
}

#ifdef DS_K7_TRACE
extern "C" int ds_debug_k7tc_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_k7tc_trace, sizeof(g_k7tc_trace));
}
#endif

// clusters of `size` CTAs of the K7-tc kernel co-resident on the GPU (0: none)
static int tc_max_clusters(int size) {
  static int cache[17] = {};
  if (size < 1 || size > 16) return 0;
  if (cache[size]) return cache[size] > 0 ? cache[size] : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1, 1, size);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = size;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, attn_decode_tc_kernel<kKStages, kVStages>, &cfg) !=
      cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[size] = n > 0 ? n : -1;
  return n;
}

int launch_attn_decode_tc(const ds_entry* entries_dev, int n_entries, const void* qkv,
                          const void* k_pool, const void* v_pool, int64_t head_stride,
                          const int32_t* pos2cell, int64_t pos_stride, int nh, int nkv,
                          int max_splits, int max_split_len, float scale, void* out,
                          float* part_o, float* part_lse, const L2Hint& l2, int* merged,
                          cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_tc_kernel<kKStages, kVStages>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    cudaFuncSetAttribute(attn_decode_tc_kernel<kKStages, kVStages>,
                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  const CUtensorMap* tk = kv_tensor_map(k_pool, static_cast<int64_t>(nkv) * head_stride, kBN);
  const CUtensorMap* tv = kv_tensor_map(v_pool, static_cast<int64_t>(nkv) * head_stride, kBN);
  if (!tk || !tv) return DS_EUNSUPPORTED;
  dim3 grid(1, nkv, n_entries * max_splits);
  const float sl2 = scale * 1.4426950408889634f;
  const int stride = (nh + 2 * nkv) * kD;
  // the splits of one (entry, kv head) merge in one cluster: up to 8 always,
  // up to kDecodeTcMaxCluster when every cluster of the grid is co-resident
  int cluster = 0;
  if (max_splits <= kDecodeMaxCluster)
    cluster = max_splits;
  else if (max_splits <= kDecodeTcMaxCluster && tc_max_clusters(max_splits) >= nkv * n_entries)
    cluster = max_splits;
  *merged = cluster > 0;
  static const bool verbose = getenv("DS_K7_VERBOSE") != nullptr;
  static bool once = false;
  if (verbose && !once) {
    once = true;
    for (int c = 8; c <= 16; ++c) fprintf(stderr, "K7-tc cluster %d: %d co-resident\n", c, tc_max_clusters(c));
  }
  if (verbose)
    fprintf(stderr, "K7-tc: %d entries x %d kv heads, %d splits, cluster %d (co-resident %d)\n",
            n_entries, nkv, max_splits, cluster,
            max_splits <= 16 ? tc_max_clusters(max_splits) : 0);
  auto kern = attn_decode_tc_kernel<kKStages, kVStages>;
  if (cluster)
    launch_pdl_cluster_z(kern, grid, dim3(kThreads), kSmemBytes, cluster, stream,
                         static_cast<const __nv_bfloat16*>(qkv), stride, entries_dev, n_entries,
                         max_splits, static_cast<const __nv_bfloat16*>(k_pool),
                         static_cast<const __nv_bfloat16*>(v_pool), pos2cell, pos_stride, nh,
                         nkv, sl2, static_cast<__nv_bfloat16*>(out), part_o, part_lse,
                         head_stride, *tk, *tv, l2, cluster);
  else
    launch_pdl(kern, grid, dim3(kThreads), kSmemBytes, stream,
               static_cast<const __nv_bfloat16*>(qkv), stride, entries_dev, n_entries, max_splits,
               static_cast<const __nv_bfloat16*>(k_pool),
               static_cast<const __nv_bfloat16*>(v_pool), pos2cell, pos_stride, nh, nkv, sl2,
               static_cast<__nv_bfloat16*>(out), part_o, part_lse, head_stride, *tk, *tv, l2, 0);
  return (int)cudaGetLastError();
}

}  // namespace ds
