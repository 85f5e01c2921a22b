// K6: delta-prefill attention on the 5th-generation tensor cores (tcgen05).
//
// Delta new query tokens attend causally over an m-token prefix that lives in
// the paged (head-major) cell pool.  One CTA per (128 packed query rows, KV
// head): GQA packing puts the G query heads of 128/G consecutive positions in
// the M=128 rows, so every K/V tile is loaded once for all G heads.
// Warp roles (6 warps, one CTA per SM, all 512 TMEM columns):
//   warp 0  TMA producer: per 128-key tile, four 2D TMA boxes (K, V x two
//           128-byte column halves, SWIZZLE_128B) when the tile's cells form
//           one run, else a cell-by-cell cp.async gather into the same layout;
//           2-stage smem ring with full/empty mbarriers.
//   warp 1  MMA issuer (one elected thread): S_j = Q.K_j^T (M=N=K=128, 8 x
//           tcgen05.mma kind::f16, A/B K-major SW128 descriptors) into a
//           double-buffered TMEM S, then O += P_j.V_j (B = V MN-major) into a
//           TMEM-resident O accumulator; completion via tcgen05.commit ->
//           mbarrier.  S_{j+1} is issued before PV_j so the tensor core
//           overlaps the softmax of tile j.
//   warps 2-5 softmax (thread = TMEM lane = query row): one batched
//           tcgen05.ld of the S row, online softmax in the log2 domain with
//           causal masking only on diagonal tiles, P (bf16) to smem in the UMMA
//           A layout.  The running max is only raised when it grows by more
//           than 2^8 (P <= 256 stays exact in bf16/fp32), so the O rescale in
//           TMEM (ld/scale/st) is rare; final O/l epilogue from TMEM.
#include "../../include/deltaserve_b200.h"
#include "common.cuh"
#include "tc.cuh"
#include "tma.h"

namespace ds {

namespace {
constexpr int kD = 128;
constexpr int kBM = 128;                  // packed query rows per CTA
constexpr int kBN = 128;                  // keys per tile
constexpr int kHalf = kBM * 128;          // one 64-column half of a 128-row tile (16 KB)
constexpr int kTile = 2 * kHalf;          // 32 KB
constexpr int kStages = 2;
constexpr int kThreads = 6 * 32;
constexpr int kSmemQ = 0;
constexpr int kSmemP = kTile;
constexpr int kSmemKV = 2 * kTile;                        // stages x (K | V)
constexpr int kSmemBar = kSmemKV + kStages * 2 * kTile;   // barriers after the ring
constexpr int kSmemBytes = kSmemBar + 256 + 1024;         // + alignment slack

DS_DEVICE int sw128(int row, int chunk16) {
  return (chunk16 >> 3) * kHalf + row * 128 + (((chunk16 & 7) ^ (row & 7)) << 4);
}
}  // namespace

__global__ void __launch_bounds__(kThreads, 1) attn_prefill_kernel(
    const __nv_bfloat16* __restrict__ qkv, int qkv_stride, const ds_entry* __restrict__ entries,
    const __nv_bfloat16* __restrict__ kpool, const __nv_bfloat16* __restrict__ vpool,
    int64_t head_stride, const int32_t* __restrict__ pos2cell, int64_t pos_stride, int nh,
    int nkv, float scale_log2, __nv_bfloat16* __restrict__ out,
    const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
  uint64_t* kv_full = bars;        // [2]
  uint64_t* kv_empty = bars + 2;   // [2]
  uint64_t* s_full = bars + 4;     // [2]
  uint64_t* s_empty = bars + 6;    // [2]
  uint64_t* pv_done = bars + 8;    // [1] PV_j complete (P smem free, O stable)
  uint64_t* p_full = bars + 12;    // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  pdl_wait();
  pdl_trigger();

  const ds_entry en = entries[blockIdx.z];
  const int G = nh / nkv;
  const int pos_per_block = kBM / G;
  const int t0 = blockIdx.x * pos_per_block;
  if (t0 >= en.q_len) return;
  const int kh = blockIdx.y;
  const int t_last = min(en.q_len, t0 + pos_per_block) - 1;
  const int kv_len = en.past + en.q_len;
  const int kv_hi = en.past + t_last + 1;  // keys any row of this block can see
  const int ntiles = (kv_hi + kBN - 1) / kBN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
    }
    mbar_init(pv_done, 1);
    mbar_init(p_full, 4);
    mbar_fence_init();
  }
  if (warp == 1) tc::alloc(tmem_slot, 512);
  if (warp >= 2) {  // Q rows (packed r = t*G + g) -> smem, UMMA A layout
    const int r = tid - 64;
    const int t = t0 + r / G, g = r - (r / G) * G;
    const bool ok = t < en.q_len;
    const uint4* src = reinterpret_cast<const uint4*>(
        qkv + static_cast<int64_t>(en.q_start + (ok ? t : 0)) * qkv_stride + (kh * G + g) * kD);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const uint4 v = ok ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(smem + kSmemQ + sw128(r, c)) = v;
    }
    tc::fence_proxy_async();
  }
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
    for (int j = 0; j < ntiles; ++j) {
      const int st = j % kStages;
      if (j >= kStages) mbar_wait(&kv_empty[st], ((j / kStages) - 1) & 1);
      uint8_t* ks = smem + kSmemKV + st * 2 * kTile;
      uint8_t* vs = ks + kTile;
      const int kt = j * kBN;
      const int nvalid = min(kBN, kv_hi - kt);
      int c[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i] = lane + 32 * i < nvalid ? __ldg(p2c + kt + lane + 32 * i) : -1;
      const int c0 = __shfl_sync(0xffffffffu, c[0], 0);
      bool ok = true;
#pragma unroll
      for (int i = 0; i < 4; ++i) ok &= (c[i] < 0) || (c[i] == c0 + lane + 32 * i);
      if (__all_sync(0xffffffffu, ok)) {
        if (lane == 0) {
          mbar_expect_tx(&kv_full[st], 2 * kTile);
          const int row = static_cast<int>(hrow + c0);
          tma_load_2d(ks, &tmk, 0, row, &kv_full[st]);
          tma_load_2d(ks + kHalf, &tmk, 64, row, &kv_full[st]);
          tma_load_2d(vs, &tmv, 0, row, &kv_full[st]);
          tma_load_2d(vs + kHalf, &tmv, 64, row, &kv_full[st]);
        }
      } else {
#pragma unroll 1
        for (int i = 0; i < 4; ++i) {
          const int r = lane + 32 * i;
          const int64_t off = (hrow + (c[i] >= 0 ? c[i] : c0)) * kD;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            cp_async16(ks + sw128(r, q), kpool + off + q * 8);
            cp_async16(vs + sw128(r, q), vpool + off + q * 8);
          }
        }
        cp_async_commit();
        cp_async_wait<0>();
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&kv_full[st]);
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16(kBM, kBN, false);
      constexpr uint32_t idesc_pv = tc::idesc_bf16(kBM, kD, true);
      const uint32_t q_base = smem_u32(smem + kSmemQ);
      const uint32_t p_base = smem_u32(smem + kSmemP);
      const uint32_t kv_base = smem_u32(smem + kSmemKV);
      auto issue_s = [&](int j) {
        const int st = j % kStages, sb = j & 1;
        mbar_wait(&kv_full[st], (j / kStages) & 1);
        if (j >= 2) mbar_wait(&s_empty[sb], ((j >> 1) - 1) & 1);
        tc::fence_after();
        const uint32_t kb = kv_base + st * 2 * kTile;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
          tc::mma(tmem + sb * kBN, tc::smem_desc(q_base + off, 16, 1024),
                  tc::smem_desc(kb + off, 16, 1024), idesc_s, kk > 0);
        }
        tc::commit(&s_full[sb]);
      };
      issue_s(0);
      for (int j = 0; j < ntiles; ++j) {
        if (j + 1 < ntiles) issue_s(j + 1);
        const int st = j % kStages;
        mbar_wait(p_full, j & 1);
        tc::fence_after();
        const uint32_t vb = kv_base + st * 2 * kTile + kTile;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          tc::mma(tmem + 256, tc::smem_desc(p_base + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024),
                  tc::smem_desc(vb + kk * 2048, kHalf, 1024), idesc_pv, (j | kk) > 0);
        }
        tc::commit(pv_done);
        tc::commit(&kv_empty[st]);
      }
    }
  } else {
    // ================ softmax / correction / epilogue ================
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int r = quad * 32 + lane;
    const int t = t0 + r / G, g = r - (r / G) * G;
    const int pos = en.past + t;  // this row's absolute position (causal bound)
    const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    const uint32_t tO = trow + 256;
    const int blk_pos_min = en.past + t0;
    float m_ref = -INFINITY, l_run = 0.f;
    uint8_t* prow = smem + kSmemP;
    uint32_t sv[kBN];
    for (int j = 0; j < ntiles; ++j) {
      const int sb = j & 1;
      const int kt = j * kBN;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc::fence_after();
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) tc::ld32_issue(trow + sb * kBN + cc * 32, sv + cc * 32);
      tc::wait_ld();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);  // S buffer is in registers now
      const bool need_mask = (kt + kBN - 1 > blk_pos_min) || (kt + kBN > kv_len);
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < kBN; ++i) {
        float x = __uint_as_float(sv[i]) * scale_log2;
        if (need_mask) x = (kt + i <= pos && kt + i < kv_len) ? x : -INFINITY;
        sv[i] = __float_as_uint(x);
        mx = fmaxf(mx, x);
      }
      // PV_{j-1} done: P smem is free and O in TMEM is stable
      if (j > 0) {
        mbar_wait(pv_done, (j - 1) & 1);
        tc::fence_after();
      }
      const float new_ref = (mx > m_ref + 8.f) ? mx : m_ref;
      const float scale_old = (m_ref == -INFINITY) ? 0.f : fast_exp2(m_ref - new_ref);
      if (j > 0 && __any_sync(0xffffffffu, new_ref != m_ref)) {  // rare O correction
        uint32_t ov[32];
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
          tc::ld32_issue(tO + cc * 32, ov);
          tc::wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * scale_old);
          tc::st32(tO + cc * 32, ov);
        }
        tc::wait_st();
      }
      l_run *= scale_old;
      m_ref = new_ref;
      const float mref = m_ref == -INFINITY ? 0.f : m_ref;
      float sum = 0.f;
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        uint32_t pk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float p0 = fast_exp2(__uint_as_float(sv[cc * 8 + 2 * q]) - mref);
          const float p1 = fast_exp2(__uint_as_float(sv[cc * 8 + 2 * q + 1]) - mref);
          sum += p0 + p1;
          pk[q] = pack_bf16(p0, p1);
        }
        *reinterpret_cast<uint4*>(prow + sw128(r, cc)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      l_run += sum;
      tc::fence_proxy_async();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(pv_done, (ntiles - 1) & 1);
    tc::fence_after();
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) tc::ld32_issue(tO + cc * 32, sv + cc * 32);
    tc::wait_ld();
    if (t < en.q_len) {
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      uint4* dst = reinterpret_cast<uint4*>(out + static_cast<int64_t>(en.q_start + t) * nh * kD +
                                            (kh * G + g) * kD);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float* o = reinterpret_cast<const float*>(sv) + 8 * q;
        dst[q] = make_uint4(pack_bf16(o[0] * inv, o[1] * inv), pack_bf16(o[2] * inv, o[3] * inv),
                            pack_bf16(o[4] * inv, o[5] * inv), pack_bf16(o[6] * inv, o[7] * inv));
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::dealloc(tmem, 512);
  }
}

int launch_attn_prefill_sm100(const void* qkv, const ds_entry* entries_host,
                              const ds_entry* entries_dev, int n_entries, const void* k_pool,
                              const void* v_pool, int64_t head_stride, const int32_t* pos2cell,
                              int64_t pos_stride, int nh, int nkv, int hd, float scale, void* out,
                              cudaStream_t stream) {
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
  int max_qb = 0;
  for (int e = 0; e < n_entries; ++e) {
    const int qb = (entries_host[e].q_len + ppb - 1) / ppb;
    max_qb = qb > max_qb ? qb : max_qb;
  }
  dim3 grid(max_qb, nkv, n_entries);
  launch_pdl(attn_prefill_kernel, grid, dim3(kThreads), kSmemBytes, stream,
             static_cast<const __nv_bfloat16*>(qkv), (nh + 2 * nkv) * kD, entries_dev,
             static_cast<const __nv_bfloat16*>(k_pool), static_cast<const __nv_bfloat16*>(v_pool),
             head_stride, pos2cell, pos_stride, nh, nkv, scale * 1.4426950408889634f,
             static_cast<__nv_bfloat16*>(out), *tk, *tv);
  return (int)cudaGetLastError();
}

}  // namespace ds
