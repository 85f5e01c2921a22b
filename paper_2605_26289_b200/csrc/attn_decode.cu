// K7 (decode / speculative verify, R = q_len * G <= 32 packed query rows).
//
// HBM-bound: every K/V byte of a split is read once and feeds all R rows (GQA
// packing: row r = t*G + g, so the G query heads sharing a KV head share its
// tiles).  Warp-specialised, one CTA per SM:
//   * producer warp: per 64-key tile, when the tile's cells form one run
//     (the common case - first-fit allocation, head-major pool) four 2D TMA
//     boxes (K and V, two 128-byte column halves, SWIZZLE_128B) complete on the
//     stage's mbarrier; otherwise the warp gathers the tile cell by cell with
//     16-byte cp.async into the same swizzled layout.  6-stage ring, up to 5
//     tiles (~160 KB) in flight per SM;
//   * 8 consumer warps = 4 key groups x 2 head-dim halves: warp (kg, dh) owns
//     16 keys of every tile and output columns [64*dh, 64*dh+64); QK^T (computed
//     by both halves of a pair - cheap next to the latency it hides) and PV on
//     mma.sync m16n8k16 (bf16 in, fp32 accumulate), online softmax with quad
//     shuffles, lazy O rescale, masks only on boundary tiles; then release the
//     stage through an "empty" mbarrier.  Two consumer warps per scheduler
//     hide the HMMA/LDSM latency chains a single warp could not.
// The 128-byte swizzle keeps ldmatrix bank-conflict free.  The 4 warp states
// merge through smem; split partials (O, lse) go to attn_combine_kernel (an
// in-kernel last-CTA merge was measured slower: its serial L2 round trips
// outlast the combine launch, which PDL already overlaps).
// Programmatic dependent launch: only q and the K/V rows of this batch's own
// positions (>= past) come from the preceding wqkv projection, so the
// producer streams every tile of older keys before the dependency wait - the
// KV read overlaps the projection's tail; consumers wait before loading q.
#include "../../include/deltaserve_b200.h"
#include "attn_plan.h"
#include "common.cuh"
#include "tma.h"

namespace ds {

namespace {
constexpr int kD = 128;
constexpr int kTile = 64;
constexpr int kHalfBytes = kTile * kD * 2;  // one K (or V) tile: 2 x [64 rows][128 B]
constexpr int kStageBytes = 2 * kHalfBytes;
constexpr int kStages = 6;
constexpr int kQRows = 32;
constexpr int kConsumers = 8;  // 4 key groups x 2 d halves
constexpr int kKeyGroups = 4;
constexpr int kThreads = (kConsumers + 1) * 32;

DS_DEVICE int qswz(int row, int chunk) {
  return row * (kD * 2) + (((chunk & 8) | ((chunk & 7) ^ (row & 7))) << 4);
}
// TMA SWIZZLE_128B layout of a [64 rows][128 d] tile: two 64-column halves of
// 128-byte rows; 16-byte chunk c of a row sits at c ^ (row & 7).
DS_DEVICE int tswz(int row, int chunk16) {
  return (chunk16 >> 3) * (kTile * 128) + row * 128 + (((chunk16 & 7) ^ (row & 7)) << 4);
}
}  // namespace

int decode_smem_bytes() {
  return 1024 + kStages * kStageBytes + kQRows * kD * 2 + 2 * kStages * 8;
}

template <int MT>
__global__ void __launch_bounds__(kThreads, 1) attn_decode_kernel(
    const __nv_bfloat16* __restrict__ qkv, int qkv_stride, const ds_entry* __restrict__ entries,
    int n_entries, int max_splits, const __nv_bfloat16* __restrict__ kpool,
    const __nv_bfloat16* __restrict__ vpool, const int32_t* __restrict__ pos2cell,
    int64_t pos_stride, int nh, int nkv, float scale_log2, __nv_bfloat16* __restrict__ out,
    float* __restrict__ part_o, float* __restrict__ part_lse, int64_t head_stride,
    int* __restrict__ counters, const __grid_constant__ CUtensorMap tmk,
    const __grid_constant__ CUtensorMap tmv) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // SW128 alignment
  uint8_t* qs = smem + kStages * kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(qs + kQRows * kD * 2);
  uint64_t* empty = full + kStages;

  const int e = blockIdx.z / max_splits;
  const int split = blockIdx.z - e * max_splits;
  const ds_entry en = entries[e];
  const int G = nh / nkv;
  const int R = en.q_len * G;
  const int kv_len = en.past + en.q_len;
  const AttnSplitPlan plan = attn_split_plan(1, kv_len, nkv, n_entries, 1);
  if (split >= plan.n_splits) return;
  const int kh = blockIdx.y;
  const int k_begin = split * plan.split_len;
  const int k_end = min(k_begin + plan.split_len, kv_len);
  const int ntiles = (k_end - k_begin + kTile - 1) / kTile;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == kConsumers && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    mbar_fence_init();
  }
  __syncthreads();  // barriers initialised

  const int32_t* p2c = pos2cell + static_cast<int64_t>(en.seq) * pos_stride;
  if (warp == kConsumers) {
    // ================= producer =================
    if (lane == 0) {
      tma_prefetch_desc(&tmk);
      tma_prefetch_desc(&tmv);
    }
    const int64_t hrow = kh * head_stride;
    // cell ids are prefetched two tiles ahead so their latency never stalls
    // the TMA issue loop
    auto cells = [&](int t, int& lo, int& hi) {
      const int kt = k_begin + t * kTile;
      const int nv = t < ntiles ? min(kTile, k_end - kt) : 0;
      lo = lane < nv ? __ldg(p2c + kt + lane) : -1;
      hi = lane + 32 < nv ? __ldg(p2c + kt + 32 + lane) : -1;
    };
    int c_lo, c_hi, n1_lo, n1_hi, n2_lo, n2_hi;
    cells(0, c_lo, c_hi);
    cells(1, n1_lo, n1_hi);
    bool waited = false;
    for (int it = 0; it < ntiles; ++it) {
      cells(it + 2, n2_lo, n2_hi);
      const int st = it % kStages;
      if (it >= kStages) mbar_wait(&empty[st], ((it / kStages) - 1) & 1);
      uint8_t* ks = smem + st * kStageBytes;
      uint8_t* vs = ks + kHalfBytes;
      const int kt = k_begin + it * kTile;
      const int nvalid = min(kTile, k_end - kt);
      if (!waited && kt + nvalid > en.past) {  // first tile holding this batch's own K/V
        pdl_wait();
        waited = true;
      }
      const int c0 = __shfl_sync(0xffffffffu, c_lo, 0);
      const bool run = __all_sync(0xffffffffu, (lane >= nvalid || c_lo == c0 + lane) &&
                                                    (lane + 32 >= nvalid || c_hi == c0 + 32 + lane));
      if (run) {  // one contiguous run of cells: 4 TMA boxes
        if (lane == 0) {
          mbar_expect_tx(&full[st], kStageBytes);
          const int row = static_cast<int>(hrow + c0);
          tma_load_2d(ks, &tmk, 0, row, &full[st]);
          tma_load_2d(ks + kTile * 128, &tmk, 64, row, &full[st]);
          tma_load_2d(vs, &tmv, 0, row, &full[st]);
          tma_load_2d(vs + kTile * 128, &tmv, 64, row, &full[st]);
        }
      } else {  // fragmented: cell-by-cell 16-byte gathers into the same layout
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          const int r = lane + 32 * h;
          const int cv = h ? c_hi : c_lo;
          const int cl = cv >= 0 ? cv : c0;  // tail rows duplicate a valid cell (masked)
          const int64_t off = (hrow + cl) * kD;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            cp_async16(ks + tswz(r, c), kpool + off + c * 8);
            cp_async16(vs + tswz(r, c), vpool + off + c * 8);
          }
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[st]);
      }
      c_lo = n1_lo; c_hi = n1_hi;
      n1_lo = n2_lo; n1_hi = n2_hi;
    }
    if (!waited) pdl_wait();
    pdl_trigger();
    return;
  }

  // ================= consumers =================
  pdl_wait();  // q comes from the preceding projection
  pdl_trigger();
  {  // Q rows -> smem (swizzled, zero padded to 32 rows)
    for (int c = tid; c < kQRows * 16; c += kConsumers * 32) {
      const int r = c >> 4, chunk = c & 15;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < R) {
        const int ti = r / G, gi = r - ti * G;
        v = *reinterpret_cast<const uint4*>(qkv +
                                            static_cast<int64_t>(en.q_start + ti) * qkv_stride +
                                            (kh * G + gi) * kD + chunk * 8);
      }
      *reinterpret_cast<uint4*>(qs + qswz(r, chunk)) = v;
    }
  }
  named_bar_sync(1, kConsumers * 32);  // q staged
  const int g8 = lane >> 2, t4 = lane & 3, mi = lane >> 3;
  const int kg = warp & (kKeyGroups - 1), dh = warp / kKeyGroups;
  int qpos[MT][2];
  float o[MT][8][4];
  float m_run[MT][2], l_run[MT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = mt * 16 + g8 + 8 * h;
      qpos[mt][h] = r < R ? en.past + r / G : -1;
      m_run[mt][h] = -INFINITY;
      l_run[mt][h] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) o[mt][j][0] = o[mt][j][1] = o[mt][j][2] = o[mt][j][3] = 0.f;
  }
  const uint32_t qs_u = smem_u32(qs);
  // per-lane ldmatrix rows inside a tile (keys of this warp's group)
  const int k_row = kg * 16 + (mi >> 1) * 8 + (lane & 7);
  const int v_row = kg * 16 + (mi & 1) * 8 + (lane & 7);

  for (int it = 0; it < ntiles; ++it) {
    const int st = it % kStages;
    mbar_wait(&full[st], (it / kStages) & 1);
    const uint32_t ks_u = smem_u32(smem + st * kStageBytes), vs_u = ks_u + kHalfBytes;
    const int kt = k_begin + it * kTile + kg * 16;
    float s[MT][2][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int j = 0; j < 2; ++j) s[mt][j][0] = s[mt][j][1] = s[mt][j][2] = s[mt][j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4(b0, b1, b2, b3, ks_u + tswz(k_row, 2 * kk + (mi & 1)));
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        uint32_t a[4];
        ldsm_x4(a[0], a[1], a[2], a[3],
                qs_u + qswz(mt * 16 + (lane & 7) + ((mi & 1) ? 8 : 0), 2 * kk + (mi >> 1)));
        mma_bf16_16816(s[mt][0], a, b0, b1);
        mma_bf16_16816(s[mt][1], a, b2, b3);
      }
    }
    const bool need_mask = (kt + 16 > k_end) || (kt + 15 > en.past);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      float mx[2] = {m_run[mt][0], m_run[mt][1]};
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float v = s[mt][j][q] * scale_log2;
          if (need_mask) {
            const int key = kt + j * 8 + 2 * t4 + (q & 1);
            v = (key < k_end && key <= qpos[mt][q >> 1]) ? v : -INFINITY;
          }
          s[mt][j][q] = v;
          mx[q >> 1] = fmaxf(mx[q >> 1], v);
        }
      float alpha[2], mref[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
        mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
        mref[h] = mx[h] == -INFINITY ? 0.f : mx[h];
        alpha[h] = fast_exp2(m_run[mt][h] - mref[h]);
        m_run[mt][h] = mx[h];
        l_run[mt][h] *= alpha[h];
      }
      if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          o[mt][j][0] *= alpha[0];
          o[mt][j][1] *= alpha[0];
          o[mt][j][2] *= alpha[1];
          o[mt][j][3] *= alpha[1];
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float p = fast_exp2(s[mt][j][q] - mref[q >> 1]);
          s[mt][j][q] = p;
          l_run[mt][q >> 1] += p;
        }
    }
    uint32_t pa[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      pa[mt][0] = pack_bf16(s[mt][0][0], s[mt][0][1]);
      pa[mt][1] = pack_bf16(s[mt][0][2], s[mt][0][3]);
      pa[mt][2] = pack_bf16(s[mt][1][0], s[mt][1][1]);
      pa[mt][3] = pack_bf16(s[mt][1][2], s[mt][1][3]);
    }
#pragma unroll
    for (int dn = 0; dn < 8; dn += 2) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(b0, b1, b2, b3, vs_u + tswz(v_row, dh * 8 + dn + (mi >> 1)));
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        mma_bf16_16816(o[mt][dn], pa[mt], b0, b1);
        mma_bf16_16816(o[mt][dn + 1], pa[mt], b2, b3);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  named_bar_sync(1, kConsumers * 32);  // all consumers done with the ring

  // ---- merge the 4 key groups' states (ring memory is free now) ----
  float* osm = reinterpret_cast<float*>(smem);  // [4][32][128]
  float* msm = osm + kKeyGroups * kQRows * kD;  // [4][32]
  float* lsm = msm + kKeyGroups * kQRows;       // [4][32]
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float l = l_run[mt][h];
      l += __shfl_xor_sync(0xffffffffu, l, 1);
      l += __shfl_xor_sync(0xffffffffu, l, 2);
      const int r = mt * 16 + g8 + 8 * h;
      if (t4 == 0 && dh == 0) {
        msm[kg * kQRows + r] = m_run[mt][h];
        lsm[kg * kQRows + r] = l;
      }
#pragma unroll
      for (int dn = 0; dn < 8; ++dn)
        *reinterpret_cast<float2*>(osm + (kg * kQRows + r) * kD + dh * 64 + dn * 8 + 2 * t4) =
            make_float2(o[mt][dn][2 * h], o[mt][dn][2 * h + 1]);
    }
  }
  named_bar_sync(1, kConsumers * 32);
  const int64_t base =
      plan.n_splits > 1 ? attn_partial_base(entries, e, n_entries, nh, nkv, 1) : 0;
  for (int idx = tid; idx < R * kD; idx += kConsumers * 32) {
    const int r = idx / kD, d = idx - r * kD;
    float mm = -INFINITY;
#pragma unroll
    for (int w = 0; w < kKeyGroups; ++w) mm = fmaxf(mm, msm[w * kQRows + r]);
    const float mref = mm == -INFINITY ? 0.f : mm;
    float L = 0.f, acc = 0.f;
#pragma unroll
    for (int w = 0; w < kKeyGroups; ++w) {
      const float sc = fast_exp2(msm[w * kQRows + r] - mref);
      L += lsm[w * kQRows + r] * sc;
      acc += osm[(w * kQRows + r) * kD + d] * sc;
    }
    const float val = L > 0.f ? acc / L : 0.f;
    if (plan.n_splits == 1) {
      const int ti = r / G, gi = r - ti * G;
      out[static_cast<int64_t>(en.q_start + ti) * nh * kD + (kh * G + gi) * kD + d] =
          __float2bfloat16_rn(val);
    } else {
      const int64_t slot = (base + static_cast<int64_t>(split) * R + r) * nkv + kh;
      part_o[slot * kD + d] = val;
      if (d == 0) part_lse[slot] = L > 0.f ? mm + __log2f(L) : -INFINITY;
    }
  }
}

int launch_attn_decode(const void* qkv, const ds_entry* entries_host, const ds_entry* entries_dev,
                       int n_entries, const void* k_pool, const void* v_pool, int64_t head_stride,
                       const int32_t* pos2cell, int64_t pos_stride, int nh, int nkv, int max_R,
                       int max_splits, float scale, void* out, float* part_o, float* part_lse,
                       int* counters, cudaStream_t stream) {
  (void)entries_host;
  const int smem = decode_smem_bytes();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_decode_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const CUtensorMap* tk = kv_tensor_map(k_pool, static_cast<int64_t>(nkv) * head_stride, kTile);
  const CUtensorMap* tv = kv_tensor_map(v_pool, static_cast<int64_t>(nkv) * head_stride, kTile);
  if (!tk || !tv) return DS_EUNSUPPORTED;
  dim3 grid(1, nkv, n_entries * max_splits);
  const float sl2 = scale * 1.4426950408889634f;
  const int stride = (nh + 2 * nkv) * kD;
  auto kern = max_R <= 16 ? attn_decode_kernel<1> : attn_decode_kernel<2>;
  launch_pdl(kern, grid, dim3(kThreads), smem, stream, static_cast<const __nv_bfloat16*>(qkv),
             stride, entries_dev, n_entries, max_splits,
             static_cast<const __nv_bfloat16*>(k_pool), static_cast<const __nv_bfloat16*>(v_pool),
             pos2cell, pos_stride, nh, nkv, sl2, static_cast<__nv_bfloat16*>(out), part_o,
             part_lse, head_stride, counters, *tk, *tv);
  return (int)cudaGetLastError();
}

}  // namespace ds
