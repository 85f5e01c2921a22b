// K7: split-KV decode / speculative-verify attention over the paged cell pool.
//
// GQA packing: the G = n_heads/n_kv_heads query heads that share a KV head are
// packed as rows r = t*G + g (t = batch row, g = head in group), so one K/V
// tile feeds all of them.  A CTA owns NW*16 packed rows, one KV head and one
// contiguous key range ("split", fixed by absolute key position); K/V rows are
// gathered cell-by-cell (page size 1, pos2cell) with 16-byte cp.async into an
// XOR-swizzled two-stage smem ring; QK^T and PV run on mma.sync m16n8k16
// (bf16 in, fp32 accumulate) with the FA2 register-resident online softmax
// (warp-shuffle row reductions).  Partial (O, lse) per split are merged by
// attn_combine_kernel.  Also serves as the generic small-Delta prefill path.
#include "../../include/deltaserve_b200.h"
#include "attn_plan.h"
#include "common.cuh"

namespace ds {

constexpr int kD = 128;
constexpr int kTileK = 64;                     // keys per smem tile
constexpr int kTileBytes = kTileK * kD * 2;    // 16 KB per K (or V) tile

// swizzled byte offset of (row, 16B chunk) inside a [64][128] bf16 tile
DS_DEVICE int tile_off(int row, int chunk) {
  return row * (kD * 2) + (((chunk & 8) | ((chunk & 7) ^ (row & 7))) << 4);
}

template <int NW>
__global__ void __launch_bounds__(NW * 32) attn_split_kernel(
    const __nv_bfloat16* __restrict__ qkv, int qkv_stride, const ds_entry* __restrict__ entries,
    int n_entries, int max_splits, const __nv_bfloat16* __restrict__ kpool,
    const __nv_bfloat16* __restrict__ vpool, const int32_t* __restrict__ pos2cell,
    int64_t pos_stride, int nh, int nkv, float scale_log2, __nv_bfloat16* __restrict__ out,
    float* __restrict__ part_o, float* __restrict__ part_lse, int64_t head_stride) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int e = blockIdx.z / max_splits;
  const int split = blockIdx.z - e * max_splits;
  const ds_entry en = entries[e];
  const int G = nh / nkv;
  const int R = en.q_len * G;
  const int qblocks = (R + NW * 16 - 1) / (NW * 16);
  if (static_cast<int>(blockIdx.x) >= qblocks) return;
  const int kv_len = en.past + en.q_len;
  const AttnSplitPlan plan = attn_split_plan(qblocks, kv_len, nkv, n_entries, 0, R);
  if (split >= plan.n_splits) return;
  const int kh = blockIdx.y;
  const int row0 = blockIdx.x * NW * 16;
  const int last_row = min(R, row0 + NW * 16) - 1;
  const int key_hi = min(kv_len, en.past + last_row / G + 1);
  const int k_begin = split * plan.split_len;
  const int k_end = min(k_begin + plan.split_len, key_hi);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int g8 = lane >> 2;  // row within 8
  const int t4 = lane & 3;

  const int wrow = row0 + warp * 16;
  const bool active = wrow < R;

  // ---- Q fragments (A operand, 16 rows x 128 d) ----
  uint32_t qa[8][4];
  int qpos[2];
  {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = wrow + g8 + 8 * h;
      qpos[h] = r < R ? en.past + r / G : -1;
    }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = wrow + g8 + ((q & 1) ? 8 : 0);
        const int col = kk * 16 + 2 * t4 + ((q & 2) ? 8 : 0);
        uint32_t v = 0;
        if (active && r < R) {
          const int ti = r / G, gi = r - (r / G) * G;
          const __nv_bfloat16* src = qkv + static_cast<int64_t>(en.q_start + ti) * qkv_stride +
                                     (kh * G + gi) * kD + col;
          v = *reinterpret_cast<const uint32_t*>(src);
        }
        qa[kk][q] = v;
      }
    }
  }

  float o[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY};
  float l_run[2] = {0.f, 0.f};

  const int32_t* p2c = pos2cell + static_cast<int64_t>(en.seq) * pos_stride;
  const int ntiles = k_end > k_begin ? (k_end - k_begin + kTileK - 1) / kTileK : 0;

  auto load_tile = [&](int it, int buf) {
    const int kt = k_begin + it * kTileK;
    uint8_t* ks = smem + buf * 2 * kTileBytes;
    uint8_t* vs = ks + kTileBytes;
    constexpr int CH = kTileK * 16;  // 16-byte chunks per tile
    for (int c = tid; c < CH; c += NW * 32) {
      const int row = c >> 4, chunk = c & 15;
      const int key = kt + row;
      const bool valid = key < k_end;
      const int64_t cell = valid ? p2c[key] : 0;
      const int64_t goff = (kh * head_stride + cell) * kD + chunk * 8;
      cp_async16_zfill(ks + tile_off(row, chunk), kpool + goff, valid);
      cp_async16_zfill(vs + tile_off(row, chunk), vpool + goff, valid);
    }
  };

  if (ntiles > 0) {
    load_tile(0, 0);
    cp_async_commit();
  }
  for (int it = 0; it < ntiles; ++it) {
    if (it + 1 < ntiles) {
      load_tile(it + 1, (it + 1) & 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (active) {
      const uint8_t* ks = smem + (it & 1) * 2 * kTileBytes;
      const uint8_t* vs = ks + kTileBytes;
      const uint32_t ks_u = smem_u32(ks), vs_u = smem_u32(vs);
      const int kt = k_begin + it * kTileK;
      float s[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const int mi = lane >> 3;
          const int key = (j + (mi >> 1)) * 8 + (lane & 7);
          const int chunk = 2 * kk + (mi & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(b0, b1, b2, b3, ks_u + tile_off(key, chunk));
          mma_bf16_16816(s[j], qa[kk], b0, b1);
          mma_bf16_16816(s[j + 1], qa[kk], b2, b3);
        }
      }
      // mask + online softmax (log2 domain)
      float mx[2] = {m_run[0], m_run[1]};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int h = q >> 1;
          const int key = kt + j * 8 + 2 * t4 + (q & 1);
          const bool ok = key < k_end && key <= qpos[h];
          const float v = ok ? s[j][q] * scale_log2 : -INFINITY;
          s[j][q] = v;
          mx[h] = fmaxf(mx[h], v);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
        mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
      }
      float alpha[2], mref[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mref[h] = mx[h] == -INFINITY ? 0.f : mx[h];
        alpha[h] = fast_exp2(m_run[h] - mref[h]);  // m_run=-inf -> 0
        m_run[h] = mx[h];
        l_run[h] *= alpha[h];
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        o[j][0] *= alpha[0];
        o[j][1] *= alpha[0];
        o[j][2] *= alpha[1];
        o[j][3] *= alpha[1];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float p = fast_exp2(s[j][q] - mref[q >> 1]);
          s[j][q] = p;
          l_run[q >> 1] += p;
        }
      }
      // O += P V
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        uint32_t pa[4];
        pa[0] = pack_bf16(s[2 * kb][0], s[2 * kb][1]);
        pa[1] = pack_bf16(s[2 * kb][2], s[2 * kb][3]);
        pa[2] = pack_bf16(s[2 * kb + 1][0], s[2 * kb + 1][1]);
        pa[3] = pack_bf16(s[2 * kb + 1][2], s[2 * kb + 1][3]);
#pragma unroll
        for (int dn = 0; dn < 16; dn += 2) {
          const int mi = lane >> 3;
          const int key = kb * 16 + ((mi & 1) ? 8 : 0) + (lane & 7);
          const int chunk = dn + (mi >> 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(b0, b1, b2, b3, vs_u + tile_off(key, chunk));
          mma_bf16_16816(o[dn], pa, b0, b1);
          mma_bf16_16816(o[dn + 1], pa, b2, b3);
        }
      }
    }
    __syncthreads();
  }

  if (!active) return;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l_run[h] += __shfl_xor_sync(0xffffffffu, l_run[h], 1);
    l_run[h] += __shfl_xor_sync(0xffffffffu, l_run[h], 2);
  }
  const float inv[2] = {l_run[0] > 0.f ? 1.f / l_run[0] : 0.f,
                        l_run[1] > 0.f ? 1.f / l_run[1] : 0.f};
  if (plan.n_splits == 1) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = wrow + g8 + 8 * h;
      if (r >= R) continue;
      const int ti = r / G, gi = r - (r / G) * G;
      __nv_bfloat16* dst =
          out + static_cast<int64_t>(en.q_start + ti) * nh * kD + (kh * G + gi) * kD;
#pragma unroll
      for (int dn = 0; dn < 16; ++dn) {
        *reinterpret_cast<uint32_t*>(dst + dn * 8 + 2 * t4) =
            pack_bf16(o[dn][2 * h] * inv[h], o[dn][2 * h + 1] * inv[h]);
      }
    }
  } else {
    const int64_t base = attn_partial_base(entries, e, n_entries, nh, nkv, 0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = wrow + g8 + 8 * h;
      if (r >= R) continue;
      const int64_t slot = (base + static_cast<int64_t>(split) * R + r) * nkv + kh;
      float* dst = part_o + slot * kD;
#pragma unroll
      for (int dn = 0; dn < 16; ++dn) {
        *reinterpret_cast<float2*>(dst + dn * 8 + 2 * t4) =
            make_float2(o[dn][2 * h] * inv[h], o[dn][2 * h + 1] * inv[h]);
      }
      if (t4 == 0)
        part_lse[slot] = l_run[h] > 0.f ? m_run[h] + __log2f(l_run[h]) : -INFINITY;
    }
  }
}

// Merge split partials: out = sum_s 2^(lse_s - lse_max) O_s / sum_s 2^(...)
__global__ void attn_combine_kernel(const ds_entry* __restrict__ entries, int n_entries, int nh,
                                    int nkv, int qblock_rows, int mode,
                                    const float* __restrict__ part_o,
                                    const float* __restrict__ part_lse,
                                    __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int e = blockIdx.z;
  const ds_entry en = entries[e];
  const int G = nh / nkv;
  const int R = en.q_len * G;
  const int r = blockIdx.x;
  if (r >= R) return;
  const int kh = blockIdx.y;
  const int qblocks = (R + qblock_rows - 1) / qblock_rows;
  const AttnSplitPlan plan =
      attn_split_plan(qblocks, en.past + en.q_len, nkv, n_entries, mode, R);
  if (plan.n_splits <= 1) return;
  const int64_t base = attn_partial_base(entries, e, n_entries, nh, nkv, mode);
  // two dependent L2 round trips in all: the split lse values (one thread
  // each) into smem, then every split's O column issued at once
  const int64_t s0 = (base + r) * nkv + kh, sstride = static_cast<int64_t>(R) * nkv;
  __shared__ float lse_s[64];
  const int d = threadIdx.x;
  if (d < plan.n_splits) lse_s[d] = __ldcg(part_lse + s0 + d * sstride);
  __syncthreads();
  float lmax = -INFINITY;
  for (int s = 0; s < plan.n_splits; ++s) lmax = fmaxf(lmax, lse_s[s]);
  float acc = 0.f, wsum = 0.f;
  for (int sb = 0; sb < plan.n_splits; sb += 16) {
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      v[i] = sb + i < plan.n_splits ? __ldcg(part_o + (s0 + (sb + i) * sstride) * kD + d) : 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (sb + i >= plan.n_splits) break;
      const float lse = lse_s[sb + i];
      const float w = lse == -INFINITY ? 0.f : exp2f(lse - lmax);
      wsum += w;
      acc += w * v[i];
    }
  }
  const int ti = r / G, gi = r - (r / G) * G;
  out[static_cast<int64_t>(en.q_start + ti) * nh * kD + (kh * G + gi) * kD + d] =
      __float2bfloat16_rn(wsum > 0.f ? acc / wsum : 0.f);
}

constexpr int kSplitNW = 4;

int launch_attn_decode(const void* qkv, const ds_entry* entries_host, const ds_entry* entries_dev,
                       int n_entries, const void* k_pool, const void* v_pool, int64_t head_stride,
                       const int32_t* pos2cell, int64_t pos_stride, int nh, int nkv, int max_R,
                       int max_splits, float scale, void* out, float* part_o, float* part_lse,
                       int* counters, cudaStream_t stream);

int launch_attn_split(const void* qkv, const ds_entry* entries_host, const ds_entry* entries_dev,
                      int n_entries, const void* k_pool, const void* v_pool, int64_t head_stride,
                      const int32_t* pos2cell, int64_t pos_stride, int nh, int nkv, int hd,
                      float scale, void* out, void* workspace, size_t ws_bytes,
                      cudaStream_t stream) {
  if (hd != kD || nh % nkv) return DS_EUNSUPPORTED;
  int max_qblocks = 0, max_R = 0;
  for (int e = 0; e < n_entries; ++e) {
    const int R = entries_host[e].q_len * (nh / nkv);
    max_R = R > max_R ? R : max_R;
    const int qb = (R + kSplitNW * 16 - 1) / (kSplitNW * 16);
    max_qblocks = qb > max_qblocks ? qb : max_qblocks;
  }
  const int mode = max_R <= kDecodeMaxRows ? 1 : 0;  // warp-specialised decode kernel vs split kernel
  int max_splits = 1;
  bool any_split = false;  // some entry needs the combine kernel
  for (int e = 0; e < n_entries; ++e) {
    const ds_entry& en = entries_host[e];
    const int R = en.q_len * (nh / nkv);
    const int qb = (R + kSplitNW * 16 - 1) / (kSplitNW * 16);
    const AttnSplitPlan p = attn_split_plan(qb, en.past + en.q_len, nkv, n_entries, mode, R);
    max_splits = p.n_splits > max_splits ? p.n_splits : max_splits;
    any_split |= p.n_splits > 1;
  }
  // workspace: [split-merge counters (zero-initialised once, self-resetting)][partials]
  constexpr size_t kCounterBytes = 64 << 10;
  if (n_entries * nkv * 4 > static_cast<int>(kCounterBytes)) return DS_EUNSUPPORTED;
  int* counters = static_cast<int*>(workspace);
  workspace = static_cast<uint8_t*>(workspace) + kCounterBytes;
  ws_bytes = ws_bytes > kCounterBytes ? ws_bytes - kCounterBytes : 0;
  const size_t need = attn_partial_bytes(entries_host, n_entries, nh, nkv, mode);
  if (need > ws_bytes) return DS_EWORKSPACE;
  float* part_o = static_cast<float*>(workspace);
  const int64_t slots = attn_partial_slots(entries_host, n_entries, nh, nkv, mode);
  float* part_lse = part_o + slots * kD;
  if (mode == 1) {
    const int rc = launch_attn_decode(qkv, entries_host, entries_dev, n_entries, k_pool, v_pool,
                                      head_stride, pos2cell, pos_stride, nh, nkv, max_R,
                                      max_splits, scale, out, part_o, part_lse, counters, stream);
    // K7 merges up to kDecodeMaxCluster key splits in-cluster; more through
    // global partials: merged by the last split to arrive for <= 8 rows,
    // else by the combine kernel (launched early: K7 has not triggered it)
    if (rc != 0 || !any_split || max_splits <= kDecodeMaxCluster ||
        max_R <= kDecodeLastMergeRows)
      return rc;
    dim3 cgrid(max_R, nkv, n_entries);
    launch_pdl(attn_combine_kernel, cgrid, dim3(kD), 0, stream, entries_dev, n_entries, nh, nkv,
               kSplitNW * 16, 1, (const float*)part_o, (const float*)part_lse,
               static_cast<__nv_bfloat16*>(out));
    return (int)cudaGetLastError();
  }
  const int smem = 2 * 2 * kTileBytes;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_split_kernel<kSplitNW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    attr_set = true;
  }
  const float scale_log2 = scale * 1.4426950408889634f;
  dim3 grid(max_qblocks, nkv, n_entries * max_splits);
  attn_split_kernel<kSplitNW><<<grid, kSplitNW * 32, smem, stream>>>(
      static_cast<const __nv_bfloat16*>(qkv), (nh + 2 * nkv) * kD, entries_dev, n_entries,
      max_splits, static_cast<const __nv_bfloat16*>(k_pool),
      static_cast<const __nv_bfloat16*>(v_pool), pos2cell, pos_stride, nh, nkv, scale_log2,
      static_cast<__nv_bfloat16*>(out), part_o, part_lse, head_stride);
  if (any_split) {
    dim3 cgrid(max_R, nkv, n_entries);
    attn_combine_kernel<<<cgrid, kD, 0, stream>>>(entries_dev, n_entries, nh, nkv, kSplitNW * 16,
                                                  0, part_o, part_lse,
                                                  static_cast<__nv_bfloat16*>(out));
  }
  return (int)cudaGetLastError();
}

}  // namespace ds
