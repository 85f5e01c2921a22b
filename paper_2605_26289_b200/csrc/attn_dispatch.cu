// K7 dispatch: decode / speculative-verify attention (R = q_len * G <= 24
// packed rows) over the paged cell pool - the split plan, the workspace
// carve-up, and the merge of split partials (O, lse) that do not merge
// in-cluster (attn_combine_kernel).  The kernels themselves live in
// attn_decode.cu (mma.sync, keys on the MMA M side) and attn_decode_tc.cu
// (tcgen05/TMEM, R > 8 over long prefixes).  Rows beyond the K7 limit are
// delta prefill and go to the tcgen05 K6 kernel (attn_prefill_sm100.cu).
#include "../../include/deltaserve_b200.h"
#include "attn_plan.h"
#include "common.cuh"

namespace ds {

constexpr int kD = 128;

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
  // ONE L2 round trip for up to 32 splits: every thread issues the splits'
  // lse values (same addresses across the CTA) and its O column together
  // (was lse -> smem -> barrier -> O in batches of 16: three round trips, and
  // the next decode launch's dependency wait sat behind them)
  const int64_t s0 = (base + r) * nkv + kh, sstride = static_cast<int64_t>(R) * nkv;
  const int d = threadIdx.x;
  const int ns = plan.n_splits;
  float acc = 0.f, wsum = 0.f, lmax = -INFINITY;
  for (int sb = 0; sb < ns; sb += 32) {
    float v[32], lv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const bool ok = sb + i < ns;
      lv[i] = ok ? __ldcg(part_lse + s0 + (sb + i) * sstride) : -INFINITY;
      v[i] = ok ? __ldcg(part_o + (s0 + (sb + i) * sstride) * kD + d) : 0.f;
    }
    float bmax = -INFINITY;
#pragma unroll
    for (int i = 0; i < 32; ++i) bmax = fmaxf(bmax, lv[i]);
    const float nmax = fmaxf(lmax, bmax);
    if (nmax != -INFINITY) {  // rescale the running sums to the new max (second batch only)
      const float c = lmax == -INFINITY ? 0.f : exp2f(lmax - nmax);
      acc *= c;
      wsum *= c;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float w = lv[i] == -INFINITY ? 0.f : exp2f(lv[i] - nmax);
        wsum += w;
        acc += w * v[i];
      }
      lmax = nmax;
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
                       int* counters, int* merged, cudaStream_t stream);

int launch_attn_prefill_sm100(const void* qkv, const ds_entry* entries_host,
                              const ds_entry* entries_dev, int n_entries, const void* k_pool,
                              const void* v_pool, int64_t head_stride, const int32_t* pos2cell,
                              int64_t pos_stride, int nh, int nkv, int hd, float scale, void* out,
                              void* workspace, size_t ws_bytes, cudaStream_t stream);

int launch_attn_split(const void* qkv, const ds_entry* entries_host, const ds_entry* entries_dev,
                      int n_entries, const void* k_pool, const void* v_pool, int64_t head_stride,
                      const int32_t* pos2cell, int64_t pos_stride, int nh, int nkv, int hd,
                      float scale, void* out, void* workspace, size_t ws_bytes,
                      cudaStream_t stream) {
  if (hd != kD || nh % nkv) return DS_EUNSUPPORTED;
  int max_R = 0;
  for (int e = 0; e < n_entries; ++e) {
    const int R = entries_host[e].q_len * (nh / nkv);
    max_R = R > max_R ? R : max_R;
  }
  if (max_R > kDecodeMaxRows)  // delta prefill rows: the tcgen05 K6 kernel
    return launch_attn_prefill_sm100(qkv, entries_host, entries_dev, n_entries, k_pool, v_pool,
                                     head_stride, pos2cell, pos_stride, nh, nkv, hd, scale, out,
                                     workspace, ws_bytes, stream);
  constexpr int mode = 1;  // split plan of the warp-specialised decode kernel
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
  {
    int merged = 0;
    const int rc = launch_attn_decode(qkv, entries_host, entries_dev, n_entries, k_pool, v_pool,
                                      head_stride, pos2cell, pos_stride, nh, nkv, max_R,
                                      max_splits, scale, out, part_o, part_lse, counters, &merged,
                                      stream);
    // K7 merges up to kDecodeMaxCluster key splits in-cluster; more through
    // global partials: merged by the last split to arrive for <= 8 rows,
    // else by the combine kernel (launched early: K7 has not triggered it)
    if (rc != 0 || !any_split || merged) return rc;
    dim3 cgrid(max_R, nkv, n_entries);
    launch_pdl(attn_combine_kernel, cgrid, dim3(kD), 0, stream, entries_dev, n_entries, nh, nkv,
               kSplitNW * 16, 1, (const float*)part_o, (const float*)part_lse,
               static_cast<__nv_bfloat16*>(out));
    return (int)cudaGetLastError();
  }
}

}  // namespace ds
