// Split-KV merge of the decode kernels (K7 and its tcgen05 variant) inside a
// thread-block cluster through distributed shared memory.  Every split CTA has
// left its normalised rows (cval [R][128]) and log-sum-exp (clse [R]) in its
// own shared memory; the cluster's CTAs then share the R x 128 outputs.
#pragma once
#include "../../include/deltaserve_b200.h"
#include "attn_plan.h"
#include "common.cuh"

namespace ds {

// Called by all `nthreads` merge threads (tid < nthreads) of every CTA in the
// cluster, between two cluster_sync_all(); `bar_id` names a barrier over those
// threads.  cw: [>= R][kDecodeMaxCluster] scratch for the split weights.
DS_DEVICE void decode_cluster_merge(const float* cval, const float* clse, float* cw, int R,
                                    int n_splits, int cluster, int tid, int nthreads, int bar_id,
                                    const ds_entry& en, int nh, int kh, int G,
                                    __nv_bfloat16* __restrict__ out) {
  constexpr int kD = 128;
  const uint32_t rank = cluster_ctarank();
  // per-row split weights 2^(lse_p - max) / sum, in split order
  for (int i = tid; i < R; i += nthreads) {
    float lmax = -INFINITY;
    for (int p = 0; p < n_splits; ++p)
      lmax = fmaxf(lmax, dsmem_ld_f32(dsmem_map(smem_u32(clse + i), p)));
    float wsum = 0.f;
    for (int p = 0; p < n_splits; ++p) {
      const float lse = dsmem_ld_f32(dsmem_map(smem_u32(clse + i), p));
      const float w = lse == -INFINITY ? 0.f : exp2f(lse - lmax);
      cw[i * kDecodeMaxCluster + p] = w;
      wsum += w;
    }
    const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
    for (int p = 0; p < n_splits; ++p) cw[i * kDecodeMaxCluster + p] *= inv;
  }
  named_bar_sync(bar_id, nthreads);
  for (int idx = static_cast<int>(rank) * nthreads + tid; idx < R * kD; idx += cluster * nthreads) {
    const int r = idx / kD, d = idx - r * kD;
    const uint32_t a = smem_u32(cval + r * kD + d);
    float acc = 0.f;
#pragma unroll 4
    for (int p = 0; p < n_splits; ++p)
      acc += cw[r * kDecodeMaxCluster + p] * dsmem_ld_f32(dsmem_map(a, p));
    const int ti = r / G, gi = r - ti * G;
    out[static_cast<int64_t>(en.q_start + ti) * nh * kD + (kh * G + gi) * kD + d] =
        __float2bfloat16_rn(acc);
  }
}

}  // namespace ds
