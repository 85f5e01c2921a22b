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
// cluster, between two cluster_sync_all().  One remote round trip per output
// float4: each thread issues the row's split lse values and its split O
// columns (float4) together, then forms the split weights 2^(lse_p - max) /
// sum in split order (the same arithmetic as a per-row weight pass, without
// its barrier and second round trip).  cw and bar_id are unused (kept for the
// callers' layout).
template <int MAXC = kDecodeMaxCluster>  // the largest cluster the caller launches
DS_DEVICE void decode_cluster_merge(const float* cval, const float* clse, float* cw, int R,
                                    int n_splits, int cluster, int tid, int nthreads, int bar_id,
                                    const ds_entry& en, int nh, int kh, int G,
                                    __nv_bfloat16* __restrict__ out) {
  constexpr int kD = 128, kD4 = kD / 4;
  (void)cw;
  (void)bar_id;
  const uint32_t rank = cluster_ctarank();
  for (int idx = static_cast<int>(rank) * nthreads + tid; idx < R * kD4;
       idx += cluster * nthreads) {
    const int r = idx / kD4, d4 = idx - r * kD4;
    const uint32_t a = smem_u32(cval + r * kD + 4 * d4), al = smem_u32(clse + r);
    float4 v[MAXC];
    float lv[MAXC];
#pragma unroll
    for (int p = 0; p < MAXC; ++p) {
      v[p] = p < n_splits ? dsmem_ld_f32x4(dsmem_map(a, p)) : make_float4(0.f, 0.f, 0.f, 0.f);
      lv[p] = p < n_splits ? dsmem_ld_f32(dsmem_map(al, p)) : -INFINITY;
    }
    float lmax = -INFINITY;
#pragma unroll
    for (int p = 0; p < MAXC; ++p) lmax = fmaxf(lmax, lv[p]);
    float wsum = 0.f;
#pragma unroll
    for (int p = 0; p < MAXC; ++p) {
      lv[p] = lv[p] == -INFINITY ? 0.f : exp2f(lv[p] - lmax);
      wsum += lv[p];
    }
    const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int p = 0; p < MAXC; ++p) {
      const float w = lv[p] * inv;
      acc.x += w * v[p].x;
      acc.y += w * v[p].y;
      acc.z += w * v[p].z;
      acc.w += w * v[p].w;
    }
    const int ti = r / G, gi = r - ti * G;
    __nv_bfloat16* dst =
        out + static_cast<int64_t>(en.q_start + ti) * nh * kD + (kh * G + gi) * kD + 4 * d4;
    *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
  }
}

// More splits than a cluster holds (long prefixes, one CTA per SM): every
// split CTA has written its normalised rows and lse to the global partials
// (slot = (base + split*R + r)*nkv + kh); the LAST split to arrive (one
// counter per (entry, kv head), self re-arming) merges them - no combine
// launch on the critical path, and the grid still triggers its dependent only
// as it retires.  Called by all `nthreads` threads of an active split CTA;
// sw: smem [kDecodeMaxRows][64] split weights, s_flag: one smem int.
DS_DEVICE void decode_global_merge(const float* part_o, const float* part_lse, int64_t base,
                                   int R, int n_splits, int nkv, int kh, int* counter, float* sw,
                                   int* s_flag, int tid, int nthreads, int bar_id,
                                   const ds_entry& en, int nh, int G,
                                   __nv_bfloat16* __restrict__ out) {
  constexpr int kD = 128;
  __threadfence();  // this thread's partial stores before the arrival
  named_bar_sync(bar_id, nthreads);
  if (tid == 0) *s_flag = atomicAdd(counter, 1) == n_splits - 1;
  named_bar_sync(bar_id, nthreads);
  if (!*s_flag) return;
  __threadfence();  // acquire: every split's partials are visible
  const int64_t sstride = static_cast<int64_t>(R) * nkv;
  for (int i = tid; i < R; i += nthreads) {
    const float* lp = part_lse + (base + i) * nkv + kh;
    float lmax = -INFINITY;
    for (int p = 0; p < n_splits; ++p) {
      const float v = __ldcg(lp + p * sstride);
      sw[i * 64 + p] = v;
      lmax = fmaxf(lmax, v);
    }
    float wsum = 0.f;
    for (int p = 0; p < n_splits; ++p) {
      const float lse = sw[i * 64 + p];
      const float w = lse == -INFINITY ? 0.f : exp2f(lse - lmax);
      sw[i * 64 + p] = w;
      wsum += w;
    }
    const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
    for (int p = 0; p < n_splits; ++p) sw[i * 64 + p] *= inv;
  }
  named_bar_sync(bar_id, nthreads);
  for (int idx = tid; idx < R * (kD / 4); idx += nthreads) {
    const int r = idx / (kD / 4), d4 = idx - r * (kD / 4);
    const float4* src =
        reinterpret_cast<const float4*>(part_o + ((base + r) * nkv + kh) * kD) + d4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p0 = 0; p0 < n_splits; p0 += 8) {
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        v[j] = p0 + j < n_splits ? __ldcg(src + (p0 + j) * sstride * (kD / 4))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float w = p0 + j < n_splits ? sw[r * 64 + p0 + j] : 0.f;
        acc.x += w * v[j].x;
        acc.y += w * v[j].y;
        acc.z += w * v[j].z;
        acc.w += w * v[j].w;
      }
    }
    const int ti = r / G, gi = r - ti * G;
    __nv_bfloat16* dst =
        out + static_cast<int64_t>(en.q_start + ti) * nh * kD + (kh * G + gi) * kD + 4 * d4;
    *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
  }
  if (tid == 0) *counter = 0;  // re-arm for the next launch (stream ordered)
}

}  // namespace ds
