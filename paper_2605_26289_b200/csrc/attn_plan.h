// Split-KV work decomposition shared by host launch code and device kernels.
// Split boundaries are a pure function of (q-blocks, kv_len): every CTA and
// the combine kernel recompute the same plan, no extra H2D per forward.
#pragma once
#include <stddef.h>
#include <stdint.h>
#include "../../include/deltaserve_b200.h"

#ifdef __CUDACC__
#define DS_HD __host__ __device__ __forceinline__
#else
#define DS_HD inline
#endif

namespace ds {

constexpr int kNumSMs = 148;
// packed query rows (q_len * G) the decode kernel K7 takes; longer entries run
// on the tcgen05 kernel K6 (mirrored by DECODE_MAX_ROWS in engine.py)
constexpr int kDecodeMaxRows = 24;
// K7's key splits of one (entry, kv head) merge inside one thread-block
// cluster (distributed shared memory) when there are at most this many; more
// splits (long contexts: one CTA per SM) write global partials and a combine
// kernel merges them.  A cluster must fit one GPC, so 8 (portable) - larger
// clusters were measured to serialise on GPCs with fewer free SMs.
constexpr int kDecodeMaxCluster = 8;
// K7 runs on tcgen05 (attn_decode_tc.cu) above this many rows when the prefix
// is long enough for the MMA pipe, not the fixed latency, to matter
constexpr int kDecodeTcMinRows = 8;
// beyond a cluster's worth of splits, K7 merges in its last-arriving split CTA
// up to this many rows (measured cheaper than a launch); more rows use the
// combine kernel
constexpr int kDecodeLastMergeRows = 8;
// measured crossover of the forward at q=5 (tools/sweep_env.sh DS_K7_TC_MIN_KEYS):
// m=1k 2.85 (mma.sync) vs 2.84 ms (tcgen05, one-stage), m=2k 2.94 vs 2.90,
// m=4k 3.20 vs 2.99 - the legacy HMMA pipe bounds the mma.sync kernel from
// ~2k keys on (DS_K7_TC_MIN_KEYS overrides, A/B)
constexpr int kDecodeTcMinKeys = 2048;
// K7-tc (R > 8 rows over >= kDecodeTcMinKeys keys) takes at most this many key
// splits and merges them in ONE (non-portable) cluster through distributed
// shared memory when the clusters fit the GPU in one wave - no combine launch
// and no global partials on the critical path.  Off by default (0): on the
// B200 only 7 clusters of 11..16 one-CTA-per-SM CTAs are co-resident (9: 15,
// 10: 11), fewer than the 8 kv heads of one verify entry, so the 16-split
// plan fell back to the combine kernel with fewer CTAs (m=32k q=5 30.5 ->
// 36.9 us); the one-CTA-per-SM plan + attn_combine_kernel stays
#ifndef DS_K7_TC_CLUSTER
#define DS_K7_TC_CLUSTER 0
#endif
constexpr int kDecodeTcMaxCluster = DS_K7_TC_CLUSTER > kDecodeMaxCluster ? DS_K7_TC_CLUSTER
                                                                           : kDecodeMaxCluster;
#ifndef DS_K7_SHORT_TILES
#define DS_K7_SHORT_TILES (8 * kDecodeMaxCluster)
#endif
constexpr int kDecodeShortTiles = DS_K7_SHORT_TILES;  // see attn_split_plan
#ifndef DS_K7_SHORT_SPLITS  // split cap for R > 8 rows over <= kDecodeShortTiles key tiles
#define DS_K7_SHORT_SPLITS kDecodeMaxCluster
#endif
#ifndef DS_K7_SHORT_SPLITS_SMALL  // the same cap for R <= 8 rows (A/B; default: none)
#define DS_K7_SHORT_SPLITS_SMALL 64
#endif
constexpr int kSplitRows = 64;  // packed rows per split-kernel CTA (4 warps x 16)

struct AttnSplitPlan {
  int n_splits;
  int split_len;
};

// mode 0: split kernel (~2 CTAs per SM, ceil); mode 1: warp-specialised decode
// kernel (one CTA per SM, floor so the grid is a single wave).
// rows: the entry's packed query rows.  Decode entries of more than
// kDecodeLastMergeRows rows merge more than a cluster's worth of splits in the
// combine kernel (one more launch, ~6 us per layer in the forward); up to
// kDecodeShortTiles key tiles (8k keys) they take at most a cluster's worth
// of splits instead: q=5 forward at m=2k 3.07 -> 2.98 ms, 4k 3.09 -> 3.02,
// 4.2k 3.10 -> 3.03, 6k 3.08 -> 3.06; a 16k cap was slower from 8k keys on.
DS_HD AttnSplitPlan attn_split_plan(int qblocks, int kv_len, int nkv, int n_entries, int mode,
                                    int rows) {
  const int ctas = qblocks * nkv * n_entries;
  int n = mode ? kNumSMs / ctas : (2 * kNumSMs + ctas - 1) / ctas;
  const int by_len = (kv_len + 127) / 128;
  if (n > by_len) n = by_len;
  if (mode && rows > kDecodeLastMergeRows && n > DS_K7_SHORT_SPLITS &&
      by_len <= kDecodeShortTiles)
    n = DS_K7_SHORT_SPLITS;
  if (mode && rows <= kDecodeLastMergeRows && n > DS_K7_SHORT_SPLITS_SMALL &&
      by_len <= kDecodeShortTiles)
    n = DS_K7_SHORT_SPLITS_SMALL;
  if (DS_K7_TC_CLUSTER > kDecodeMaxCluster && mode && rows > kDecodeTcMinRows &&
      kv_len >= kDecodeTcMinKeys && n > kDecodeTcMaxCluster)
    n = kDecodeTcMaxCluster;
  if (n > 64) n = 64;
  if (n < 1) n = 1;
  const int gran = mode ? 128 : 64;  // key tile of the kernel
  int split_len = ((kv_len + n - 1) / n + gran - 1) / gran * gran;
  n = (kv_len + split_len - 1) / split_len;
  if (n < 1) n = 1;
  return {n, split_len};
}

// rows of partial storage used by entries [0, e)
DS_HD int64_t attn_partial_base(const ds_entry* entries, int e, int n_entries, int nh, int nkv,
                                int mode) {
  int64_t base = 0;
  const int G = nh / nkv;
  for (int i = 0; i < e; ++i) {
    const int R = entries[i].q_len * G;
    const int qb = (R + kSplitRows - 1) / kSplitRows;
    const AttnSplitPlan p =
        attn_split_plan(qb, entries[i].past + entries[i].q_len, nkv, n_entries, mode, R);
    if (p.n_splits > 1) base += static_cast<int64_t>(p.n_splits) * R;
  }
  return base;
}

inline int64_t attn_partial_slots(const ds_entry* entries, int n, int nh, int nkv, int mode) {
  return attn_partial_base(entries, n, n, nh, nkv, mode) * nkv;
}

inline size_t attn_partial_bytes(const ds_entry* entries, int n, int nh, int nkv, int mode) {
  const int64_t slots = attn_partial_slots(entries, n, nh, nkv, mode);
  return static_cast<size_t>(slots) * (128 + 1) * sizeof(float);
}

// upper bound of attn_partial_bytes for any batch (sum over
// split entries of n_splits*qblocks*nkv <= 4*kNumSMs)
size_t prefill_partial_bytes_bound();
inline size_t attn_partial_bytes_bound() {
  const size_t dec = static_cast<size_t>(4 * kNumSMs) * kSplitRows * (128 + 1) * sizeof(float);
  const size_t pre = prefill_partial_bytes_bound();
  return (dec > pre ? dec : pre) + (64 << 10);  // + split-merge counters
}

}  // namespace ds
