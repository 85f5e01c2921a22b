// K7 (decode / speculative verify, R = q_len * G <= 24 packed query rows).
//
// HBM-bound: every K/V byte of a split is read once and feeds all R rows (GQA
// packing: row r = t*G + g, so the G query heads sharing a KV head share its
// tiles).  With so few query rows the MMAs run "swapped": keys are the M side
// of m16n8k16 and the packed query rows the N side (n-tiles of 8 rows), so no
// MMA lane is spent on padding rows beyond 8*ceil(R/8):
//   S^T[key][row]  = K[key][:] . Q^T           (A = K tile via ldmatrix,
//                                               B = q rows, held in registers
//                                               for R <= 16, else ldmatrix'd
//                                               from a swizzled smem copy)
//   O^T[d][row]   += V^T[d][key] . P^T[key][row] (A = V tile via ldmatrix.trans,
//                                               B = P^T: the S^T accumulators
//                                               packed to bf16 and transposed
//                                               in registers with movmatrix)
// Warp-specialised, one CTA per SM (9 warps: at most 168 registers per
// thread, since a sub-partition holds three of them):
//   * producer warp: per 128-key tile, when the tile's cells form one run
//     (the common case - first-fit allocation, head-major pool) four 2D TMA
//     boxes (K and V, two 128-byte column halves, SWIZZLE_128B) complete on the
//     stage's mbarrier; otherwise the warp gathers the tile cell by cell with
//     16-byte cp.async into the same swizzled layout.  3 stages x 64 KB;
//   * 8 consumer warps: warp w owns keys [16w, 16w+16) of every tile and keeps
//     its own online-softmax state (running max per row, lazily rescaled O^T);
//     the 8 states merge through smem at the end.
// Programmatic dependent launch: only q and the K/V rows of this batch's own
// positions (>= past) come from the preceding wqkv projection, so the
// producer streams every tile of older keys before the dependency wait - the
// KV read overlaps the projection's tail; consumers wait before loading q.
// Key splits: when a launch has at most kDecodeMaxCluster splits per (entry,
// kv head), those CTAs form a thread-block cluster; each leaves its normalised
// rows + log-sum-exp in shared memory and the cluster merges them through
// distributed shared memory (no global partials, no combine launch - the
// short-context case, where that fixed cost dominates).  Longer contexts write
// split partials (O, lse) for attn_combine_kernel.
#include "../../include/deltaserve_b200.h"
#include "attn_decode_merge.cuh"
#include "attn_plan.h"
#include "common.cuh"
#include "tma.h"

namespace ds {

#ifdef DS_K7_TRACE
// debug build only: per-CTA globaltimer stamps (tools/k7_trace.py)
__device__ unsigned long long g_k7_trace[1024][8];
DS_DEVICE unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// (globaltimer reads are slow enough to perturb the phases: only the cross-CTA
// anchors 6 / 0 / 1 / 5 read it; the phases in between use clock64)
#define K7_STAMP(i)                                                                        \
  if (threadIdx.x == 0 && ((i) == 6 || (i) <= 1 || (i) == 5))                              \
  g_k7_trace[(blockIdx.z * gridDim.y + blockIdx.y) & 1023][i] = gtime()
// SM-clock stamps of thread 0 (same SM: exact intra-CTA deltas)
__device__ long long g_k7_clk[1024][16];
#define K7_CLK(i)                                                                          \
  do {                                                                                     \
    __syncwarp();                                                                          \
    if (threadIdx.x == 0) g_k7_clk[(blockIdx.z * gridDim.y + blockIdx.y) & 1023][i] = clock64(); \
  } while (0)
#else
#define K7_STAMP(i)
#define K7_CLK(i)
#endif

namespace {
constexpr int kD = 128;
constexpr int kTile = 128;                   // keys per stage
constexpr int kBoxBytes = kTile * 128;       // [128 keys][64 d] bf16 = one TMA box
constexpr int kHalfBytes = 2 * kBoxBytes;    // a K (or V) tile
constexpr int kStageBytes = 2 * kHalfBytes;  // K + V = 64 KB
constexpr int kStages = 3;
constexpr int kConsumers = 8;
constexpr int kKeysPerWarp = kTile / kConsumers;  // 16 = the MMA M side
constexpr int kThreads = (kConsumers + 1) * 32;
constexpr int kMaxRows = kDecodeMaxRows;  // NT <= 3; more rows go to K6
constexpr int kQBytes = 32 * kD * 2;

// TMA SWIZZLE_128B layout of a [128 keys][128 d] tile: two 64-column halves of
// 128-byte rows; 16-byte chunk c of a row sits at c ^ (row & 7).
DS_DEVICE int tswz(int row, int chunk16) {
  return (chunk16 >> 3) * kBoxBytes + row * 128 + (((chunk16 & 7) ^ (row & 7)) << 4);
}

// swizzled [row][128 d] bf16 q copy: 16-byte chunk c of row r at c ^ (r & 7)
DS_DEVICE int qswz(int row, int chunk) {
  return row * (kD * 2) + (((chunk & 8) | ((chunk & 7) ^ (row & 7))) << 4);
}

// transpose an 8x8 bf16 matrix held as one packed pair per lane
DS_DEVICE uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}
constexpr int kOsmStride = kD + 4;  // padded [warp][row] stride of the merge buffer (no conflicts)
}  // namespace

// one-shot hint from the forward runtime: bytes to pull into L2 while the
// attention runs (consumed by the next decode launch on this thread)
static thread_local L2Hint g_l2 = {{nullptr, nullptr}, {0, 0}};
void set_attn_l2_prefetch(const void* ptr, int64_t bytes, const void* ptr2, int64_t bytes2) {
  g_l2 = L2Hint{{static_cast<const char*>(ptr), static_cast<const char*>(ptr2)}, {bytes, bytes2}};
}

int launch_attn_decode_tc(const ds_entry* entries_dev, int n_entries, const void* qkv,
                          const void* k_pool, const void* v_pool, int64_t head_stride,
                          const int32_t* pos2cell, int64_t pos_stride, int nh, int nkv,
                          int max_splits, int max_split_len, float scale, void* out,
                          float* part_o, float* part_lse, const L2Hint& l2, int* merged,
                          cudaStream_t stream);

constexpr int kBarBytes = 64;                                     // full/empty mbarriers
constexpr int kMergeBytes = (kMaxRows * kD + kMaxRows + kMaxRows * 8) * 4;  // cval/clse/cw
int decode_smem_bytes(int n_stages) {
  return 1024 + n_stages * kStageBytes + kQBytes + kBarBytes + kMergeBytes;
}

template <int NT>  // n-tiles of 8 packed query rows
__global__ void __launch_bounds__(kThreads, 1) attn_decode_kernel(
    const __nv_bfloat16* __restrict__ qkv, int qkv_stride, const ds_entry* __restrict__ entries,
    int n_entries, int max_splits, const __nv_bfloat16* __restrict__ kpool,
    const __nv_bfloat16* __restrict__ vpool, const int32_t* __restrict__ pos2cell,
    int64_t pos_stride, int nh, int nkv, float scale_log2, __nv_bfloat16* __restrict__ out,
    float* __restrict__ part_o, float* __restrict__ part_lse, int64_t head_stride,
    int* __restrict__ counters, const __grid_constant__ CUtensorMap tmk,
    const __grid_constant__ CUtensorMap tmv, const L2Hint l2,
    int last_merge, int n_stages, int early_trigger, int one_pass) {
  K7_STAMP(6);
  const bool cluster_merge = max_splits <= kDecodeMaxCluster;  // launched with clusters
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // SW128 alignment
  // [ring: n_stages x 64 KB][q 8 KB][barriers][split-merge buffers].  With one
  // stage (every split one tile) the CTA needs < 100 KB, so the next
  // projection's CTA fits beside it and fills its weight ring meanwhile.
  uint8_t* qs = smem + n_stages * kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(qs + kQBytes);
  uint64_t* empty = full + kStages;
  float* cval = reinterpret_cast<float*>(qs + kQBytes + kBarBytes);  // [R][128] this split's rows
  float* clse = cval + kMaxRows * kD;                                 // [R]
  float* cw = clse + kMaxRows;                                        // [R][8] split weights

  const int e = blockIdx.z / max_splits;
  const int split = blockIdx.z - e * max_splits;
  const ds_entry en = entries[e];
  const int G = nh / nkv;
  const int R = en.q_len * G;
  const int kv_len = en.past + en.q_len;
  const AttnSplitPlan plan = attn_split_plan(1, kv_len, nkv, n_entries, 1, R);
  const bool active = split < plan.n_splits;  // idle CTAs still join the cluster merge
  const int kh = blockIdx.y;
  const int k_begin = split * plan.split_len;
  const int k_end = min(k_begin + plan.split_len, kv_len);
  const int ntiles = (k_end - k_begin + kTile - 1) / kTile;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == kConsumers && lane == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    mbar_fence_init();
  }
  __syncthreads();  // barriers initialised

  const int32_t* p2c = pos2cell + static_cast<int64_t>(en.seq) * pos_stride;
  if (!active) {
  } else if (warp == kConsumers) {
    // ================= producer =================
    if (lane == 0) {
      tma_prefetch_desc(&tmk);
      tma_prefetch_desc(&tmv);
    }
    const int64_t hrow = kh * head_stride;
    // cell ids (4 per lane per tile) are prefetched two tiles ahead so their
    // latency never stalls the TMA issue loop
    auto cells = [&](int t, int (&c)[4]) {
      const int kt = k_begin + t * kTile;
      const int nv = t < ntiles ? min(kTile, k_end - kt) : 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i] = lane + 32 * i < nv ? __ldg(p2c + kt + lane + 32 * i) : -1;
    };
    int cur[4], nx1[4], nx2[4];
    cells(0, cur);
    cells(1, nx1);
    bool waited = false;
    for (int it = 0; it < ntiles; ++it) {
      cells(it + 2, nx2);
      const int st = it % n_stages;
      if (it >= n_stages) mbar_wait(&empty[st], ((it / n_stages) - 1) & 1);
      uint8_t* ks = smem + st * kStageBytes;
      uint8_t* vs = ks + kHalfBytes;
      const int kt = k_begin + it * kTile;
      const int nvalid = min(kTile, k_end - kt);
      if (!waited && kt + nvalid > en.past) {  // first tile holding this batch's own K/V
        pdl_wait();
        waited = true;
      }
      const int c0 = __shfl_sync(0xffffffffu, cur[0], 0);
      bool mine = true;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        mine &= lane + 32 * i >= nvalid || cur[i] == c0 + lane + 32 * i;
      if (__all_sync(0xffffffffu, mine)) {  // one contiguous run of cells: 4 TMA boxes
        if (lane == 0) {
          mbar_expect_tx(&full[st], kStageBytes);
          const int row = static_cast<int>(hrow + c0);
          tma_load_2d(ks, &tmk, 0, row, &full[st]);
          tma_load_2d(ks + kBoxBytes, &tmk, 64, row, &full[st]);
          tma_load_2d(vs, &tmv, 0, row, &full[st]);
          tma_load_2d(vs + kBoxBytes, &tmv, 64, row, &full[st]);
        }
      } else {  // fragmented: cell-by-cell 16-byte gathers into the same layout
#pragma unroll 1
        for (int i = 0; i < 4; ++i) {
          const int r = lane + 32 * i;
          const int cl = cur[i] >= 0 ? cur[i] : c0;  // tail rows duplicate a valid cell (masked)
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
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        cur[i] = nx1[i];
        nx1[i] = nx2[i];
      }
    }
    if (!waited) pdl_wait();
    if (early_trigger) pdl_trigger();  // combine kernel / co-resident projection
    if (lane == 0)  // this CTA's share of the next projections' weights -> L2
      l2_prefetch_share(l2, blockIdx.z * gridDim.y + blockIdx.y,
                        static_cast<int64_t>(gridDim.y) * gridDim.z);
  } else {
    // ================= consumers =================
    K7_STAMP(0);
    pdl_wait();  // q comes from the preceding projection
    K7_STAMP(1);
    K7_CLK(0);
    if (early_trigger) pdl_trigger();
    const int g = lane >> 2, t = lane & 3;
    // Q^T as the B operand: qb[j][kk] covers rows 8j + g, d [16kk + 2t, +1] and
    // [16kk + 8 + 2t, +1] - registers for NT <= 2, else a swizzled smem copy
    constexpr bool kQSmem = NT >= 3;
    uint32_t qb[kQSmem ? 1 : NT][8][2];
    int qpos[NT][2];  // absolute position of rows 8j + 2t + h (-1: padding row)
    if constexpr (kQSmem) {
      for (int c = tid; c < 8 * NT * 16; c += kConsumers * 32) {
        const int r = c >> 4, chunk = c & 15;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < R)
          v = *reinterpret_cast<const uint4*>(qkv +
                                              static_cast<int64_t>(en.q_start + r / G) * qkv_stride +
                                              (kh * G + r % G) * kD + chunk * 8);
        *reinterpret_cast<uint4*>(qs + qswz(r, chunk)) = v;
      }
      named_bar_sync(1, kConsumers * 32);
    }
  #pragma unroll
    for (int j = 0; j < NT; ++j) {
      if constexpr (!kQSmem) {
        const int r = 8 * j + g;
        const bool valid = r < R;
        const int rr = valid ? r : 0;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(
            qkv + static_cast<int64_t>(en.q_start + rr / G) * qkv_stride + (kh * G + rr % G) * kD);
  #pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          qb[j][kk][0] = valid ? src[8 * kk + t] : 0u;
          qb[j][kk][1] = valid ? src[8 * kk + 4 + t] : 0u;
        }
      }
  #pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rh = 8 * j + 2 * t + h;
        qpos[j][h] = rh < R ? en.past + rh / G : -1;
      }
    }
    const int64_t base =
        plan.n_splits > 1 && !cluster_merge ? attn_partial_base(entries, e, n_entries, nh, nkv, 1)
                                            : 0;
    if (one_pass) {
      // ---- every tile of the split resident in the ring (short prefixes) ----
      // One softmax pass: the warps' row maxima over all of the split's keys
      // are exchanged first, so every warp's P is relative to the split's max;
      // the P^T fragments are shared through shared memory and the PV product
      // is split by head dimension (warp w: d rows [16w, 16w+16) over every
      // key).  No per-warp O states exist, so there is no online rescaling and
      // no 8-warp merge (the two-round merge was ~2.5 us of the ~8 us a
      // one-tile launch spends after its dependency wait, tools/k7_trace.py).
      float* mxs = cw;  // [8 warps][24 rows] row maxima (cw is free until the cluster merge)
      const int kw = warp * kKeysPerWarp;
      const int k_row = kw + (lane & 7) + ((lane >> 3) & 1) * 8, k_chunk = lane >> 4;
      float s[kStages][NT][4];
      float mx[NT][2];
  #pragma unroll
      for (int j = 0; j < NT; ++j) mx[j][0] = mx[j][1] = -INFINITY;
  #pragma unroll
      for (int it = 0; it < kStages; ++it) {
        if (it >= ntiles) break;
        mbar_wait(&full[it], 0);
        if (it == 0) {
          K7_STAMP(2);
          K7_CLK(1);
        }
        const uint32_t ks_u = smem_u32(smem + it * kStageBytes);
  #pragma unroll
        for (int j = 0; j < NT; ++j) s[it][j][0] = s[it][j][1] = s[it][j][2] = s[it][j][3] = 0.f;
  #pragma unroll
        for (int kk = 0; kk < 8; kk += 2) {
          uint32_t a0[4], a1[4];
          ldsm_x4(a0[0], a0[1], a0[2], a0[3], ks_u + tswz(k_row, 2 * kk + k_chunk));
          ldsm_x4(a1[0], a1[1], a1[2], a1[3], ks_u + tswz(k_row, 2 * kk + 2 + k_chunk));
  #pragma unroll
          for (int j = 0; j < NT; ++j) {
            uint32_t b[4];
            if constexpr (kQSmem) {
              ldsm_x4(b[0], b[1], b[2], b[3],
                      smem_u32(qs) + qswz(8 * j + (lane & 7), 2 * kk + (lane >> 3)));
            } else {
              b[0] = qb[j][kk][0];
              b[1] = qb[j][kk][1];
              b[2] = qb[j][kk + 1][0];
              b[3] = qb[j][kk + 1][1];
            }
            mma_bf16_16816(s[it][j], a0, b[0], b[1]);
            mma_bf16_16816(s[it][j], a1, b[2], b[3]);
          }
        }
        // s[it][j][q]: key kt + g (+8 for q >= 2), row 8j + 2t + (q & 1)
        const int kt = k_begin + it * kTile + kw;
        const bool need_mask = (kt + kKeysPerWarp > k_end) || (kt + kKeysPerWarp - 1 > en.past);
  #pragma unroll
        for (int j = 0; j < NT; ++j)
  #pragma unroll
          for (int q = 0; q < 4; ++q) {
            float v = s[it][j][q] * scale_log2;
            if (need_mask) {
              const int key = kt + g + ((q >> 1) << 3);
              v = (key < k_end && key <= qpos[j][q & 1]) ? v : -INFINITY;
            }
            s[it][j][q] = v;
            mx[j][q & 1] = fmaxf(mx[j][q & 1], v);
          }
      }
  #pragma unroll
      for (int j = 0; j < NT; ++j)
  #pragma unroll
        for (int h = 0; h < 2; ++h) {  // the warp's row max (lanes sharing t)
          float m = mx[j][h];
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
          if (g == 0) mxs[warp * kMaxRows + 8 * j + 2 * t + h] = m;
        }
      named_bar_sync(1, kConsumers * 32);  // maxima published; every warp is done with K
      K7_CLK(2);
      // the K halves of the stages are free now: each tile's P^T fragments go
      // into its own K half, the row sums after stage 0's fragments
      constexpr int kPbsBytes = kConsumers * 3 * 32 * 8;  // [8 warps][NT <= 3][32 lanes] uint2
      float* lsm = reinterpret_cast<float*>(smem + kPbsBytes);  // [8][24]
      float mref[NT][2];
  #pragma unroll
      for (int j = 0; j < NT; ++j)
  #pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = 8 * j + 2 * t + h;
          float m = -INFINITY;
  #pragma unroll
          for (int w = 0; w < kConsumers; ++w) m = fmaxf(m, mxs[w * kMaxRows + r]);
          mref[j][h] = m == -INFINITY ? 0.f : m;
        }
      float l[NT][2];
  #pragma unroll
      for (int j = 0; j < NT; ++j) l[j][0] = l[j][1] = 0.f;
  #pragma unroll
      for (int it = 0; it < kStages; ++it) {
        if (it >= ntiles) break;
        uint2* pbs = reinterpret_cast<uint2*>(smem + it * kStageBytes);
  #pragma unroll
        for (int j = 0; j < NT; ++j) {
          float p[4];
  #pragma unroll
          for (int q = 0; q < 4; ++q) {
            p[q] = fast_exp2(s[it][j][q] - mref[j][q & 1]);
            l[j][q & 1] += p[q];
          }
          // (keys g | g+8, rows 2t, 2t+1) -> transposed: (keys 2t, 2t+1 | +8, row g)
          pbs[(warp * NT + j) * 32 + lane] =
              make_uint2(movm_t(pack_bf16(p[0], p[1])), movm_t(pack_bf16(p[2], p[3])));
        }
      }
  #pragma unroll
      for (int j = 0; j < NT; ++j)
  #pragma unroll
        for (int h = 0; h < 2; ++h) {
          float v = l[j][h];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          if (g == 0) lsm[warp * kMaxRows + 8 * j + 2 * t + h] = v;
        }
      named_bar_sync(1, kConsumers * 32);  // every warp's P^T and row sums published
      K7_CLK(3);
      float o[NT][4];
  #pragma unroll
      for (int j = 0; j < NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
      const int v_row = (lane & 7) + ((lane >> 4) << 3), v_chunk = (lane >> 3) & 1;
  #pragma unroll
      for (int it = 0; it < kStages; ++it) {
        if (it >= ntiles) break;
        const uint32_t vs_u = smem_u32(smem + it * kStageBytes) + kHalfBytes;
        const uint2* pbs = reinterpret_cast<const uint2*>(smem + it * kStageBytes);
  #pragma unroll
        for (int kc = 0; kc < kConsumers; ++kc) {  // keys [16kc, 16kc+16) of the tile
          uint32_t a[4];
          ldsm_x4_t(a[0], a[1], a[2], a[3], vs_u + tswz(16 * kc + v_row, 2 * warp + v_chunk));
  #pragma unroll
          for (int j = 0; j < NT; ++j) {
            const uint2 b2 = pbs[(kc * NT + j) * 32 + lane];
            mma_bf16_16816(o[j], a, b2.x, b2.y);
          }
        }
      }
      K7_STAMP(3);
#ifdef DS_K7_TRACE
      {  // trace build: the stamp waits for the PV products (register dependency)
        float dep = 0.f;
  #pragma unroll
        for (int j = 0; j < NT; ++j) dep += o[j][0] + o[j][3];
        if (dep == 1.2345e30f) g_k7_clk[1023][15] = 1;
      }
#endif
      K7_CLK(4);
      // o[j][q]: d = 16w + g (+8 for q >= 2), row 8j + 2t + (q & 1)
  #pragma unroll
      for (int j = 0; j < NT; ++j) {
        float inv[2], lse[2];
  #pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = 8 * j + 2 * t + h;
          float L = 0.f;
  #pragma unroll
          for (int w = 0; w < kConsumers; ++w) L += lsm[w * kMaxRows + r];
          inv[h] = L > 0.f ? 1.f / L : 0.f;
          lse[h] = L > 0.f ? mref[j][h] + __log2f(L) : -INFINITY;
        }
        if (j == 0) K7_CLK(9);
  #pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = 8 * j + 2 * t + (q & 1), d = 16 * warp + g + ((q >> 1) << 3);
          if (r >= R) continue;
          const float val = o[j][q] * inv[q & 1];
          const bool lead = warp == 0 && g == 0 && q < 2;  // one writer per row's lse
          if (plan.n_splits == 1) {
            const int ti = r / G, gi = r - ti * G;
            out[static_cast<int64_t>(en.q_start + ti) * nh * kD + (kh * G + gi) * kD + d] =
                __float2bfloat16_rn(val);
          } else if (cluster_merge) {
            cval[r * kD + d] = val;
            if (lead) clse[r] = lse[q & 1];
          } else {
            const int64_t slot = (base + static_cast<int64_t>(split) * R + r) * nkv + kh;
            part_o[slot * kD + d] = val;
            if (lead) part_lse[slot] = lse[q & 1];
          }
        }
      }
      K7_CLK(10);
    } else {
      float o[8][NT][4];
      float m_run[NT][2], l_run[NT][2];  // l_run: this lane's keys only (reduced at the end)
    #pragma unroll
      for (int j = 0; j < NT; ++j) {
        m_run[j][0] = m_run[j][1] = -INFINITY;
        l_run[j][0] = l_run[j][1] = 0.f;
    #pragma unroll
        for (int i = 0; i < 8; ++i) o[i][j][0] = o[i][j][1] = o[i][j][2] = o[i][j][3] = 0.f;
      }
      const int kw = warp * kKeysPerWarp;
      // per-lane ldmatrix rows: K (A, row-major) and V (A = V^T via .trans)
      const int k_row = kw + (lane & 7) + ((lane >> 3) & 1) * 8, k_chunk = lane >> 4;
      const int v_row = kw + (lane & 7) + ((lane >> 4) << 3), v_chunk = (lane >> 3) & 1;

      for (int it = 0; it < ntiles; ++it) {
        const int st = it % n_stages;
        mbar_wait(&full[st], (it / n_stages) & 1);
        if (it == 0) K7_STAMP(2);
        const uint32_t ks_u = smem_u32(smem + st * kStageBytes), vs_u = ks_u + kHalfBytes;
        float s[NT][4];
    #pragma unroll
        for (int j = 0; j < NT; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
    #pragma unroll
        for (int kk = 0; kk < 8; kk += 2) {
          uint32_t a0[4], a1[4];
          ldsm_x4(a0[0], a0[1], a0[2], a0[3], ks_u + tswz(k_row, 2 * kk + k_chunk));
          ldsm_x4(a1[0], a1[1], a1[2], a1[3], ks_u + tswz(k_row, 2 * kk + 2 + k_chunk));
    #pragma unroll
          for (int j = 0; j < NT; ++j) {
            uint32_t b[4];
            if constexpr (kQSmem) {
              ldsm_x4(b[0], b[1], b[2], b[3], smem_u32(qs) + qswz(8 * j + (lane & 7), 2 * kk + (lane >> 3)));
            } else {
              b[0] = qb[j][kk][0];
              b[1] = qb[j][kk][1];
              b[2] = qb[j][kk + 1][0];
              b[3] = qb[j][kk + 1][1];
            }
            mma_bf16_16816(s[j], a0, b[0], b[1]);
            mma_bf16_16816(s[j], a1, b[2], b[3]);
          }
        }
        // s[j][q]: key kt + g (+8 for q >= 2), row 8j + 2t + (q & 1)
        const int kt = k_begin + it * kTile + kw;
        const bool need_mask = (kt + kKeysPerWarp > k_end) || (kt + kKeysPerWarp - 1 > en.past);
        uint32_t pb[NT][2];
    #pragma unroll
        for (int j = 0; j < NT; ++j) {
          float mx[2] = {m_run[j][0], m_run[j][1]};
    #pragma unroll
          for (int q = 0; q < 4; ++q) {
            float v = s[j][q] * scale_log2;
            if (need_mask) {
              const int key = kt + g + ((q >> 1) << 3);
              v = (key < k_end && key <= qpos[j][q & 1]) ? v : -INFINITY;
            }
            s[j][q] = v;
            mx[q & 1] = fmaxf(mx[q & 1], v);
          }
          float alpha[2], mref[2];
    #pragma unroll
          for (int h = 0; h < 2; ++h) {  // row max over the warp's 16 keys (lanes sharing t)
            mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 4));
            mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 8));
            mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 16));
            mref[h] = mx[h] == -INFINITY ? 0.f : mx[h];
            alpha[h] = fast_exp2(m_run[j][h] - mref[h]);
            m_run[j][h] = mx[h];
            l_run[j][h] *= alpha[h];
          }
          if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
    #pragma unroll
            for (int i = 0; i < 8; ++i) {
              o[i][j][0] *= alpha[0];
              o[i][j][1] *= alpha[1];
              o[i][j][2] *= alpha[0];
              o[i][j][3] *= alpha[1];
            }
          }
          float p[4];
    #pragma unroll
          for (int q = 0; q < 4; ++q) {
            p[q] = fast_exp2(s[j][q] - mref[q & 1]);
            l_run[j][q & 1] += p[q];
          }
          // (keys g | g+8, rows 2t, 2t+1) -> transposed: (keys 2t, 2t+1 | +8, row g)
          pb[j][0] = movm_t(pack_bf16(p[0], p[1]));
          pb[j][1] = movm_t(pack_bf16(p[2], p[3]));
        }
    #pragma unroll
        for (int i = 0; i < 8; ++i) {  // d rows [16i, 16i+16)
          uint32_t a[4];
          ldsm_x4_t(a[0], a[1], a[2], a[3], vs_u + tswz(v_row, 2 * i + v_chunk));
    #pragma unroll
          for (int j = 0; j < NT; ++j) mma_bf16_16816(o[i][j], a, pb[j][0], pb[j][1]);
        }
        // generic-proxy reads of the stage complete before the producer's TMA
        // (async proxy) refills it (measured necessary in the skinny GEMM ring)
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
      named_bar_sync(1, kConsumers * 32);  // all consumers done with the ring
      K7_STAMP(3);

      // ---- merge the 8 warps' states (ring memory is free now) ----
      // Two rounds through a [4][24][132] buffer (fits the one-stage ring):
      // warps 4-7 publish (m, l, O), warps 0-3 fold their partner's state into
      // registers and publish the result; then per-row weights are computed once
      // and every output element is a 4-term dot product (independent loads).
      constexpr int kHalfW = kConsumers / 2;
      float* osm = reinterpret_cast<float*>(smem);             // [4][24][132]
      float* msm = osm + kHalfW * kMaxRows * kOsmStride;       // [4][24]
      float* lsm = msm + kHalfW * kMaxRows;                    // [4][24]
      float* wsm = lsm + kHalfW * kMaxRows;                    // [24][4] row weights
      float* rlse = wsm + kMaxRows * kHalfW;                   // [24] row log2-sum-exp
      const int slotw = warp & (kHalfW - 1);
    #pragma unroll
      for (int j = 0; j < NT; ++j)
    #pragma unroll
        for (int h = 0; h < 2; ++h) {
          float l = l_run[j][h];
          l += __shfl_xor_sync(0xffffffffu, l, 4);
          l += __shfl_xor_sync(0xffffffffu, l, 8);
          l += __shfl_xor_sync(0xffffffffu, l, 16);
          l_run[j][h] = l;  // the warp's row total
        }
      auto publish = [&]() {
    #pragma unroll
        for (int j = 0; j < NT; ++j) {
    #pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = 8 * j + 2 * t + h;
            if (g == 0) {
              msm[slotw * kMaxRows + r] = m_run[j][h];
              lsm[slotw * kMaxRows + r] = l_run[j][h];
            }
          }
    #pragma unroll
          for (int i = 0; i < 8; ++i)
    #pragma unroll
            for (int q = 0; q < 4; ++q)
              osm[(slotw * kMaxRows + 8 * j + 2 * t + (q & 1)) * kOsmStride + 16 * i + g +
                  ((q >> 1) << 3)] = o[i][j][q];
        }
      };
      if (warp >= kHalfW) publish();
      named_bar_sync(1, kConsumers * 32);
      if (warp < kHalfW) {  // fold the partner warp (warp + 4): same fragment positions
    #pragma unroll
        for (int j = 0; j < NT; ++j)
    #pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = 8 * j + 2 * t + h;
            const float mb = msm[slotw * kMaxRows + r], lb = lsm[slotw * kMaxRows + r];
            const float ma = m_run[j][h];
            const float mm = fmaxf(ma, mb);
            const float mref = mm == -INFINITY ? 0.f : mm;
            const float sa = fast_exp2(ma - mref), sb = fast_exp2(mb - mref);
            m_run[j][h] = mm;
            l_run[j][h] = l_run[j][h] * sa + lb * sb;
    #pragma unroll
            for (int i = 0; i < 8; ++i)
    #pragma unroll
              for (int q = 0; q < 4; ++q)
                if ((q & 1) == h) {
                  const float ob = osm[(slotw * kMaxRows + r) * kOsmStride + 16 * i + g +
                                       ((q >> 1) << 3)];
                  o[i][j][q] = o[i][j][q] * sa + ob * sb;
                }
          }
      }
      named_bar_sync(1, kConsumers * 32);
      if (warp < kHalfW) publish();
      named_bar_sync(1, kConsumers * 32);
      if (tid < R) {
        float mv[kHalfW], lv[kHalfW];
    #pragma unroll
        for (int w = 0; w < kHalfW; ++w) {
          mv[w] = msm[w * kMaxRows + tid];
          lv[w] = lsm[w * kMaxRows + tid];
        }
        float mm = -INFINITY;
    #pragma unroll
        for (int w = 0; w < kHalfW; ++w) mm = fmaxf(mm, mv[w]);
        const float mref = mm == -INFINITY ? 0.f : mm;
        float L = 0.f;
    #pragma unroll
        for (int w = 0; w < kHalfW; ++w) {
          mv[w] = fast_exp2(mv[w] - mref);
          L += lv[w] * mv[w];
        }
        const float inv = L > 0.f ? 1.f / L : 0.f;
    #pragma unroll
        for (int w = 0; w < kHalfW; ++w) wsm[tid * kHalfW + w] = mv[w] * inv;
        rlse[tid] = L > 0.f ? mm + __log2f(L) : -INFINITY;
      }
      named_bar_sync(1, kConsumers * 32);
      for (int idx = tid; idx < R * kD; idx += kConsumers * 32) {
        const int r = idx / kD, d = idx - r * kD;
        float ov[kHalfW];
    #pragma unroll
        for (int w = 0; w < kHalfW; ++w) ov[w] = osm[(w * kMaxRows + r) * kOsmStride + d];
        float val = 0.f;
    #pragma unroll
        for (int w = 0; w < kHalfW; ++w) val += wsm[r * kHalfW + w] * ov[w];
        if (plan.n_splits == 1) {  // no split: write the row directly
          const int ti = r / G, gi = r - ti * G;
          out[static_cast<int64_t>(en.q_start + ti) * nh * kD + (kh * G + gi) * kD + d] =
              __float2bfloat16_rn(val);
        } else if (cluster_merge) {  // this split's normalised rows -> its cluster buffer
          cval[r * kD + d] = val;
          if (d == 0) clse[r] = rlse[r];
        } else {  // -> global partials
          const int64_t slot = (base + static_cast<int64_t>(split) * R + r) * nkv + kh;
          part_o[slot * kD + d] = val;
          if (d == 0) part_lse[slot] = rlse[r];
        }
      }
    }
    if (plan.n_splits > 1 && !cluster_merge && last_merge)  // last split to arrive merges
      decode_global_merge(part_o, part_lse, base, R, plan.n_splits, nkv, kh,
                          counters + e * nkv + kh, cval, reinterpret_cast<int*>(clse), tid,
                          kConsumers * 32, 1, en, nh, G, out);
  }

  // ---- split merge across the cluster (distributed shared memory) ----
  K7_CLK(11);
  K7_STAMP(4);
  K7_CLK(5);
  if (cluster_merge && plan.n_splits > 1) {
    cluster_sync_all();  // every split's rows are in its cbuf
    K7_CLK(6);
    if (tid < kConsumers * 32)
      decode_cluster_merge(cval, clse, cw, R, plan.n_splits, max_splits, tid, kConsumers * 32, 1,
                           en, nh, kh, G, out);
    K7_CLK(7);
    cluster_sync_all();  // peers keep their smem until every read is done
    K7_CLK(8);
  }
  // PDL: when the dependent is the next projection it launches only as this
  // grid retires - an earlier trigger (even after the main loop) let its CTAs
  // onto the SMs while the attention ran and the forward was measured ~25%
  // slower; the small combine kernel (R > 8 beyond a cluster) is triggered
  // early above.
  K7_STAMP(5);
  pdl_trigger();
}

#ifdef DS_K7_TRACE
extern "C" int ds_debug_k7_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_k7_trace, sizeof(g_k7_trace));
}
extern "C" int ds_debug_k7_clk(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_k7_clk, sizeof(g_k7_clk));
}
#endif

int launch_attn_decode(const void* qkv, const ds_entry* entries_host, const ds_entry* entries_dev,
                       int n_entries, const void* k_pool, const void* v_pool, int64_t head_stride,
                       const int32_t* pos2cell, int64_t pos_stride, int nh, int nkv, int max_R,
                       int max_splits, float scale, void* out, float* part_o, float* part_lse,
                       int* counters, int* merged, cudaStream_t stream) {
  if (max_R > kMaxRows) return DS_EUNSUPPORTED;
  *merged = max_splits <= kDecodeMaxCluster || max_R <= kDecodeLastMergeRows;
  int max_kv = 0, max_split_len = 0;
  for (int e = 0; e < n_entries; ++e) {
    const int kv = entries_host[e].past + entries_host[e].q_len;
    max_kv = kv > max_kv ? kv : max_kv;
    const AttnSplitPlan p =
        attn_split_plan(1, kv, nkv, n_entries, 1, entries_host[e].q_len * (nh / nkv));
    max_split_len = p.split_len > max_split_len ? p.split_len : max_split_len;
  }
  // one K/V tile per split (short prefixes): a one-stage ring keeps the CTA
  // small enough for the next projection's CTA to sit beside it
  const int n_stages = max_split_len <= kTile ? 1 : kStages;
  const int smem = decode_smem_bytes(n_stages);
  static bool attr = false;
  if (!attr) {
    const int mx = decode_smem_bytes(kStages);
    cudaFuncSetAttribute(attn_decode_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(attn_decode_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(attn_decode_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    attr = true;
  }
  const CUtensorMap* tk = kv_tensor_map(k_pool, static_cast<int64_t>(nkv) * head_stride, kTile);
  const CUtensorMap* tv = kv_tensor_map(v_pool, static_cast<int64_t>(nkv) * head_stride, kTile);
  if (!tk || !tv) return DS_EUNSUPPORTED;
  dim3 grid(1, nkv, n_entries * max_splits);
  const float sl2 = scale * 1.4426950408889634f;
  const int stride = (nh + 2 * nkv) * kD;
  // more splits than a cluster: up to 8 rows the last split to arrive merges
  // (cheap: R*128 values), more rows go to attn_combine_kernel (attn_split.cu)
  const int last_merge = max_R <= kDecodeLastMergeRows;
  // PDL trigger right after the dependency wait when the dependent is the
  // combine kernel, or (DS_K7_EARLY) when a one-stage CTA leaves room for the
  // next projection's
  static const int early_env = getenv("DS_K7_EARLY") ? atoi(getenv("DS_K7_EARLY")) : 1;
  const int early = (max_splits > kDecodeMaxCluster && !last_merge) || (early_env && n_stages == 1);
  static const int one_pass_env = getenv("DS_K7_ONEPASS") ? atoi(getenv("DS_K7_ONEPASS")) : 1;
  // every split's tiles fit the ring at once: the one-pass softmax (no refills)
  const int one_pass = one_pass_env && max_split_len <= kStages * kTile;
  const L2Hint l2 = g_l2;
  g_l2 = L2Hint{{nullptr, nullptr}, {0, 0}};
  // more than 8 rows over a long prefix: the legacy HMMA pipe would bound the
  // mma.sync kernel below the HBM rate - run the tcgen05 variant
  static const int tc_min_keys =
      getenv("DS_K7_TC_MIN_KEYS") ? atoi(getenv("DS_K7_TC_MIN_KEYS")) : kDecodeTcMinKeys;
  if (max_R > kDecodeTcMinRows && max_kv >= tc_min_keys)
    return launch_attn_decode_tc(entries_dev, n_entries, qkv, k_pool, v_pool, head_stride,
                                 pos2cell, pos_stride, nh, nkv, max_splits, max_split_len, scale,
                                 out, part_o, part_lse, l2, merged, stream);
  auto kern = max_R <= 8 ? attn_decode_kernel<1>
              : max_R <= 16 ? attn_decode_kernel<2>
                            : attn_decode_kernel<3>;
  if (max_splits <= kDecodeMaxCluster)
    launch_pdl_cluster_z(kern, grid, dim3(kThreads), smem, max_splits, stream,
                         static_cast<const __nv_bfloat16*>(qkv), stride, entries_dev, n_entries,
                         max_splits, static_cast<const __nv_bfloat16*>(k_pool),
                         static_cast<const __nv_bfloat16*>(v_pool), pos2cell, pos_stride, nh, nkv,
                         sl2, static_cast<__nv_bfloat16*>(out), part_o, part_lse, head_stride,
                         counters, *tk, *tv, l2, last_merge, n_stages, early, one_pass);
  else
    launch_pdl(kern, grid, dim3(kThreads), smem, stream, static_cast<const __nv_bfloat16*>(qkv),
               stride, entries_dev, n_entries, max_splits,
               static_cast<const __nv_bfloat16*>(k_pool),
               static_cast<const __nv_bfloat16*>(v_pool), pos2cell, pos_stride, nh, nkv, sl2,
               static_cast<__nv_bfloat16*>(out), part_o, part_lse, head_stride, counters, *tk,
               *tv, l2, last_merge, n_stages, early, one_pass);
  return (int)cudaGetLastError();
}

}  // namespace ds
