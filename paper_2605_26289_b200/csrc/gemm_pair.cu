// K11: projection GEMM for large row counts (prefill chunks of hundreds of
// tokens, batched multi-session plans) on CTA pairs:  Y[T][N] (+)= X[T][K] . W[N][K]^T.
//
// The compute-bound regime (T >= ~256; the weight-streaming regime below it is
// K10 / the library path).  Tile = 256 tokens (UMMA M,
// 128 per CTA of the pair) x 256 features (UMMA N, each CTA loads 128 weight
// rows) x K in 64-column stages: one `tcgen05.mma.cta_group::2` (M=256, N=256,
// K=16) issued by the leader CTA covers both SMs, each CTA holding half of
// both operands in its shared memory and its 128 token rows x 256 features of
// the fp32 accumulator in its own TMEM.  Operand bytes per SM per stage: 32 KB
// for 2 x 256 x 256 x 64 FLOP of the pair.
//
// Orientation: tokens on the MMA M side (TMEM lanes), features on N
// (columns), so an epilogue thread owns one token row and 32 consecutive
// features per tcgen05.ld - the fused epilogues need no transpose: RoPE pairs
// (features f, f+8 of a 16-row tile) and gate/up (8-row interleave) are in one
// thread's registers, row scales and row sums are per thread.
//
// Schedule: persistent, one CTA pair per two SMs, tiles round-robin over the
// pairs, token tiles of one weight tile adjacent (the weight tile's second
// read hits L2); the accumulator is double-buffered (2 x 256 TMEM columns) so
// a tile's epilogue overlaps the next tile's main loop.
//
// Warp roles (224 threads):
//   warps 0, 6  TMA producers (both CTAs): per stage one 16 KB box of this
//            CTA's 128 token rows (warp 0) and one of its 128 weight rows
//            (warp 6); the completion bytes of BOTH CTAs land on the leader's
//            `full` barrier (cta_group::2 TMA, peer bit cleared); the weight
//            boxes of the first ring round are issued before the
//            programmatic-dependency wait;
//   warp 1   TMEM allocation (cta_group::2, both CTAs) and, in the leader,
//            the single-thread MMA issue; stage release / accumulator hand-off
//            through tcgen05.commit multicast to both CTAs' barriers;
//   warps 2-5 epilogue (both CTAs), thread = token row (TMEM lane quadrant
//            warp & 3); arrive on the leader's `acc_empty` when the
//            accumulator buffer is read.
#include "../../include/deltaserve_b200.h"
#include "common.cuh"
#include "tc.cuh"
#include "tma.h"

#include <cstdio>
#include <cstdlib>

namespace ds {

namespace {
constexpr int kPM = 128;                 // token rows per CTA (256 per pair)
constexpr int kPN = 256;                 // features per tile (128 loaded per CTA)
constexpr int kBoxA = kPM * 128;         // 16 KB: 128 token rows x 64 columns
constexpr int kBoxB = (kPN / 2) * 128;   // 16 KB: 128 weight rows x 64 columns
constexpr int kStage = kBoxA + kBoxB;
constexpr int kPairThreads = 11 * 32;  // producers 0 / 6, MMA 1, epilogue 2-5 + 7-10
constexpr int kPairSmemMax = 227 * 1024;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // leader's barrier in the shared::cluster window

struct PairArgs {
  void* Y;
  float* partials;  // [pairs][2 CTAs][kPM rows][kPN] fp32 (stream-K segments)
  int* flags;       // [pairs][2]: partial written (self re-arming)
  int T, N, K, y_f32, accumulate;
  int n_tt, tiles, kt, stages;
  int full_waves, rem, split;  // tiles = full_waves * groups + rem; tail tiles split `split` ways
  int G;                       // pairs per cluster sharing the token tile (1, or 2: multicast)
};

// segment `idx` of pair `pair`: the full-wave tiles round-robin (concurrent
// tiles adjacent: a weight tile and the token tiles stay in L2), then at most
// one unit of the tail - the last rem < pairs tiles, each cut into `split`
// equal k ranges (split 0 finishes the tile, the others leave fp32 partials)
struct Seg {
  int tile, kb, ke, j;
};
DS_DEVICE int n_segs(const PairArgs& a, int pair) {
  return a.full_waves + (pair < a.rem * a.split ? 1 : 0);
}
DS_DEVICE Seg seg_of(const PairArgs& a, int pair, int n_pairs, int idx) {
  Seg g;
  if (idx < a.full_waves) {
    g.tile = idx * n_pairs + pair;
    g.kb = 0;
    g.ke = a.kt;
    g.j = 0;
  } else {
    g.tile = a.full_waves * n_pairs + pair / a.split;
    g.j = pair % a.split;
    g.kb = g.j * a.kt / a.split;
    g.ke = (g.j + 1) * a.kt / a.split;
  }
  return g;
}

DS_DEVICE void tma_load_3d_pair(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar) & kPeerMask)
      : "memory");
}
// the same, multicast to the cluster CTAs in `mask` (each pair's leader barrier)
DS_DEVICE void tma_load_3d_pair_mc(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                   uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar) & kPeerMask), "h"(mask)
      : "memory");
}
DS_DEVICE void alloc_pair(uint32_t* smem_dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(smem_dst)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
}
DS_DEVICE void dealloc_pair(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(cols));
}
DS_DEVICE void mma_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                        uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// every prior MMA of this thread complete -> one arrive on `bar` in the
// cluster CTAs of `mask`
DS_DEVICE void commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;\n" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
DS_DEVICE int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
DS_DEVICE void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
DS_DEVICE void arrive_leader(uint64_t* bar, uint32_t leader_rank) {  // the pair leader's copy
  const uint32_t ra = dsmem_map(smem_u32(bar), leader_rank);
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(ra)
               : "memory");
}

constexpr float kSsScale = 16777216.f;  // 2^24 fixed point row sums (as K10 / the decode GEMM)
DS_DEVICE float bf16r(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
DS_DEVICE uint32_t pk(float x, float y) { return pack_bf16(x, y); }

// per token row and tile: the row scalars of the fused epilogues
struct RowCtx {
  float inv;     // norm consumer: rsqrt(row_ss / K + eps)
  int pos;       // RoPE position
  int64_t cell;  // KV-store cell
  long long ssq; // residual producer: sum of x^2 in 2^-24 fixed point
  unsigned long long amax;  // LM head: packed (value, lowest column) max
};

// the fused epilogue of 32 consecutive features [f0, f0 + 32) of token row t,
// thread = row (the same semantics and bf16 storage points as K10's
// epilogue_chunk / the decode GEMM, gemm_skinny.cu)
DS_DEVICE void pair_epilogue(float* v, const PairArgs& a, const ds_skinny_epi& epi, int t, int f0,
                             RowCtx& rc) {
  if (epi.row_ss) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] *= rc.inv;
  }
  if (epi.rope) {
    constexpr int kHd = 128, kHalf = 64;
    const int qk_width = (epi.n_heads + epi.n_kv_heads) * kHd;
    if (f0 < qk_width) {
      // two 16-feature groups; in a group, features jj < 8 hold dims 8b + jj
      // and jj >= 8 the partner dims 64 + 8b + (jj - 8)  (b = group in head)
      const int head = f0 / kHd;
      __nv_bfloat16* row =
          head < epi.n_heads
              ? static_cast<__nv_bfloat16*>(a.Y) + static_cast<int64_t>(t) * a.N + head * kHd
              : static_cast<__nv_bfloat16*>(epi.k_pool_l) +
                    ((head - epi.n_heads) * epi.kv_head_stride + rc.cell) * kHd;
#pragma unroll
      for (int gq = 0; gq < 2; ++gq) {
        const int b = ((f0 % kHd) >> 4) + gq;  // group within the head
        const float4* cs4 =
            reinterpret_cast<const float4*>(epi.rope_cos + static_cast<int64_t>(rc.pos) * kHalf + 8 * b);
        const float4* sn4 =
            reinterpret_cast<const float4*>(epi.rope_sin + static_cast<int64_t>(rc.pos) * kHalf + 8 * b);
        const float4 c0 = __ldg(cs4), c1 = __ldg(cs4 + 1), s0 = __ldg(sn4), s1 = __ldg(sn4 + 1);
        const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        const float ss[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
        float lo[8], hi[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float x = bf16r(v[16 * gq + j]), p = bf16r(v[16 * gq + 8 + j]);  // stored in bf16
          lo[j] = x * cc[j] - p * ss[j];
          hi[j] = p * cc[j] + x * ss[j];
        }
        *reinterpret_cast<uint4*>(row + 8 * b) =
            make_uint4(pk(lo[0], lo[1]), pk(lo[2], lo[3]), pk(lo[4], lo[5]), pk(lo[6], lo[7]));
        *reinterpret_cast<uint4*>(row + kHalf + 8 * b) =
            make_uint4(pk(hi[0], hi[1]), pk(hi[2], hi[3]), pk(hi[4], hi[5]), pk(hi[6], hi[7]));
      }
      return;
    }
    const int fv = f0 - qk_width;  // v rows: 32 consecutive dims of one kv head
    uint4* d = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(epi.v_pool_l) +
                                        ((fv / kHd) * epi.kv_head_stride + rc.cell) * kHd + fv % kHd);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      d[q] = make_uint4(pk(v[8 * q], v[8 * q + 1]), pk(v[8 * q + 2], v[8 * q + 3]),
                        pk(v[8 * q + 4], v[8 * q + 5]), pk(v[8 * q + 6], v[8 * q + 7]));
    return;
  }
  if (epi.swiglu) {  // gate jj < 8, up jj >= 8 of the same 8 FFN units per group
    float o[16];
#pragma unroll
    for (int gq = 0; gq < 2; ++gq)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float gg = bf16r(v[16 * gq + j]), uu = bf16r(v[16 * gq + 8 + j]);
        o[8 * gq + j] = gg / (1.f + expf(-gg)) * uu;
      }
    uint4* d = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.Y) +
                                        static_cast<int64_t>(t) * (a.N / 2) + f0 / 2);
    d[0] = make_uint4(pk(o[0], o[1]), pk(o[2], o[3]), pk(o[4], o[5]), pk(o[6], o[7]));
    d[1] = make_uint4(pk(o[8], o[9]), pk(o[10], o[11]), pk(o[12], o[13]), pk(o[14], o[15]));
    return;
  }
  const int64_t off = static_cast<int64_t>(t) * a.N + f0;
  if (epi.argmax_out) {
    if (a.Y) {
      float4* y = reinterpret_cast<float4*>(static_cast<float*>(a.Y) + off);
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const unsigned long long k = argmax_key(v[j], f0 + j);
      rc.amax = k > rc.amax ? k : rc.amax;
    }
    return;
  }
  if (a.y_f32) {
    float4* yp = reinterpret_cast<float4*>(static_cast<float*>(a.Y) + off);
    if (a.accumulate) {
      float4 old[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) old[q] = yp[q];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[4 * q] += old[q].x;
        v[4 * q + 1] += old[q].y;
        v[4 * q + 2] += old[q].z;
        v[4 * q + 3] += old[q].w;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) yp[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
    uint4* yp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.Y) + off);
    if (a.accumulate) {
      uint4 old[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) old[q] = yp[q];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t pw[4] = {old[q].x, old[q].y, old[q].z, old[q].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pw[j]));
          v[8 * q + 2 * j] += f.x;
          v[8 * q + 2 * j + 1] += f.y;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = bf16r(v[j]);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      yp[q] = make_uint4(pk(v[8 * q], v[8 * q + 1]), pk(v[8 * q + 2], v[8 * q + 3]),
                         pk(v[8 * q + 4], v[8 * q + 5]), pk(v[8 * q + 6], v[8 * q + 7]));
  }
  if (epi.ss_out) {  // residual producer: next RMSNorm's weight multiply + row sums
    if (epi.h_out && epi.h_w) {
      const uint4* hw = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(epi.h_w) + f0);
      uint4* ho = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(epi.h_out) + off);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 wu = __ldg(hw + q);
        const uint32_t ww[4] = {wu.x, wu.y, wu.z, wu.w};
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 w2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ww[j]));
          o[j] = pk(v[8 * q + 2 * j] * w2.x, v[8 * q + 2 * j + 1] * w2.y);
        }
        ho[q] = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) rc.ssq += __float2ll_rn(v[j] * v[j] * kSsScale);
  }
}

// plain / residual outputs through a per-warp transpose: the warp's 32 token
// rows x 32 features staged in shared memory, then 8 lanes per row move one
// contiguous 128-byte fp32 (64-byte bf16) row segment, 4 rows per
// instruction - the residual read-modify-write and the h stores are whole
// segments (thread-per-row 16-byte pieces left the epilogue exposed at the
// end of the GEMM: +30 us on wo at 4096 rows).  Row sums of x^2 collect in
// ss_acc[32] (one global atomic per row and tile).
constexpr int kStgP = 33;  // staging row stride (floats): conflict-free both ways
DS_DEVICE void pair_store_staged(const float* v, const PairArgs& a, const ds_skinny_epi& epi,
                                 int t0w, int f0, float* stg, long long* ss_acc, int lane) {
#pragma unroll
  for (int j = 0; j < 32; ++j) stg[lane * kStgP + j] = v[j];
  __syncwarp();
  const int g = lane & 7, rr = lane >> 3;
  float4 hw4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const bool h = epi.ss_out && epi.h_out && epi.h_w;
  if (h) {
    const uint2 hu = __ldg(reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(epi.h_w) + f0 + 4 * g));
    const float2 h0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hu.x));
    const float2 h1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hu.y));
    hw4 = make_float4(h0.x, h0.y, h1.x, h1.y);
  }
  float4 y4[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float* sp = stg + (rr + 4 * i) * kStgP + 4 * g;
    y4[i] = make_float4(sp[0], sp[1], sp[2], sp[3]);
  }
  if (a.accumulate) {  // every old value in flight before the first use
    float4 old[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int t = t0w + rr + 4 * i;
      const int64_t o = static_cast<int64_t>(t) * a.N + f0 + 4 * g;
      old[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < a.T) {
        if (a.y_f32) {
          old[i] = *reinterpret_cast<const float4*>(static_cast<const float*>(a.Y) + o);
        } else {
          const uint2 u = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(a.Y) + o);
          const float2 p0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
          const float2 p1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
          old[i] = make_float4(p0.x, p0.y, p1.x, p1.y);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      y4[i].x += old[i].x;
      y4[i].y += old[i].y;
      y4[i].z += old[i].z;
      y4[i].w += old[i].w;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = rr + 4 * i, t = t0w + row;
    const bool ok = t < a.T;
    const int64_t o = static_cast<int64_t>(t) * a.N + f0 + 4 * g;
    float4 y = y4[i];
    if (ok) {
      if (a.y_f32) {
        *reinterpret_cast<float4*>(static_cast<float*>(a.Y) + o) = y;
      } else {
        y = make_float4(bf16r(y.x), bf16r(y.y), bf16r(y.z), bf16r(y.w));
        *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.Y) + o) = make_uint2(pk(y.x, y.y), pk(y.z, y.w));
      }
    }
    if (epi.ss_out) {
      if (ok && h)
        *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(epi.h_out) + o) =
            make_uint2(pk(y.x * hw4.x, y.y * hw4.y), pk(y.z * hw4.z, y.w * hw4.w));
      long long q = ok ? __float2ll_rn(y.x * y.x * kSsScale) + __float2ll_rn(y.y * y.y * kSsScale) +
                             __float2ll_rn(y.z * y.z * kSsScale) + __float2ll_rn(y.w * y.w * kSsScale)
                       : 0ll;
#pragma unroll
      for (int m = 4; m >= 1; m >>= 1)
        q += static_cast<long long>(__shfl_xor_sync(0xffffffffu, static_cast<unsigned long long>(q), m));
      if (g == 0) ss_acc[row] += q;
    }
  }
  __syncwarp();  // the staging tile is reused by the next chunk
}

__global__ void __launch_bounds__(kPairThreads, 1) gemm_pair_kernel(
    PairArgs a, const ds_skinny_epi epi, const __grid_constant__ CUtensorMap tx,
    const __grid_constant__ CUtensorMap tw) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // SW128 atoms
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * kStage);
  uint64_t* empty = full + a.stages;
  uint64_t* acc_full = empty + a.stages;  // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2] (the leader's are used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // per epilogue warp: a [32][kStgP] fp32 staging tile and 32 int64 row sums
  uint8_t* stg_base = smem + a.stages * kStage + 256;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // cluster = G CTA pairs; the pairs of a cluster work on adjacent weight
  // tiles of the SAME token tile, each CTA loading 1/G of the token rows for
  // all (multicast): the L2 -> SM token traffic drops by G
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1;             // rank in the pair
  const int gp = static_cast<int>(crank >> 1);  // pair in the cluster
  const bool leader = rank == 0;
  const uint32_t leader_rank = crank & ~1u;
  const uint16_t pair_mask = static_cast<uint16_t>(3u << (2 * gp));
  const uint16_t all_mask = static_cast<uint16_t>((1u << (2 * a.G)) - 1);
  const int grp = blockIdx.x / (2 * a.G), n_grp = gridDim.x / (2 * a.G);
  const int pair = grp * a.G + gp;  // global pair id (partial slots, flags)
  const int kt = a.kt;

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], a.G);  // every pair sharing the token stage releases it
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 16);  // 8 epilogue warps x 2 CTAs
    }
    mbar_fence_init();
  }
  if (warp == 1) alloc_pair(tmem_slot, 512);
  tc::fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in every CTA
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == 6) {
    // TMA producers: token boxes (warp 0, after the dependency wait) and weight
    // boxes (warp 6, the first ring round before it) from separate threads - a
    // thread issues one box per ~190 ns, two boxes per stage from one thread
    // would bound the stage rate below the pair's MMA rate (~280 ns per stage)
    if (lane == 0) {
      const bool is_w = warp == 6;
      tma_prefetch_desc(is_w ? &tw : &tx);
      const int ns_ = n_segs(a, grp);
      int it = 0;
      bool waited = false;
      const int xrows = kPM / a.G;  // token rows this CTA loads (for every pair)
      const uint16_t x_mask = static_cast<uint16_t>((1u << rank) | (1u << (2 + rank)));
      for (int q = 0; q < ns_; ++q) {
        const Seg g = seg_of(a, grp, n_grp, q);
        const int nt = (g.tile / a.n_tt) * a.G + gp, tt = g.tile % a.n_tt;
        const int rx = tt * 2 * kPM + static_cast<int>(rank) * kPM + gp * xrows;
        const int rw = nt * kPN + static_cast<int>(rank) * (kPN / 2);
        for (int k = g.kb; k < g.ke; ++k, ++it) {
          const int st = it % a.stages;
          if (it >= a.stages) mbar_wait(&empty[st], static_cast<uint32_t>((it / a.stages) - 1) & 1);
          uint8_t* sp = smem + st * kStage;
          if (is_w) {
            // the leader's barrier expects both CTAs' four boxes (a box may land
            // before this arrive: the tx count goes transiently negative)
            if (leader) mbar_expect_tx(&full[st], 2 * kStage);
            tma_load_3d_pair(sp + kBoxA, &tw, 0, rw, k, &full[st]);
          } else {
            if (!waited) {
              pdl_wait();  // the activations come from the previous kernel
              waited = true;
            }
            if (a.G > 1)
              tma_load_3d_pair_mc(sp + gp * xrows * 128, &tx, 0, rx, k, &full[st], x_mask);
            else
              tma_load_3d_pair(sp, &tx, 0, rx, k, &full[st]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader && lane == 0) {
      const uint32_t idesc = tc::idesc_bf16(2 * kPM, kPN, false);
      const uint32_t base = smem_u32(smem);
      const int ns_ = n_segs(a, grp);
      int n = 0;  // ring iteration
      for (int i = 0; i < ns_; ++i) {
        const Seg g = seg_of(a, grp, n_grp, i);
        const int acc = i & 1;
        if (i >= 2) mbar_wait(&acc_empty[acc], static_cast<uint32_t>((i >> 1) - 1) & 1);
        tc::fence_after();
        const uint32_t d = tmem + acc * kPN;
        for (int k = g.kb; k < g.ke; ++k, ++n) {
          const int st = n % a.stages;
          mbar_wait(&full[st], static_cast<uint32_t>(n / a.stages) & 1);
          tc::fence_after();
          const uint32_t pa = base + st * kStage, pb = pa + kBoxA;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_pair(d, tc::smem_desc(pa + kk * 32, 16, 1024), tc::smem_desc(pb + kk * 32, 16, 1024),
                     idesc, (k > g.kb || kk > 0) ? 1u : 0u);
          commit_pair(&empty[st], all_mask);  // every cluster CTA may refill the stage
        }
        commit_pair(&acc_full[acc], pair_mask);
      }
    }
    __syncwarp();
  } else if (warp >= 2 && warp != 6) {
    // ---- epilogue: thread = token row of this CTA, 32 features per load ----
    pdl_wait();  // the residual / previous contents of Y
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    // two warps per TMEM lane quadrant (warps 2-5, 7-10), alternate 32-feature
    // chunks: the epilogue's dependent loads (residual rows) run twice as wide
    const int half = warp >= 7;
    const int et = (warp - 2 - half) * 32 + lane;  // 0..255
    const int ew = et >> 5;                          // epilogue warp 0..7
    float* stg = reinterpret_cast<float*>(stg_base + ew * (32 * kStgP * 4 + 32 * 8));
    long long* ss_acc = reinterpret_cast<long long*>(stg + 32 * kStgP);
    const bool staged = !(epi.rope || epi.swiglu || epi.argmax_out);
    ss_acc[lane] = 0;
    __syncwarp();
    int* my_flag = a.flags + pair * 2 + rank;
    float* my_part = a.partials + (static_cast<int64_t>(pair) * 2 + rank) * kPM * kPN;
    const int ns_ = n_segs(a, grp);
    for (int i = 0; i < ns_; ++i) {
      const Seg g = seg_of(a, grp, n_grp, i);
      const int tile = g.tile;
      const bool finisher = g.j == 0;
      const int acc = i & 1;
      const int nt = (tile / a.n_tt) * a.G + gp, tt = tile % a.n_tt;
      const int t = tt * 2 * kPM + static_cast<int>(rank) * kPM + r;
      mbar_wait(&acc_full[acc], static_cast<uint32_t>(i >> 1) & 1);
      tc::fence_after();
      const uint32_t taddr = tmem + (static_cast<uint32_t>(quad * 32) << 16) + acc * kPN;
      if (!finisher) {
        // partial layout [chunk][float4 j][row]: a warp's store is 512 contiguous bytes
        float4* pr = reinterpret_cast<float4*>(my_part) + r;
#pragma unroll 1
        for (int c = half; c < kPN / 32; c += 2) {
          float v[32];
          tc::ld32(taddr + c * 32, v);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            __stcg(pr + (c * 8 + q) * kPM,
                   make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader)
            mbar_arrive(&acc_empty[acc]);
          else
            arrive_leader(&acc_empty[acc], leader_rank);
        }
        __threadfence();
        named_bar_sync(1, 256);
        if (et == 0) st_release_gpu(my_flag, 1);
        continue;
      }
      // participants: the same pair of the next groups, holding the tile's later
      // k ranges, in k order
      const int n_part = g.ke < a.kt ? a.split - 1 : 0;
      auto partner = [&](int d) { return (grp + 1 + d) * a.G + gp; };
      if (n_part > 0) {
        if (et < n_part)
          while (ld_acquire_gpu(a.flags + partner(et) * 2 + rank) == 0) __nanosleep(64);
        named_bar_sync(1, 256);
      }
      RowCtx rc{};
      rc.inv = 1.f;
      if (t < a.T) {
        if (epi.row_ss)
          rc.inv = rsqrtf(__ull2float_rn(__ldcg(reinterpret_cast<const unsigned long long*>(epi.row_ss) + t)) /
                              (kSsScale * static_cast<float>(a.K)) +
                          epi.eps);
        if (epi.rope) {
          rc.pos = __ldg(epi.row_pos + t);
          const int sq = __ldg(epi.row_seq + t);
          rc.cell = __ldg(epi.pos2cell + static_cast<int64_t>(sq) * epi.pos_stride + rc.pos);
        }
        if (epi.ss_zero && nt == 0 && !half) epi.ss_zero[t] = 0;
      }
#pragma unroll 1
      for (int c = half; c < kPN / 32; c += 2) {
        float v[32];
        tc::ld32(taddr + c * 32, v);
        for (int d = 0; d < n_part; ++d) {  // fixed k order: deterministic
          const float4* pq = reinterpret_cast<const float4*>(
                                 a.partials + (static_cast<int64_t>(partner(d)) * 2 + rank) * kPM * kPN) +
                             c * 8 * kPM + r;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 x = __ldcg(pq + j * kPM);
            v[4 * j] += x.x;
            v[4 * j + 1] += x.y;
            v[4 * j + 2] += x.z;
            v[4 * j + 3] += x.w;
          }
        }
        if (staged) {
          if (epi.row_ss) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= rc.inv;
          }
          pair_store_staged(v, a, epi, t - lane, nt * kPN + c * 32, stg, ss_acc, lane);
          continue;
        }
        if (t >= a.T) continue;
        pair_epilogue(v, a, epi, t, nt * kPN + c * 32, rc);
      }
      if (staged && epi.ss_out) {
        __syncwarp();
        rc.ssq = ss_acc[lane];
        ss_acc[lane] = 0;
      }
      if (t < a.T) {
        if (epi.ss_out)
          atomicAdd(reinterpret_cast<unsigned long long*>(epi.ss_out) + t,
                    static_cast<unsigned long long>(rc.ssq));
        if (epi.argmax_out) atomicMax(reinterpret_cast<unsigned long long*>(epi.argmax_out) + t, rc.amax);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&acc_empty[acc]);
        else
          arrive_leader(&acc_empty[acc], leader_rank);
      }
      if (n_part > 0) {  // re-arm the participants' flags (their partials are read)
        named_bar_sync(1, 256);
        if (et < n_part) a.flags[partner(et) * 2 + rank] = 0;
      }
    }
  }
  pdl_trigger();
  tc::fence_before();
  cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    tc::fence_after();
    dealloc_pair(tmem, 512);
  }
}
}  // namespace

}  // namespace ds

namespace ds {
// tail partials + flags for every pair the GPU holds: allocated once per
// device (outside any graph capture: the runtime reserves it at init), flags
// self re-arming
struct PairWorkspace {
  float* ws = nullptr;
  int* flags = nullptr;
  int pairs = 0;
  int device = -1;
};
PairWorkspace& pair_workspace() {
  static thread_local PairWorkspace w;
  int dev = 0;
  cudaGetDevice(&dev);
  if (w.device != dev) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int pairs = sms / 2 > 0 ? sms / 2 : 74;
    w = PairWorkspace{};
    if (cudaMalloc(&w.ws, static_cast<size_t>(pairs) * 2 * kPM * kPN * 4) == cudaSuccess &&
        cudaMalloc(&w.flags, static_cast<size_t>(pairs) * 2 * 4) == cudaSuccess &&
        cudaMemset(w.flags, 0, static_cast<size_t>(pairs) * 2 * 4) == cudaSuccess) {
      w.pairs = pairs;
      w.device = dev;
    } else {
      cudaGetLastError();
    }
  }
  return w;
}
void gemm_pair_reserve() { (void)pair_workspace(); }
}  // namespace ds

extern "C" int ds_gemm_pair(const void* X, const void* W, void* Y, int T, int N, int K, int y_f32,
                            int accumulate, const ds_skinny_epi* epi, ds_stream_t stream) {
  using namespace ds;
  if (T <= 0 || N % kPN || K % 64 || K < 64) return DS_EINVAL;
  ds_skinny_epi e{};
  if (epi) e = *epi;
  if ((e.swiglu && (y_f32 || accumulate)) || (e.rope && (y_f32 || accumulate)) ||
      (e.argmax_out && (!y_f32 || accumulate)) || (!Y && !e.argmax_out) ||
      (e.ss_out && !(y_f32 && accumulate)))
    return DS_EINVAL;
  if (e.rope && (e.n_heads <= 0 || e.n_kv_heads <= 0)) return DS_EINVAL;
  PairArgs a{};
  a.Y = Y;
  a.T = T;
  a.N = N;
  a.K = K;
  a.y_f32 = y_f32;
  a.accumulate = accumulate;
  a.n_tt = (T + 2 * kPM - 1) / (2 * kPM);
  a.kt = K / 64;
  // DS_PAIR_MC=1 (A/B): two pairs per cluster sharing the token tile through
  // multicast when the weight tiles pair up (N % 512).  Correct, but measured
  // slower (T=4096 gate_up 674 vs 649 us, down 345-358 vs 336): one pair per
  // cluster by default
  static const int mc_env = getenv("DS_PAIR_MC") ? atoi(getenv("DS_PAIR_MC")) : 0;
  a.G = (mc_env && N % (2 * kPN) == 0) ? 2 : 1;
  a.tiles = (N / (kPN * a.G)) * a.n_tt;  // cluster tiles
  static const int st_env = getenv("DS_PAIR_STAGES") ? atoi(getenv("DS_PAIR_STAGES")) : 0;
  const int fixed = 1024 + 256 + 8 * (32 * kStgP * 4 + 32 * 8);  // + epilogue staging
  int ns = (kPairSmemMax - fixed) / kStage;
  if (st_env > 1 && st_env < ns) ns = st_env;
  a.stages = ns;
  const int smem = fixed + ns * kStage;
  const CUtensorMap* tx = slab_tensor_map(X, T, K, kPM / a.G, 1);
  const CUtensorMap* tw = slab_tensor_map(W, N, K, kPN / 2, 1);
  if (!tx || !tw) return DS_EUNSUPPORTED;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmemMax);
    cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  // every cluster must be co-resident (the tail's partial hand-off spins)
  static int max_cl[3] = {0, 0, 0};
  if (!max_cl[a.G]) {
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(2 * a.G, 1, 1);
    q.blockDim = dim3(kPairThreads);
    q.dynamicSmemBytes = smem;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = 2 * a.G;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_pair_kernel, &q) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      int sms = 0, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      n = sms / (2 * a.G);
    }
    max_cl[a.G] = n;
  }
  static const int pairs_env = getenv("DS_PAIR_CTAS") ? atoi(getenv("DS_PAIR_CTAS")) / 2 : 0;
  int groups = max_cl[a.G];
  if (pairs_env > 0 && pairs_env / a.G < groups) groups = pairs_env / a.G;
  if (groups > a.tiles * 4) groups = a.tiles * 4;
  // full waves data-parallel; the tail tiles (< groups) cut into up to 4 k ranges
  a.full_waves = a.tiles / groups;
  a.rem = a.tiles - a.full_waves * groups;
  static const int split_max = getenv("DS_PAIR_SPLIT") ? atoi(getenv("DS_PAIR_SPLIT")) : 4;
  a.split = 1;
  if (a.rem) {
    a.split = groups / a.rem;
    if (a.split > split_max) a.split = split_max;
    if (a.split > a.kt) a.split = a.kt;
    if (a.split < 1) a.split = 1;
  }
  if (a.full_waves == 0) groups = a.rem * a.split;  // only the tail: idle clusters not launched
  const int pairs = groups * a.G;
  PairWorkspace& w = pair_workspace();
  if (!w.ws || pairs > w.pairs) return DS_EWORKSPACE;
  a.partials = w.ws;
  a.flags = w.flags;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs, 1, 1);  // groups x G pairs x 2 CTAs
  cfg.blockDim = dim3(kPairThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr2[2];
  attr2[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr2[0].val.programmaticStreamSerializationAllowed = 1;
  attr2[1].id = cudaLaunchAttributeClusterDimension;
  attr2[1].val.clusterDim.x = 2 * a.G;
  attr2[1].val.clusterDim.y = 1;
  attr2[1].val.clusterDim.z = 1;
  cfg.attrs = attr2;
  cfg.numAttrs = 2;
  cudaError_t err = cudaLaunchKernelEx(&cfg, gemm_pair_kernel, a, e, *tx, *tw);
  if (err != cudaSuccess) return static_cast<int>(err);
  return static_cast<int>(cudaGetLastError());
}
