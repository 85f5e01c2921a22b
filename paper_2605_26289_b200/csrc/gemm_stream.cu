// K10: projection GEMM for prefill chunks and batched plans (33..16k rows) on
// the 5th-generation tensor cores, with the forward's elementwise work fused
// into the epilogue:  Y[T][N] (+)= X[T][K] . W[N][K]^T.
//
// Replaces the library GEMM on every M > 32 projection of the forward (the
// reference executes plan entries serially through a mock engine,
// scheduler.py:652-660; the B200 forward runs a whole plan as one varlen
// pass with M = sum of rows).
//
// Tiling: a tile is 128 weight rows (UMMA M) x NT tokens (UMMA N = every
// token of a chunk up to 256, so a weight byte is read once per 256 tokens)
// x all of K, in 64-column k-iterations (one SWIZZLE_128B slab of each
// operand per TMA box).  Tiles are ordered weight-tile-major with the token
// tiles of one weight tile adjacent (their second weight read hits L2).
//
// Schedule: persistent stream-K.  One CTA per SM; CTA c owns the contiguous
// k-iteration range [c*W/P, (c+1)*W/P) of the W = tiles * K/64 iterations, so
// every SM gets the same work whatever the shape (48 qkv tiles or 1002 LM-head
// tiles on 148 SMs - no wave quantisation).  A tile cut by a range boundary
// is finished by the CTA holding its FIRST k-iteration (the "head", which
// reaches it at the end of its range); the others write fp32 partials to a
// global workspace at the start of theirs and bump the tile's arrival count.
// The head adds the partials in k order (deterministic) and re-arms the
// counter.  Dependencies only point from a CTA's last tile to later CTAs'
// first tiles, so there is no cycle; all CTAs are co-resident.
//
// Warp roles (192 threads):
//   warp 0   TMA producer: per k-iteration one box of the 128 weight rows and
//            one box of the NT token rows (token rows past T zero-filled)
//            into an mbarrier ring; the first round of weight boxes is issued
//            before the programmatic-dependency wait;
//   warp 1   TMEM allocation (2 x 256 columns) and the single-thread MMA issue:
//            4 x tcgen05.mma kind::f16 (K=16) per iteration, stage release
//            and the accumulator hand-off through tcgen05.commit;
//   warps 2-5 epilogue, thread = weight row: tcgen05.ld of the accumulator
//            (double-buffered, so tile i's epilogue overlaps tile i+1's
//            main loop), then the fused ds_skinny_epi work, same semantics as
//            the decode GEMM (gemm_skinny.cu):
//            * norm consumer: rows scaled by rsqrt(row_ss/K + eps);
//            * residual producer: x += acc (fp32), h = bf16(x * w_norm), row
//              sums of x^2 in 2^-24 fixed point (integer atomics, each
//              element converted separately - bit-identical in any order);
//            * SwiGLU: gate/up rows 16b+j / 16b+j+8 are lanes l / l^8;
//            * RoPE + KV store: pair dims i / i+64 are lanes l / l^8; q to Y,
//              k / v straight into the paged pools at pos2cell;
//            * LM-head argmax: packed (value, lowest column) keys reduced per
//              token across the tile, one global atomicMax per token and tile.
#include "../../include/deltaserve_b200.h"
#include "common.cuh"
#include "tc.cuh"
#include "tma.h"

#include <cstdio>
#include <cstdlib>
#include <mutex>

namespace ds {

namespace {
constexpr int kBM = 128;
constexpr int kSlabA = kBM * 128;  // 16 KB: 128 weight rows x 64 columns
constexpr int kThreads = 10 * 32;  // producer, MMA, 8 epilogue warps
constexpr int kEpiThreads = 8 * 32;
constexpr int kMaxNT = 256;
constexpr int kAccCols = 256;
constexpr int kSmemMax = 227 * 1024;
// s_inv, s_pos, s_cell, s_amax + the epilogue warps' staging tiles
constexpr int kScalarBytes = kMaxNT * (4 + 4 + 8 + 8) + 8 * 32 * 36 * 4;
constexpr int kMaxFlags = 1 << 16;
// one CTA partial tile: [kMaxNT/32 chunks][kBM rows][36] fp32 (2 slots per CTA)
constexpr int64_t kSlotFloats = static_cast<int64_t>(kMaxNT / 32) * kBM * 36;
constexpr float kSsScale = 16777216.f;  // 2^24 fixed point (as the decode GEMM)

struct StreamArgs {
  void* Y;
  const __nv_bfloat16* h_w;
  float* partials;  // [n_ctas][kBM rows][NT + 4] fp32 (slot stride kSlotFloats)
  int* flags;       // [tiles] arrival counts (self re-arming)
  int64_t total;    // tiles * kt
  int T, N, K, y_f32, accumulate;
  int NT, n_tt, kt, stages;
  unsigned long long* trace;  // DS_STREAM_TRACE: per-CTA globaltimer stamps [P][16]
};

DS_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
  return t;
}

DS_DEVICE float bf16r_(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

DS_DEVICE int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// first iteration of CTA c's range
__host__ __device__ __forceinline__ int64_t range_begin(int64_t total, int P, int c) {
  return total * c / P;
}
// the CTA whose range holds iteration it
DS_DEVICE int cta_of(int64_t total, int P, int64_t it) {
  int g = static_cast<int>((it * P) / total);
  while (g + 1 < P && range_begin(total, P, g + 1) <= it) ++g;
  while (g > 0 && range_begin(total, P, g) > it) --g;
  return g;
}

DS_DEVICE unsigned long long shfl_xor_u64(unsigned long long v, int m) {
  const uint32_t lo = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(v), m);
  const uint32_t hi = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), m);
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}

// ---- the fused epilogue of 32 consecutive token columns of one tile ----
// v[j]: accumulator of weight row r (feature f) and tile-local token c0 + j,
// one thread per row.  Values are finished in that layout (the lane ^ 8
// partner exchanges of SwiGLU / RoPE are warp shuffles), then each warp
// transposes its 32 rows x 32 tokens through a private shared-memory tile
// (stg, row stride kStg floats) and writes whole token-row segments with
// vector stores: 8 lanes per token row, 4 token rows per instruction (per
// thread-per-row scalar stores were measured 5x slower).  Validity depends
// on the token only, so it is warp-uniform.
constexpr int kStg = 36;  // staging row stride (floats): 16-byte aligned, conflict-free

DS_DEVICE void stg_put(float* stg, int lane, const float* v) {
#pragma unroll
  for (int j = 0; j < 32; ++j) stg[j * kStg + lane] = v[j];
  __syncwarp();
}

// store the staged [32 tokens][width] tile: dst(j) = destination row of token
// j (nullptr: skip), `width` features (multiple of 4, <= 32) from column col0
template <typename OutT, typename Dst>
DS_DEVICE void stg_store(const float* stg, int lane, int n_valid, int col0, int width, Dst dst) {
  const int g = lane & 7, rr = lane >> 3;
  if (4 * g >= width) return;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = rr + 4 * i;
    if (j >= n_valid) break;
    OutT* d = dst(j);
    if (!d) continue;
    const float4 x = *reinterpret_cast<const float4*>(stg + j * kStg + col0 + 4 * g);
    if constexpr (sizeof(OutT) == 4) {
      *reinterpret_cast<float4*>(d + 4 * g) = x;
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(d + 4 * g) = u;
    }
  }
}

DS_DEVICE void epilogue_chunk(float* v, const StreamArgs& a, const ds_skinny_epi& epi, int wt,
                              int t0, int c0, int r, const float* s_inv, const int* s_pos,
                              const int64_t* s_cell, unsigned long long* s_amax,
                              const __nv_bfloat16* hw_row, float* stg) {
  const int f = wt * kBM + r;
  const int lane = r & 31;
  const int fw = wt * kBM + (r & ~31);  // first feature of this warp's 32 rows
  const int n_valid = min(32, min(a.NT - c0, a.T - t0 - c0));
  if (n_valid <= 0) return;
  const int tb = t0 + c0;  // first token of the chunk
  if (epi.row_ss) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] *= s_inv[c0 + j];
  }
  if (epi.rope) {
    constexpr int kHd = 128, kHalf = 64;
    const int qk_width = (epi.n_heads + epi.n_kv_heads) * kHd;
    __nv_bfloat16* kp = static_cast<__nv_bfloat16*>(epi.k_pool_l);
    __nv_bfloat16* vp = static_cast<__nv_bfloat16*>(epi.v_pool_l);
    if (wt * kBM < qk_width) {  // a q or k head (one head per 128-row tile)
      // warp q of the head holds dims [16q, 16q+16) (lanes l & 8 == 0) and
      // [64+16q, 64+16q+16) (lanes l & 8 != 0); staged as [token][32 slots]
      const int head = wt, jj = r & 15, i = 8 * (r >> 4) + (jj & 7);
      const bool lo = jj < 8;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x = bf16r_(v[j]);  // the unfused path stores qkv in bf16
        const float p = __shfl_xor_sync(0xffffffffu, x, 8);
        const int tk = min(c0 + j, kMaxNT - 1);
        const int64_t tp = static_cast<int64_t>(s_pos[tk]) * kHalf + i;
        const float c = j < n_valid ? __ldg(epi.rope_cos + tp) : 0.f;
        const float sn = j < n_valid ? __ldg(epi.rope_sin + tp) : 0.f;
        v[j] = lo ? x * c - p * sn : x * c + p * sn;
      }
      // slot of this lane: lo lanes -> [0,16), hi lanes -> [16,32)
      const int slot = (lo ? 0 : 16) + (i & 15);
#pragma unroll
      for (int j = 0; j < 32; ++j) stg[j * kStg + slot] = v[j];
      __syncwarp();
      const int d0 = i & ~15;  // 16 * (warp within the head)
      auto row = [&](int j) -> __nv_bfloat16* {
        return head < epi.n_heads
                   ? static_cast<__nv_bfloat16*>(a.Y) + static_cast<int64_t>(tb + j) * a.N +
                         head * kHd
                   : kp + ((head - epi.n_heads) * epi.kv_head_stride + s_cell[c0 + j]) * kHd;
      };
      stg_store<__nv_bfloat16>(stg, lane, n_valid, 0, 16, [&](int j) { return row(j) + d0; });
      stg_store<__nv_bfloat16>(stg, lane, n_valid, 16, 16,
                               [&](int j) { return row(j) + kHalf + d0; });
      return;
    }
    // v rows: the warp's 32 rows are 32 consecutive dims of one kv head
    stg_put(stg, lane, v);
    const int fv0 = fw - qk_width;
    __nv_bfloat16* base = vp + (fv0 / kHd) * epi.kv_head_stride * kHd + fv0 % kHd;
    stg_store<__nv_bfloat16>(stg, lane, n_valid, 0, 32, [&](int j) {
      return base + s_cell[c0 + j] * kHd;
    });
    return;
  }
  if (epi.swiglu) {  // lanes l (gate, l & 8 == 0) and l ^ 8 (up) of the same FFN unit
    const bool gate = (r & 8) == 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float u = __shfl_xor_sync(0xffffffffu, v[j], 8);
      const float gg = bf16r_(v[j]), uu = bf16r_(u);  // the unfused path stores gate|up in bf16
      v[j] = gg / (1.f + expf(-gg)) * uu;
    }
    // the warp's 16 units: gate lanes 0-7 -> units 0-7, 16-23 -> 8-15
    if (gate) {
      const int ul = (lane >> 4) * 8 + (lane & 7);
#pragma unroll
      for (int j = 0; j < 32; ++j) stg[j * kStg + ul] = v[j];
    }
    __syncwarp();
    const int u0 = fw / 2;
    __nv_bfloat16* y = static_cast<__nv_bfloat16*>(a.Y);
    const int64_t stride = a.N / 2;
    stg_store<__nv_bfloat16>(stg, lane, n_valid, 0, 16, [&](int j) {
      return y + static_cast<int64_t>(tb + j) * stride + u0;
    });
    return;
  }
  if (epi.argmax_out) {  // LM head
    if (a.Y) {
      stg_put(stg, lane, v);
      float* y = static_cast<float*>(a.Y);
      stg_store<float>(stg, lane, n_valid, 0, 32, [&](int j) {
        return y + static_cast<int64_t>(tb + j) * a.N + fw;
      });
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j >= n_valid) break;  // warp-uniform
      unsigned long long k = argmax_key(v[j], f);
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) {
        const unsigned long long o = shfl_xor_u64(k, m);
        k = o > k ? o : k;
      }
      if (lane == 0) atomicMax(&s_amax[c0 + j], k);
    }
    return;
  }
  // plain / residual: stage the chunk, then each lane owns 4 features x 8
  // token rows: old values (accumulate) loaded as vectors, stored as vectors
  stg_put(stg, lane, v);
  const int g = lane & 7, rr = lane >> 3;
  float4 w4 = make_float4(0.f, 0.f, 0.f, 0.f);
  if (epi.ss_out && epi.h_out && hw_row) {
    const uint2 hu = *reinterpret_cast<const uint2*>(hw_row + fw + 4 * g);
    const float2 h0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hu.x));
    const float2 h1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hu.y));
    w4 = make_float4(h0.x, h0.y, h1.x, h1.y);
  }
  float4 y4[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = rr + 4 * i;
    y4[i] = *reinterpret_cast<const float4*>(stg + j * kStg + 4 * g);
  }
  if (a.accumulate) {  // every old value in flight before the first use
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = rr + 4 * i;
      if (j >= n_valid) break;
      const int64_t o = static_cast<int64_t>(tb + j) * a.N + fw + 4 * g;
      float4 old;
      if (a.y_f32) {
        old = *reinterpret_cast<const float4*>(static_cast<const float*>(a.Y) + o);
      } else {
        const uint2 u = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(a.Y) + o);
        const float2 p0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 p1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        old = make_float4(p0.x, p0.y, p1.x, p1.y);
      }
      y4[i].x += old.x;
      y4[i].y += old.y;
      y4[i].z += old.z;
      y4[i].w += old.w;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = rr + 4 * i;
    const bool ok = j < n_valid;
    const int64_t o = static_cast<int64_t>(tb + j) * a.N + fw + 4 * g;
    float4 y = y4[i];
    if (ok) {
      if (a.y_f32) {
        *reinterpret_cast<float4*>(static_cast<float*>(a.Y) + o) = y;
      } else {
        __nv_bfloat162 lo = __floats2bfloat162_rn(y.x, y.y), hi = __floats2bfloat162_rn(y.z, y.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.Y) + o) = u;
        const float2 r0 = __bfloat1622float2(lo), r1 = __bfloat1622float2(hi);
        y = make_float4(r0.x, r0.y, r1.x, r1.y);
      }
    }
    if (epi.ss_out) {  // residual producer: next RMSNorm's weight multiply + row sums
      if (ok && epi.h_out) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(y.x * w4.x, y.y * w4.y);
        __nv_bfloat162 hi = __floats2bfloat162_rn(y.z * w4.z, y.w * w4.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(epi.h_out) + o) = u;
      }
      // 2^-24 fixed point per element: the integer sum is order independent
      long long q = ok ? __float2ll_rn(y.x * y.x * kSsScale) + __float2ll_rn(y.y * y.y * kSsScale) +
                             __float2ll_rn(y.z * y.z * kSsScale) + __float2ll_rn(y.w * y.w * kSsScale)
                       : 0ll;
#pragma unroll
      for (int m = 4; m >= 1; m >>= 1) q += static_cast<long long>(shfl_xor_u64(q, m));
      if (ok && g == 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(epi.ss_out) + tb + j,
                  static_cast<unsigned long long>(q));
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) gemm_stream_kernel(
    StreamArgs a, ds_skinny_epi epi, const __grid_constant__ CUtensorMap tw,
    const __grid_constant__ CUtensorMap tx) {
  extern __shared__ uint8_t smem_raw[];
  if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 16] = gtimer();
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // SW128 atoms
  const int stage_bytes = kSlabA + a.NT * 128;
  uint8_t* tail = smem + a.stages * stage_bytes;
  float* s_inv = reinterpret_cast<float*>(tail);
  int* s_pos = reinterpret_cast<int*>(s_inv + kMaxNT);
  int64_t* s_cell = reinterpret_cast<int64_t*>(s_pos + kMaxNT);
  unsigned long long* s_amax = reinterpret_cast<unsigned long long*>(s_cell + kMaxNT);
  float* stg_all = reinterpret_cast<float*>(s_amax + kMaxNT);  // [8 warps][32][kStg]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg_all + 8 * 32 * kStg);
  uint64_t* empty = full + a.stages;
  uint64_t* acc_full = empty + a.stages;  // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint64_t* red_bar = acc_empty + 2;      // [2] partial-chunk bulk copies (finalize, per half)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_bar + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = gridDim.x, cta = blockIdx.x;
  const int64_t it_b = range_begin(a.total, P, cta), it_e = range_begin(a.total, P, cta + 1);
  const int kt = a.kt;

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 8);  // one arrive per epilogue warp
      mbar_init(&red_bar[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) tc::alloc(tmem_slot, 2 * kAccCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  unsigned long long* tr = a.trace ? a.trace + cta * 16 : nullptr;
  if (tr && threadIdx.x == 0) tr[1] = gtimer();

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tw);
      tma_prefetch_desc(&tx);
      const int64_t n = it_e - it_b;
      const int pre = static_cast<int>(n < a.stages ? n : a.stages);
      for (int i = 0; i < pre; ++i) {
        const int64_t it = it_b + i;
        const int tile = static_cast<int>(it / kt), kk = static_cast<int>(it % kt);
        mbar_expect_tx(&full[i], stage_bytes);
        tma_load_3d(smem + i * stage_bytes, &tw, 0, (tile / a.n_tt) * kBM, kk, &full[i]);
      }
      pdl_wait();  // the activations come from the previous kernel
      for (int i = 0; i < pre; ++i) {
        const int64_t it = it_b + i;
        const int tile = static_cast<int>(it / kt), kk = static_cast<int>(it % kt);
        tma_load_3d(smem + i * stage_bytes + kSlabA, &tx, 0, (tile % a.n_tt) * a.NT, kk,
                    &full[i]);
      }
      for (int64_t i = pre; i < n; ++i) {
        const int st = static_cast<int>(i % a.stages);
        mbar_wait(&empty[st], static_cast<uint32_t>((i / a.stages) - 1) & 1);
        const int64_t it = it_b + i;
        const int tile = static_cast<int>(it / kt), kk = static_cast<int>(it % kt);
        uint8_t* sp = smem + st * stage_bytes;
        mbar_expect_tx(&full[st], stage_bytes);
        tma_load_3d(sp, &tw, 0, (tile / a.n_tt) * kBM, kk, &full[st]);
        tma_load_3d(sp + kSlabA, &tx, 0, (tile % a.n_tt) * a.NT, kk, &full[st]);
      }
      if (tr) tr[2] = gtimer();
    }
    __syncwarp();  // reconverge before the CTA barrier (bar.sync is warp-aligned)
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_bf16(kBM, a.NT, false);
      const uint32_t base = smem_u32(smem);
      int64_t i = 0;
      int seg = 0;
      for (int64_t it = it_b; it < it_e; ++seg) {
        const int tile = static_cast<int>(it / kt);
        const int64_t seg_end = min(it_e, static_cast<int64_t>(tile + 1) * kt);
        const int acc = seg & 1;
        if (seg >= 2) mbar_wait(&acc_empty[acc], static_cast<uint32_t>((seg >> 1) - 1) & 1);
        tc::fence_after();
        const uint32_t d = tmem + acc * kAccCols;
        for (const int64_t s0 = it; it < seg_end; ++it, ++i) {
          const int st = static_cast<int>(i % a.stages);
          mbar_wait(&full[st], static_cast<uint32_t>(i / a.stages) & 1);
          tc::fence_after();
          const uint32_t pa = base + st * stage_bytes, pb = pa + kSlabA;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc::mma(d, tc::smem_desc(pa + k * 32, 16, 1024), tc::smem_desc(pb + k * 32, 16, 1024),
                    idesc, (it != s0 || k > 0) ? 1u : 0u);
          tc::commit(&empty[st]);  // the stage is free once its MMAs completed
        }
        tc::commit(&acc_full[acc]);
      }
      if (tr) tr[3] = gtimer();
    }
    __syncwarp();
  } else {
    // ---- epilogue warps 2-9: TMEM lane quadrant (warp & 3), thread = weight
    // row; the two halves (warps 2-5, 6-9) take alternate 32-column chunks ----
    pdl_wait();  // row scalars / the residual come from the previous kernel
    const int quad = warp & 3, r = quad * 32 + lane;
    const int half = (warp - 2) >> 2;
    const int et = threadIdx.x - 64;          // 0..255
    const int ht = et & 127;                  // thread within the half
    float* stg = stg_all + (warp - 2) * 32 * kStg;
    const int ncols = (a.NT + 31) & ~31, nch = ncols / 32;
    // per-token scalars of one chunk (computed by 32 threads of the half)
    auto chunk_scalars = [&](int wt, int t0, int c0) {
      if (ht < 32) {
        const int tk = c0 + ht, t = t0 + tk;
        s_amax[tk] = 0;
        if (tk < a.NT && t < a.T) {
          if (epi.row_ss) {
            const unsigned long long rs =
                __ldcg(reinterpret_cast<const unsigned long long*>(epi.row_ss) + t);
            s_inv[tk] =
                rsqrtf(__ull2float_rn(rs) / (kSsScale * static_cast<float>(a.K)) + epi.eps);
          }
          if (epi.rope) {
            const int r_pos = __ldg(epi.row_pos + t), r_seq = __ldg(epi.row_seq + t);
            s_pos[tk] = r_pos;
            s_cell[tk] =
                __ldg(epi.pos2cell + static_cast<int64_t>(r_seq) * epi.pos_stride + r_pos);
          }
          if (epi.ss_zero && wt == 0) epi.ss_zero[t] = 0;
        }
      }
      named_bar_sync(2 + half, 128);
    };
    auto chunk_flush_argmax = [&](int t0, int c0) {
      if (!epi.argmax_out) return;
      named_bar_sync(2 + half, 128);
      if (ht < 32 && c0 + ht < a.NT && t0 + c0 + ht < a.T)
        atomicMax(reinterpret_cast<unsigned long long*>(epi.argmax_out) + t0 + c0 + ht,
                  s_amax[c0 + ht]);
    };
    int cut_tile[2] = {-1, -1};  // tiles this CTA shares with others (first / last segment)
    int seg = 0;
    for (int64_t it = it_b; it < it_e; ++seg) {
      const int tile = static_cast<int>(it / kt);
      const int64_t k0 = static_cast<int64_t>(tile) * kt;
      const int64_t seg_end = min(it_e, k0 + kt);
      const bool cut = !(it == k0 && seg_end == k0 + kt);
      it = seg_end;
      const int wt = tile / a.n_tt, t0 = (tile % a.n_tt) * a.NT;
      const int acc = seg & 1;
      const uint32_t taddr = tmem + (static_cast<uint32_t>(quad * 32) << 16) + acc * kAccCols;
      mbar_wait(&acc_full[acc], static_cast<uint32_t>(seg >> 1) & 1);
      tc::fence_after();
      if (cut) {
        // partial tile -> this CTA's slot (first segment: slot 0, last: slot 1),
        // chunk-major [chunk][128 rows][kStg]: one chunk of one participant
        // is a contiguous 18 KB block for the finalizing CTA's bulk copy
        const int slot = seg == 0 ? 0 : 1;
        float* part = a.partials + (static_cast<int64_t>(cta) * 2 + slot) * kSlotFloats;
        for (int c = half; c < nch; c += 2) {
          float v[32];
          tc::ld32(taddr + c * 32, v);
          float4* pr = reinterpret_cast<float4*>(part + (c * kBM + r) * kStg);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            __stcg(pr + k, make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[acc]);
        __threadfence();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) atomicAdd(a.flags + tile, 1);
        cut_tile[slot] = tile;
        if (tr && et == 0) tr[4] = gtimer();
        continue;
      }
      // a whole tile: epilogue straight from TMEM (overlaps the next tile's MMAs)
      for (int c = half; c < nch; c += 2) {
        chunk_scalars(wt, t0, c * 32);
        float v[32];
        tc::ld32(taddr + c * 32, v);
        epilogue_chunk(v, a, epi, wt, t0, c * 32, r, s_inv, s_pos, s_cell, s_amax, a.h_w, stg);
        chunk_flush_argmax(t0, c * 32);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
    // ---- finalize the shared tiles: every participant reduces and finishes
    // its share of the chunks (chunk c -> participant c mod S), adding the S
    // partials in k order (deterministic) from shared memory (the ring is idle
    // now: every MMA of this CTA has completed) ----
    const int64_t ring_bytes = static_cast<int64_t>(a.stages) * stage_bytes;
    const uint32_t pc_bytes = kBM * kStg * 4;  // one participant's chunk
    const int fit = static_cast<int>((ring_bytes / 2) / pc_bytes);  // per half
    uint8_t* hring = smem + half * (ring_bytes / 2);
    int phase = 0;
    for (int w = 0; w < 2; ++w) {
      const int tile = cut_tile[w];
      if (tile < 0 || (w == 1 && tile == cut_tile[0])) continue;
      const int64_t k0 = static_cast<int64_t>(tile) * kt;
      const int c_first = cta_of(a.total, P, k0), c_last = cta_of(a.total, P, k0 + kt - 1);
      const int S = c_last - c_first + 1, me = cta - c_first;
      const int wt = tile / a.n_tt, t0 = (tile % a.n_tt) * a.NT;
      if (tr && et == 0) tr[5] = gtimer();
      if (et == 0)
        while (ld_acquire(a.flags + tile) < S) __nanosleep(32);
      named_bar_sync(1, kEpiThreads);
      if (tr && et == 0) tr[6] = gtimer();
      int k_mine = 0;
      for (int c = me; c < nch; c += S, ++k_mine) {
        if ((k_mine & 1) != half) continue;
        chunk_scalars(wt, t0, c * 32);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
        for (int q0 = 0; q0 < S; q0 += fit) {
          const int nq = min(fit, S - q0);
          named_bar_sync(2 + half, 128);  // the previous batch is consumed
          if (ht == 0) {
            tc::fence_proxy_async();
            mbar_expect_tx(&red_bar[half], nq * pc_bytes);
            for (int q = 0; q < nq; ++q) {
              const int pc = c_first + q0 + q;
              // slot 0 if the tile is pc's first segment, else its last (slot 1)
              const int slot = range_begin(a.total, P, pc) / kt == tile ? 0 : 1;
              bulk_g2s(hring + q * pc_bytes,
                       a.partials + (static_cast<int64_t>(pc) * 2 + slot) * kSlotFloats +
                           static_cast<int64_t>(c) * kBM * kStg,
                       pc_bytes, &red_bar[half]);
            }
          }
          mbar_wait(&red_bar[half], static_cast<uint32_t>(phase) & 1);
          ++phase;
          for (int q = 0; q < nq; ++q) {
            const float4* pq =
                reinterpret_cast<const float4*>(hring + q * pc_bytes) + (r * kStg) / 4;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float4 x = pq[k];
              v[4 * k] += x.x;
              v[4 * k + 1] += x.y;
              v[4 * k + 2] += x.z;
              v[4 * k + 3] += x.w;
            }
          }
        }
        epilogue_chunk(v, a, epi, wt, t0, c * 32, r, s_inv, s_pos, s_cell, s_amax, a.h_w, stg);
        chunk_flush_argmax(t0, c * 32);
      }
      named_bar_sync(1, kEpiThreads);  // this CTA's reads of the tile's partials are done
      if (et == 0 && atomicAdd(a.flags + tile, 1) == 2 * S - 1) a.flags[tile] = 0;  // re-arm
      if (tr && et == 0) tr[10] = gtimer();
    }
  }
  tc::fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) {
    __threadfence();
    tr[7] = gtimer();
  }
  if (warp == 1) {
    tc::fence_after();
    tc::dealloc(tmem, 2 * kAccCols);
  }
}

// ---- token-row epilogue (cluster mode): one warp = one token row of the
// tile's 128 features, lane l = features 4l..4l+3 - every global access is a
// contiguous 8- or 16-byte piece of a 256 / 512-byte row segment; the
// gate/up and RoPE-pair partners (features f, f ^ 8) are lanes l, l ^ 2 ----
DS_DEVICE void epilogue_tokrow(float4 y, const StreamArgs& a, const ds_skinny_epi& epi, int wt,
                               int tk, int lane, const float* s_inv, const int* s_pos,
                               const int64_t* s_cell) {
  const int fl = 4 * lane, f = wt * kBM + fl;
  const int t = tk;  // cluster mode: one token tile, t0 = 0
  float v[4] = {y.x, y.y, y.z, y.w};
  if (epi.row_ss) {
    const float sc = s_inv[tk];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] *= sc;
  }
  auto st_bf4 = [](__nv_bfloat16* d, float a0, float a1, float a2, float a3) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(a0, a1), hi = __floats2bfloat162_rn(a2, a3);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(d) = u;
  };
  if (epi.rope) {
    constexpr int kHd = 128, kHalf = 64;
    const int qk_width = (epi.n_heads + epi.n_kv_heads) * kHd;
    if (wt * kBM < qk_width) {
      const int head = wt, c = fl;  // features within the head
      const bool lo = (c & 15) < 8;
      const int i0 = 8 * (c >> 4) + (c & 7);  // dims i0..i0+3 (or +64)
      float x[4], p[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        x[k] = bf16r_(v[k]);  // the unfused path stores qkv in bf16
        p[k] = __shfl_xor_sync(0xffffffffu, x[k], 2);
      }
      const int64_t tp = static_cast<int64_t>(s_pos[tk]) * kHalf + i0;
      const float4 cs = *reinterpret_cast<const float4*>(epi.rope_cos + tp);
      const float4 sn = *reinterpret_cast<const float4*>(epi.rope_sin + tp);
      const float cc[4] = {cs.x, cs.y, cs.z, cs.w}, ss[4] = {sn.x, sn.y, sn.z, sn.w};
      float o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = lo ? x[k] * cc[k] - p[k] * ss[k] : x[k] * cc[k] + p[k] * ss[k];
      __nv_bfloat16* row =
          head < epi.n_heads
              ? static_cast<__nv_bfloat16*>(a.Y) + static_cast<int64_t>(t) * a.N + head * kHd
              : static_cast<__nv_bfloat16*>(epi.k_pool_l) +
                    ((head - epi.n_heads) * epi.kv_head_stride + s_cell[tk]) * kHd;
      st_bf4(row + (lo ? i0 : i0 + kHalf), o[0], o[1], o[2], o[3]);
    } else {
      const int fv = f - qk_width;
      __nv_bfloat16* d = static_cast<__nv_bfloat16*>(epi.v_pool_l) +
                         ((fv / kHd) * epi.kv_head_stride + s_cell[tk]) * kHd + fv % kHd;
      st_bf4(d, v[0], v[1], v[2], v[3]);
    }
    return;
  }
  if (epi.swiglu) {
    float u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = __shfl_xor_sync(0xffffffffu, v[k], 2);
    if ((fl & 15) >= 8) return;  // up lanes
    float o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float gg = bf16r_(v[k]), uu = bf16r_(u[k]);  // the unfused path stores gate|up in bf16
      o[k] = gg / (1.f + expf(-gg)) * uu;
    }
    const int unit = wt * (kBM / 2) + (fl >> 4) * 8 + (fl & 7);
    st_bf4(static_cast<__nv_bfloat16*>(a.Y) + static_cast<int64_t>(t) * (a.N / 2) + unit, o[0],
           o[1], o[2], o[3]);
    return;
  }
  const int64_t off = static_cast<int64_t>(t) * a.N + f;
  if (epi.argmax_out) {
    if (a.Y) *reinterpret_cast<float4*>(static_cast<float*>(a.Y) + off) = make_float4(v[0], v[1], v[2], v[3]);
    unsigned long long k = argmax_key(v[0], f);
#pragma unroll
    for (int q = 1; q < 4; ++q) {
      const unsigned long long kq = argmax_key(v[q], f + q);
      k = kq > k ? kq : k;
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      const unsigned long long o = shfl_xor_u64(k, m);
      k = o > k ? o : k;
    }
    if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(epi.argmax_out) + t, k);
    return;
  }
  if (a.y_f32) {
    float* yp = static_cast<float*>(a.Y) + off;
    if (a.accumulate) {
      const float4 old = *reinterpret_cast<const float4*>(yp);
      v[0] += old.x;
      v[1] += old.y;
      v[2] += old.z;
      v[3] += old.w;
    }
    *reinterpret_cast<float4*>(yp) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    __nv_bfloat16* yp = static_cast<__nv_bfloat16*>(a.Y) + off;
    if (a.accumulate) {
      const uint2 uo = *reinterpret_cast<const uint2*>(yp);
      const float2 p0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uo.x));
      const float2 p1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uo.y));
      v[0] += p0.x;
      v[1] += p0.y;
      v[2] += p1.x;
      v[3] += p1.y;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = bf16r_(v[k]);
    st_bf4(yp, v[0], v[1], v[2], v[3]);
  }
  if (epi.ss_out) {  // residual producer: next RMSNorm's weight multiply + row sums
    if (epi.h_out && a.h_w) {
      const uint2 hu = *reinterpret_cast<const uint2*>(a.h_w + f);
      const float2 h0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hu.x));
      const float2 h1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hu.y));
      st_bf4(static_cast<__nv_bfloat16*>(epi.h_out) + off, v[0] * h0.x, v[1] * h0.y,
             v[2] * h1.x, v[3] * h1.y);
    }
    long long q = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) q += __float2ll_rn(v[k] * v[k] * kSsScale);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) q += static_cast<long long>(shfl_xor_u64(q, m));
    if (lane == 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(epi.ss_out) + t,
                static_cast<unsigned long long>(q));
  }
}

// ---- cluster split-K mode: one token tile (T <= 256) and fewer weight tiles
// than SMs (qkv / wo / down at prefill-chunk sizes).  The S CTAs of a cluster
// take S equal k ranges of ONE tile; each leaves its partial tile in its own
// shared memory (the ring, idle once the MMAs completed) and the cluster
// reduces through distributed shared memory in fixed order - the partials
// never touch L2 / HBM (through global memory they cost as much traffic as
// the weights at these shapes, measured) - then each CTA finishes its share
// of the chunks with the same fused epilogue.
template <int kSl>
__global__ void __launch_bounds__(kThreads, 1) gemm_cluster_kernel(
    StreamArgs a, ds_skinny_epi epi, const __grid_constant__ CUtensorMap tw,
    const __grid_constant__ CUtensorMap tx) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // SW128 atoms
  // a stage = kSl 64-column slabs of both operands (one TMA box each: a
  // thread issues a box every ~190 ns whatever its size, so the weight rate
  // of one issuing thread doubles with two-slab boxes; kSl = 1 keeps the ring
  // small enough for two CTAs per SM)
  const int w_bytes = kSl * kSlabA, x_slab = a.NT * 128, x_bytes = kSl * x_slab;
  const int stage_bytes = w_bytes + x_bytes;
  uint8_t* tail = smem + a.stages * stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  uint64_t* empty = full + a.stages;
  uint64_t* acc_full = empty + a.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  // epilogue-phase scalars live in the (then idle) ring after the partial tile
  constexpr int kPT = kBM + 4;  // token-major partial row (features + pad)
  const int ncols = (a.NT + 31) & ~31, nch = ncols / 32;
  float* s_inv = reinterpret_cast<float*>(smem + ncols * kPT * 4);
  int* s_pos = reinterpret_cast<int*>(s_inv + kMaxNT);
  int64_t* s_cell = reinterpret_cast<int64_t*>(s_pos + kMaxNT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = gridDim.x, split = blockIdx.x;  // cluster = the S splits of one tile
  const int wt = blockIdx.y;
  const int n2 = (a.kt + kSl - 1) / kSl;  // stage steps (an odd last slab reads zero-filled)
  const int s_beg = split * n2 / S, s_end = (split + 1) * n2 / S;
  const int n = s_end - s_beg;
  unsigned long long* tr =
      a.trace ? a.trace + (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 16 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtimer();

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 2);  // the weight and the token producer each arrive
      mbar_init(&empty[i], 1);
    }
    mbar_init(acc_full, 1);
    mbar_fence_init();
  }
  if (warp == 1) tc::alloc(tmem_slot, kAccCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  if (tr && threadIdx.x == 0) tr[1] = gtimer();

  if (warp == 0) {
    if (lane == 0) {  // weight boxes: independent of the previous kernel
      tma_prefetch_desc(&tw);
      for (int i = 0; i < n; ++i) {
        const int st = i % a.stages;
        if (i >= a.stages) mbar_wait(&empty[st], static_cast<uint32_t>((i / a.stages) - 1) & 1);
        mbar_expect_tx(&full[st], w_bytes);
        tma_load_3d(smem + st * stage_bytes, &tw, 0, wt * kBM, kSl * (s_beg + i), &full[st]);
      }
      if (tr) tr[2] = gtimer();
    }
    __syncwarp();
  } else if (warp == 2 && lane == 0) {  // token boxes (then this warp joins the epilogue)
    tma_prefetch_desc(&tx);
    pdl_wait();  // the activations come from the previous kernel
    for (int i = 0; i < n; ++i) {
      const int st = i % a.stages;
      if (i >= a.stages) mbar_wait(&empty[st], static_cast<uint32_t>((i / a.stages) - 1) & 1);
      mbar_expect_tx(&full[st], x_bytes);
      tma_load_3d(smem + st * stage_bytes + w_bytes, &tx, 0, 0, kSl * (s_beg + i), &full[st]);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_bf16(kBM, a.NT, false);
      const uint32_t base = smem_u32(smem);
      for (int i = 0; i < n; ++i) {
        const int st = i % a.stages;
        mbar_wait(&full[st], static_cast<uint32_t>(i / a.stages) & 1);
        tc::fence_after();
        const uint32_t pa = base + st * stage_bytes, pb = pa + w_bytes;
#pragma unroll
        for (int j = 0; j < kSl; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc::mma(tmem, tc::smem_desc(pa + j * kSlabA + k * 32, 16, 1024),
                    tc::smem_desc(pb + j * x_slab + k * 32, 16, 1024), idesc,
                    (i > 0 || j > 0 || k > 0) ? 1u : 0u);
        tc::commit(&empty[st]);
      }
      tc::commit(acc_full);
    }
    __syncwarp();
  }
  __syncwarp();
  // partial tiles token-major in shared memory: [NT tokens][kPT features]
  // (padded row: the thread-per-feature writes and the warp-per-token reads
  // are both bank-conflict free)
  const bool epi_warp = warp >= 2;
  const int quad = warp & 3, r = quad * 32 + lane, half = (warp - 2) >> 2;
  const int et = threadIdx.x - 64;  // 0..255
  const int w8 = warp - 2;          // 0..7
  float* part = reinterpret_cast<float*>(smem);
  if (epi_warp) {
    pdl_wait();
    mbar_wait(acc_full, 0);
    tc::fence_after();
    if (tr && threadIdx.x == 64) tr[3] = gtimer();
    // every MMA has completed: the ring is idle and holds the partial tile
    for (int c = half; c < nch; c += 2) {
      float v[32];
      tc::ld32(tmem + (static_cast<uint32_t>(quad * 32) << 16) + c * 32, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) part[(c * 32 + j) * kPT + r] = v[j];
    }
  }
  if (tr && threadIdx.x == 64) tr[4] = gtimer();
  if (S > 1) {
    cluster_sync_all();  // every split's partial tile is in its shared memory
  } else {
    __syncthreads();
  }
  if (tr && threadIdx.x == 64) tr[5] = gtimer();
  if (epi_warp) {
    // split q finishes token rows [rb, re): an equal share for every split
    const int Tn = a.T < a.NT ? a.T : a.NT;
    const int rb = split * Tn / S, re = (split + 1) * Tn / S;
    if (et < re - rb) {  // per-token scalars of the share
      const int tk = rb + et, t = tk;
      if (epi.row_ss) {
        const unsigned long long rs =
            __ldcg(reinterpret_cast<const unsigned long long*>(epi.row_ss) + t);
        s_inv[tk] = rsqrtf(__ull2float_rn(rs) / (kSsScale * static_cast<float>(a.K)) + epi.eps);
      }
      if (epi.rope) {
        const int r_pos = __ldg(epi.row_pos + t), r_seq = __ldg(epi.row_seq + t);
        s_pos[tk] = r_pos;
        s_cell[tk] = __ldg(epi.pos2cell + static_cast<int64_t>(r_seq) * epi.pos_stride + r_pos);
      }
      if (epi.ss_zero && wt == 0) epi.ss_zero[t] = 0;
    }
    named_bar_sync(1, kEpiThreads);
    const uint32_t part_u = smem_u32(part);
    // warp w8 reduces rows rb + w8 + 8i, four at a time: all S splits' rows
    // loaded before the fixed-order sum (deterministic)
    for (int g = rb + w8; g < re; g += 32) {
      float4 acc[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = 0; q < S; ++q) {
        float4 x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int tk = g + 8 * i < re ? g + 8 * i : g;
          const uint32_t ad = part_u + static_cast<uint32_t>((tk * kPT + 4 * lane) * 4);
          x[i] = S > 1 ? dsmem_ld_f32x4(dsmem_map(ad, q))
                       : *reinterpret_cast<const float4*>(smem + (ad - part_u));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[i].x += x[i].x;
          acc[i].y += x[i].y;
          acc[i].z += x[i].z;
          acc[i].w += x[i].w;
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int tk = g + 8 * i;
        if (tk < re)  // warp-uniform
          epilogue_tokrow(acc[i], a, epi, wt, tk, lane, s_inv, s_pos, s_cell);
      }
    }
  }
  if (tr && threadIdx.x == 64) tr[9] = gtimer();
  if (S > 1) cluster_sync_all();  // peers keep their shared memory until every read is done
  tc::fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) {
    __threadfence();
    tr[7] = gtimer();
  }
  if (warp == 1) {
    tc::fence_after();
    tc::dealloc(tmem, kAccCols);
  }
}

unsigned long long* g_trace = nullptr;  // DS_STREAM_TRACE buffer

struct StreamPlan {
  int NT, n_tt, kt, tiles, stages, smem, P;
  int64_t total;
};

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

StreamPlan stream_plan(int T, int N, int K) {
  StreamPlan p{};
  p.n_tt = (T + kMaxNT - 1) / kMaxNT;
  p.NT = ((T + p.n_tt - 1) / p.n_tt + 15) / 16 * 16;
  p.kt = K / 64;
  p.tiles = (N / kBM) * p.n_tt;
  p.total = static_cast<int64_t>(p.tiles) * p.kt;
  static const int ctas_env = getenv("DS_STREAM_CTAS") ? atoi(getenv("DS_STREAM_CTAS")) : 0;
  p.P = ctas_env > 0 ? ctas_env : num_sms();
  if (p.P > p.total) p.P = static_cast<int>(p.total);
  const int stage = kSlabA + p.NT * 128;
  const int fixed = 1024 + kScalarBytes + 256;
  int ns = (kSmemMax - fixed) / stage;
  if (ns > 8) ns = 8;
  p.stages = ns;
  p.smem = fixed + ns * stage;
  // the finalize batches reuse half the ring each: one participant chunk must fit
  if (static_cast<int64_t>(ns) * stage / 2 < static_cast<int64_t>(kBM) * 36 * 4) p.stages = 0;
  return p;
}

// co-resident clusters of `size` CTAs of gemm_cluster_kernel at `smem` bytes
int max_clusters(int size, int smem) {
  static int cache[9][2] = {};
  const int wide = smem > 120 * 1024;
  if (size < 1 || size > 8) return 0;
  if (cache[size][wide]) return cache[size][wide];
  cudaFuncSetAttribute(gemm_cluster_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
  cudaFuncSetAttribute(gemm_cluster_kernel<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(size, 1, 1);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = size;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_cluster_kernel<2>, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = num_sms() / size;
  }
  return cache[size][wide] = n;
}

struct Workspace {
  float* partials = nullptr;
  int* flags = nullptr;
  int P = 0;
};

Workspace* workspace(int P) {
  static std::mutex mu;
  static Workspace ws[16];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  Workspace& w = ws[dev & 15];
  if (w.P < P) {
    if (w.partials) cudaFree(w.partials);
    if (!w.flags) {
      if (cudaMalloc(&w.flags, kMaxFlags * sizeof(int)) != cudaSuccess) return nullptr;
      cudaMemset(w.flags, 0, kMaxFlags * sizeof(int));
    }
    if (cudaMalloc(&w.partials, static_cast<size_t>(P) * 2 * kSlotFloats * sizeof(float)) !=
        cudaSuccess)
      return nullptr;
    cudaDeviceSynchronize();  // the flags' memset lands before any launch
    w.P = P;
  }
  return &w;
}
}  // namespace

}  // namespace ds


// DS_STREAM_TRACE debug: the last traced launch's per-CTA globaltimer stamps
// [ctas][8] (start, setup done, producer done, MMA done, first contribution
// published, head wait start, head wait end, exit)
namespace ds {
namespace {
__global__ void stamp_kernel(unsigned long long* out) { *out = gtimer(); }
}  // namespace
}  // namespace ds

// debug: one globaltimer stamp on the stream (brackets a traced launch)
extern "C" int ds_debug_stamp(unsigned long long* dev_out, ds_stream_t stream) {
  ds::stamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(dev_out);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int ds_gemm_stream_trace(unsigned long long* host_out, int n_ctas) {
  if (!ds::g_trace) return DS_EINVAL;
  return static_cast<int>(
      cudaMemcpy(host_out, ds::g_trace, static_cast<size_t>(n_ctas) * 128, cudaMemcpyDeviceToHost));
}

extern "C" int ds_gemm_stream(const void* X, const void* W, void* Y, int T, int N, int K,
                              int y_f32, int accumulate, const ds_skinny_epi* epi_in,
                              ds_stream_t stream) {
  using namespace ds;
  if (T <= 0 || N % kBM || K % 64 || K < 64) return DS_EINVAL;
  ds_skinny_epi epi{};
  if (epi_in) epi = *epi_in;
  if ((epi.swiglu && (y_f32 || accumulate)) || (epi.rope && (y_f32 || accumulate)) ||
      (epi.argmax_out && (!y_f32 || accumulate)) || (!Y && !epi.argmax_out) ||
      (epi.ss_out && !(y_f32 && accumulate)))
    return DS_EINVAL;
  if (epi.rope && (epi.n_heads <= 0 || epi.n_kv_heads <= 0)) return DS_EINVAL;
  const StreamPlan p = stream_plan(T, N, K);
  if (p.tiles > kMaxFlags || p.stages < 2) return DS_EUNSUPPORTED;
  Workspace* ws = workspace(p.P);
  if (!ws) return DS_EWORKSPACE;
  const CUtensorMap* tw = slab_tensor_map(W, N, K, kBM, 1);
  const CUtensorMap* tx = slab_tensor_map(X, T, K, p.NT, 1);
  if (!tw || !tx) return DS_EUNSUPPORTED;
  static int attr_smem = 0;
  if (p.smem > attr_smem) {
    cudaFuncSetAttribute(gemm_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmemMax);
    attr_smem = kSmemMax;
  }
  if (getenv("DS_STREAM_VERBOSE"))
    fprintf(stderr, "gemm_stream T=%d N=%d K=%d: NT=%d n_tt=%d tiles=%d iters=%lld ctas=%d "
            "stages=%d smem=%d\n", T, N, K, p.NT, p.n_tt, p.tiles,
            static_cast<long long>(p.total), p.P, p.stages, p.smem);
  // one token tile and fewer weight tiles than SMs: cluster split-K (the
  // partials reduce through distributed shared memory), two-slab stages
  static const int cl_env = getenv("DS_STREAM_CLUSTER") ? atoi(getenv("DS_STREAM_CLUSTER")) : 1;
  int S = 0, cl_stages = 0, cl_smem = 0;
  // one-token-tile shapes with up to two tiles per SM (gate_up at T <= 256:
  // 224 tiles) run unsplit, single-slab stages, two CTAs per SM
  // (DS_STREAM_CL_BIG=0 sends them to stream-K)
  static const int cl_big = getenv("DS_STREAM_CL_BIG") ? atoi(getenv("DS_STREAM_CL_BIG")) : 1;
  const bool big = cl_big && p.n_tt == 1 && p.tiles >= num_sms() && p.tiles <= 2 * num_sms();
  int sl = 2;  // slabs per ring stage
  if (cl_env && p.n_tt == 1 && (p.tiles < num_sms() || big)) {
    // partial tile + the epilogue scalars (s_inv, s_pos, s_cell) in the ring
    const int64_t part = static_cast<int64_t>((p.NT + 31) & ~31) * (kBM + 4) * 4 +
                         kMaxNT * (4 + 4 + 8);
    const int fixed = 1024 + 256;  // alignment slack + barriers
    if (big) {
      // unsplit, two CTAs per SM: single-slab stages, a ring of ~110 KB
      sl = 1;
      const int stage = kSlabA + p.NT * 128;
      cl_stages = static_cast<int>((part + stage - 1) / stage);
      if (cl_stages < 3) cl_stages = 3;
      cl_smem = fixed + cl_stages * stage;
      S = cl_smem <= kSmemMax ? 1 : 0;
    } else {
      // two-slab stages (weights 32 KB + tokens NT x 256 B per stage)
      const int stage = 2 * (kSlabA + p.NT * 128);
      cl_stages = (kSmemMax - fixed) / stage;
      if (cl_stages > 4) cl_stages = 4;
      if (static_cast<int64_t>(cl_stages) * stage < part)
        cl_stages = static_cast<int>((part + stage - 1) / stage);
      cl_smem = fixed + cl_stages * stage;
      if (cl_stages >= 2 && cl_smem <= kSmemMax) {
        static const int smax = getenv("DS_STREAM_SMAX") ? atoi(getenv("DS_STREAM_SMAX")) : 8;
        const int n2 = (p.kt + 1) / 2;
        S = num_sms() / p.tiles;
        if (S > smax) S = smax;
        if (S < 1) S = 1;
        while (S > 1 && n2 / S < 2) --S;
        while (S > 1 && max_clusters(S, cl_smem) < p.tiles) --S;
      }
    }
  }
  StreamArgs a{};
  a.Y = Y;
  a.h_w = static_cast<const __nv_bfloat16*>(epi.h_w);
  a.partials = ws->partials;
  a.flags = ws->flags;
  a.total = p.total;
  a.T = T;
  a.N = N;
  a.K = K;
  a.y_f32 = y_f32;
  a.accumulate = accumulate;
  a.NT = p.NT;
  a.n_tt = p.n_tt;
  a.kt = p.kt;
  a.stages = p.stages;
  a.trace = nullptr;
  if (getenv("DS_STREAM_TRACE")) {
    if (!g_trace) {
      cudaMalloc(&g_trace, 4096 * 16 * 8);
      cudaMemset(g_trace, 0, 4096 * 16 * 8);
    }
    a.trace = g_trace;
  }
  static const bool no_pdl = getenv("DS_STREAM_NOPDL") && atoi(getenv("DS_STREAM_NOPDL"));
  cudaError_t e;
  if (S >= 1) {
    static bool cl_attr = false;
    if (!cl_attr) {
      for (auto k : {gemm_cluster_kernel<1>, gemm_cluster_kernel<2>}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      }
      cl_attr = true;
    }
    if (getenv("DS_STREAM_VERBOSE"))
      fprintf(stderr, "gemm_stream cluster mode: %d tiles x %d splits, %d stages, %d B smem\n",
              p.tiles, S, cl_stages, cl_smem);
    a.stages = cl_stages;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(S, p.tiles, 1);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = cl_smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = S;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (getenv("DS_STREAM_TRACE")) {
      if (!g_trace) {
        cudaMalloc(&g_trace, 4096 * 16 * 8);
        cudaMemset(g_trace, 0, 4096 * 16 * 8);
      }
      a.trace = g_trace;
    }
    const CUtensorMap* tw2 = slab_tensor_map(W, N, K, kBM, sl);
    const CUtensorMap* tx2 = slab_tensor_map(X, T, K, p.NT, sl);
    if (!tw2 || !tx2) return DS_EUNSUPPORTED;
    e = cudaLaunchKernelEx(&cfg, sl == 1 ? gemm_cluster_kernel<1> : gemm_cluster_kernel<2>, a,
                           epi, *tw2, *tx2);
    if (e != cudaSuccess) return static_cast<int>(e);
    return static_cast<int>(cudaGetLastError());
  }
  if (no_pdl) {
    gemm_stream_kernel<<<p.P, kThreads, p.smem, (cudaStream_t)stream>>>(a, epi, *tw, *tx);
    e = cudaGetLastError();
  } else {
    e = launch_pdl(gemm_stream_kernel, dim3(p.P), dim3(kThreads), p.smem, (cudaStream_t)stream,
                   a, epi, *tw, *tx);
  }
  if (e != cudaSuccess) return static_cast<int>(e);
  return static_cast<int>(cudaGetLastError());
}
