// K9: projection GEMM for prefill chunks and batched plans (33..4096 rows) on
// the 5th-generation tensor cores: Y[T][N] (+)= X[T][K] . W[N][K]^T.
//
// Tile = 128 weight rows (UMMA M) x NT tokens (UMMA N <= 256, every token of a
// chunk up to 256 in one tile, so each weight byte is read once per 256
// tokens) x a K range.  The accumulator lives in TMEM (NT fp32 columns).
// Warp roles (192 threads):
//   warp 0  TMA producer: per 64-column slab one box of the 128 weight rows
//           and one box of the NT token rows (3D slab tensor maps, SWIZZLE_128B,
//           token rows past T zero-filled) into an mbarrier ring; the weight
//           boxes of the first round are issued before the programmatic-
//           dependency wait (weights do not depend on the previous kernel);
//   warp 1  TMEM allocation and the single-thread MMA issue: 4 x
//           tcgen05.mma kind::f16 (K=16) per slab, stage release and the
//           accumulator hand-off through tcgen05.commit;
//   warps 2-5 epilogue: tcgen05.ld of the accumulator, thread = weight row.
// Split-K (wo/down/wqkv have 32-48 row tiles for 148 SMs): the S splits of a
// tile form a thread-block cluster; each leaves its partial tile in its own
// shared memory (over the drained ring) and the cluster reduces it through
// distributed shared memory in fixed split order - deterministic, no global
// workspace, no second launch.
// Epilogue: bf16 store, or fp32 store / accumulate (the residual stream).
#include "../../include/deltaserve_b200.h"
#include "common.cuh"
#include "tc.cuh"
#include "tma.h"

#include <cstdio>
#include <cstdlib>

namespace ds {

namespace {
constexpr int kBM = 128;                  // weight rows per tile (UMMA M)
constexpr int kSlabA = kBM * 128;         // one 64-column slab of the weight tile (16 KB)
constexpr int kThreads = 6 * 32;
constexpr int kTmemCols = 256;
constexpr int kSmemBudget = 112 * 1024;   // two CTAs per SM
constexpr int kSmemBudgetWide = 220 * 1024;  // one CTA per SM
constexpr int kMaxSplits = 8;
}  // namespace

__global__ void __launch_bounds__(kThreads, 1) gemm_tc_kernel(
    void* __restrict__ Y, int T, int N, int K, int y_f32, int accumulate, int NT, int n_stages,
    int ks, const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // SW128 atoms
  // a stage holds ks 64-column slabs: [ks][128 rows][128 B] weights, then
  // [ks][NT rows][128 B] tokens
  const int a_bytes = ks * kSlabA, stage_bytes = a_bytes + ks * NT * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + n_stages * stage_bytes);
  uint64_t* empty = full + n_stages;
  uint64_t* acc_full = empty + n_stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  float* red = reinterpret_cast<float*>(smem);  // [NT][128] partial tile (ring drained)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int splits = gridDim.z, split = blockIdx.z;
  const int f0 = blockIdx.y * kBM, t0 = blockIdx.x * NT;  // token tiles of one weight tile adjacent
  const int slabs = K / (64 * ks);  // stages along K
  const int s_beg = split * slabs / splits, s_end = (split + 1) * slabs / splits;
  const int nsl = s_end - s_beg;

  if (threadIdx.x == 0) {
    for (int i = 0; i < n_stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(acc_full, 1);
    mbar_fence_init();
  }
  if (warp == 1) tc::alloc(tmem_slot, kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tw);
      tma_prefetch_desc(&tx);
      const int pre = nsl < n_stages ? nsl : n_stages;
      const uint32_t tx_bytes = stage_bytes;
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(&full[i], tx_bytes);
        tma_load_3d(smem + i * stage_bytes, &tw, 0, f0, (s_beg + i) * ks, &full[i]);
      }
      pdl_wait();  // the activations come from the previous kernel
      for (int i = 0; i < pre; ++i)
        tma_load_3d(smem + i * stage_bytes + a_bytes, &tx, 0, t0, (s_beg + i) * ks, &full[i]);
      for (int i = pre; i < nsl; ++i) {
        const int st = i % n_stages;
        mbar_wait(&empty[st], ((i / n_stages) - 1) & 1);
        uint8_t* sp = smem + st * stage_bytes;
        mbar_expect_tx(&full[st], tx_bytes);
        tma_load_3d(sp, &tw, 0, f0, (s_beg + i) * ks, &full[st]);
        tma_load_3d(sp + a_bytes, &tx, 0, t0, (s_beg + i) * ks, &full[st]);
      }
    }
    __syncwarp();  // reconverge before the CTA barrier (bar.sync is warp-aligned)
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_bf16(kBM, NT, false);
      const uint32_t base = smem_u32(smem);
      for (int i = 0; i < nsl; ++i) {
        const int st = i % n_stages;
        mbar_wait(&full[st], (i / n_stages) & 1);
        tc::fence_after();
        const uint32_t a = base + st * stage_bytes, b = a + a_bytes;
        for (int k = 0; k < 4 * ks; ++k)
          tc::mma(tmem, tc::smem_desc(a + (k >> 2) * kSlabA + (k & 3) * 32, 16, 1024),
                  tc::smem_desc(b + (k >> 2) * NT * 128 + (k & 3) * 32, 16, 1024), idesc,
                  (i | k) > 0);
        tc::commit(&empty[st]);  // the stage is free once its MMAs completed
      }
      tc::commit(acc_full);
    }
    __syncwarp();
  } else {
    // epilogue warps 2-5: TMEM lane quadrant (warp & 3), thread = weight row
    pdl_wait();  // the residual (accumulate) comes from the previous kernel
    const int quad = warp & 3, f = quad * 32 + lane;
    mbar_wait(acc_full, 0);
    tc::fence_after();
    const uint32_t taddr = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    for (int c = 0; c < NT; c += 32) {
      float v[32];
      tc::ld32(taddr + c, v);
      if (splits > 1) {  // partial tile -> own smem (the ring is drained: acc_full)
        if (c == 0) tc::fence_proxy_async();  // generic writes after the async-proxy traffic
#pragma unroll
        for (int j = 0; j < 32; ++j) red[(c + j) * kBM + f] = v[j];
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int t = t0 + c + j;
          if (t >= T) continue;
          const int64_t o = static_cast<int64_t>(t) * N + f0 + f;
          if (y_f32) {
            float* yp = static_cast<float*>(Y) + o;
            *yp = accumulate ? *yp + v[j] : v[j];
          } else {
            __nv_bfloat16* yp = static_cast<__nv_bfloat16*>(Y) + o;
            *yp = __float2bfloat16_rn(accumulate ? __bfloat162float(*yp) + v[j] : v[j]);
          }
        }
      }
    }
  }
  pdl_trigger();
  tc::fence_before();
  __syncthreads();
  if (splits > 1) {
    // cluster reduction: CTA `split` owns token rows j = split, split + S, ...;
    // item = (owned row, 4 features), all 6 warps, two items in flight per
    // thread with every split's float4 loaded before the fixed-order sum
    cluster_sync_all();  // every split's partial tile is in its smem
    const int own = (NT - split + splits - 1) / splits, items = own * (kBM / 4);
    for (int i0 = threadIdx.x; i0 < items; i0 += 2 * kThreads) {
      float4 p[2][kMaxSplits];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int it = i0 + u * kThreads;
        const int j = split + (it >> 5) * splits;
        const uint32_t a = smem_u32(red + j * kBM + (it & 31) * 4);
#pragma unroll
        for (int q = 0; q < kMaxSplits; ++q)
          p[u][q] = (q < splits && it < items) ? dsmem_ld_f32x4(dsmem_map(a, q))
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int it = i0 + u * kThreads;
        const int t = t0 + split + (it >> 5) * splits;
        if (it >= items || t >= T) continue;
        float4 s = p[u][0];
#pragma unroll
        for (int q = 1; q < kMaxSplits; ++q) {  // fixed split order
          s.x += p[u][q].x;
          s.y += p[u][q].y;
          s.z += p[u][q].z;
          s.w += p[u][q].w;
        }
        const int64_t o = static_cast<int64_t>(t) * N + f0 + (it & 31) * 4;
        if (y_f32) {
          float4* yp = reinterpret_cast<float4*>(static_cast<float*>(Y) + o);
          if (accumulate) {
            const float4 r = *yp;
            s.x += r.x;
            s.y += r.y;
            s.z += r.z;
            s.w += r.w;
          }
          *yp = s;
        } else {
          uint2* yp = reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(Y) + o);
          if (accumulate) {
            const uint2 r = *yp;
            const float2 r0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
            const float2 r1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
            s.x += r0.x;
            s.y += r0.y;
            s.z += r1.x;
            s.w += r1.y;
          }
          __nv_bfloat162 b0 = __floats2bfloat162_rn(s.x, s.y), b1 = __floats2bfloat162_rn(s.z, s.w);
          *yp = make_uint2(*reinterpret_cast<uint32_t*>(&b0), *reinterpret_cast<uint32_t*>(&b1));
        }
      }
    }
    cluster_sync_all();  // peers keep their smem until every read is done
  }
  if (warp == 1) {
    tc::fence_after();
    tc::dealloc(tmem, kTmemCols);
  }
}

namespace {
// co-resident clusters of `size` one-CTA-per-SM CTAs (kSmemBudgetWide)
int max_clusters(int size) {
  static int cache[kMaxSplits + 1] = {0};
  if (size < 1 || size > kMaxSplits) return 0;
  if (cache[size]) return cache[size];
  cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kSmemBudgetWide);
  cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1, 1, size);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBudgetWide;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = size;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 148 / size;
  }
  return cache[size] = n;
}

struct TcPlan {
  int NT, n_tt, splits, n_stages, smem, ks;
};

TcPlan tc_plan(int T, int N, int K) {
  TcPlan p{};
  p.n_tt = (T + 255) / 256;
  p.NT = ((T + p.n_tt - 1) / p.n_tt + 15) / 16 * 16;
  if (p.NT < 32) p.NT = 32;
  const int tiles = (N / kBM) * p.n_tt, slabs = K / 64;
  // splits: tiles < 148 (wo/down/wqkv) split K so that one wave of one CTA
  // per SM holds them all, each CTA with a deep (~200 KB) ring; tiles >= 148
  // (gate_up) run unsplit, two 112 KB CTAs per SM
  static const int splits_env = getenv("DS_TC_SPLITS") ? atoi(getenv("DS_TC_SPLITS")) : 0;
  p.splits = 1;
  int budget = kSmemBudget;
  if (tiles < 148) {
    p.splits = 148 / tiles;
    if (p.splits > kMaxSplits) p.splits = kMaxSplits;
    while (p.splits > 1 && slabs / p.splits < 4) --p.splits;
    // a cluster is placed inside one GPC: fewer clusters of S fit than 148/S
    // (e.g. 3-CTA clusters of 222 KB CTAs: < 48), and one more would be a
    // second wave
    while (p.splits > 1 && tiles > max_clusters(p.splits)) --p.splits;
    budget = kSmemBudgetWide;
  }
  if (splits_env > 0) p.splits = splits_env;
  static const int kb_env = getenv("DS_TC_KB") ? atoi(getenv("DS_TC_KB")) * 1024 : 0;
  if (kb_env) budget = kb_env;
  static const int ks_env = getenv("DS_TC_KS") ? atoi(getenv("DS_TC_KS")) : 1;
  p.ks = ks_env;
  while (p.ks > 1 && (K / 64) % p.ks) --p.ks;
  const int stage = p.ks * (kSlabA + p.NT * 128);
  int ns = (budget - 1024 - 2048) / stage;
  if (ns < 2) ns = 2;
  if (ns > 8) ns = 8;
  // the split partial tile [NT][128] fp32 reuses the ring
  while (p.splits > 1 && ns * stage < p.NT * kBM * 4) ++ns;
  p.n_stages = ns;
  p.smem = 1024 + ns * stage + 2 * ns * 8 + 16 + 64;
  return p;
}
}  // namespace

}  // namespace ds

extern "C" int ds_gemm_tc(const void* X, const void* W, void* Y, int T, int N, int K, int y_f32,
                          int accumulate, ds_stream_t stream) {
  using namespace ds;
  if (T <= 0 || N % kBM || K % 64 || K < 128) return DS_EINVAL;
  const TcPlan p = tc_plan(T, N, K);
  if (p.smem > 227 * 1024) return DS_EUNSUPPORTED;
  if (getenv("DS_TC_VERBOSE"))
    fprintf(stderr,
            "gemm_tc T=%d N=%d K=%d: NT=%d tiles=%d splits=%d ks=%d stages=%d smem=%d "
            "(clusters of 2..8: %d %d %d %d %d %d %d)\n",
            T, N, K, p.NT, (N / kBM) * p.n_tt, p.splits, p.ks, p.n_stages, p.smem,
            max_clusters(2), max_clusters(3), max_clusters(4), max_clusters(5), max_clusters(6),
            max_clusters(7), max_clusters(8));
  const CUtensorMap* tw = slab_tensor_map(W, N, K, kBM, p.ks);
  const CUtensorMap* tx = slab_tensor_map(X, T, K, p.NT, p.ks);
  if (!tw || !tx) return DS_EUNSUPPORTED;
  static int attr_smem = 0;
  if (p.smem > attr_smem) {
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem);
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_smem = p.smem;
  }
  const dim3 grid(p.n_tt, N / kBM, p.splits);
  cudaError_t e;
  if (p.splits > 1)
    e = launch_pdl_cluster_z(gemm_tc_kernel, grid, dim3(kThreads), p.smem, p.splits,
                             (cudaStream_t)stream, Y, T, N, K, y_f32, accumulate, p.NT,
                             p.n_stages, p.ks, *tw, *tx);
  else
    e = launch_pdl(gemm_tc_kernel, grid, dim3(kThreads), p.smem, (cudaStream_t)stream, Y, T, N,
                   K, y_f32, accumulate, p.NT, p.n_stages, p.ks, *tw, *tx);
  if (e != cudaSuccess) return static_cast<int>(e);
  return static_cast<int>(cudaGetLastError());
}
