// Shared device helpers for the deltaserve B200 kernels (sm_100a only).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "deltaserve_b200 targets sm_100a only"
#endif

#define DS_DEVICE __device__ __forceinline__

namespace ds {

constexpr uint64_t kFnv64Offset = 0xCBF29CE484222325ull;
constexpr uint64_t kFnv64Prime = 0x100000001B3ull;
constexpr uint32_t kFnv32Offset = 0x811C9DC5u;
constexpr uint32_t kFnv32Prime = 0x01000193u;

DS_DEVICE uint64_t fnv64_token(uint64_t h, int32_t tok) {
  const uint32_t t = static_cast<uint32_t>(tok);
  h = (h ^ (t & 0xFFu)) * kFnv64Prime;
  h = (h ^ ((t >> 8) & 0xFFu)) * kFnv64Prime;
  h = (h ^ ((t >> 16) & 0xFFu)) * kFnv64Prime;
  h = (h ^ (t >> 24)) * kFnv64Prime;
  return h;
}

DS_DEVICE uint32_t fnv32_token(uint32_t h, int32_t tok) {
  const uint32_t t = static_cast<uint32_t>(tok);
  h = (h ^ (t & 0xFFu)) * kFnv32Prime;
  h = (h ^ ((t >> 8) & 0xFFu)) * kFnv32Prime;
  h = (h ^ ((t >> 16) & 0xFFu)) * kFnv32Prime;
  h = (h ^ (t >> 24)) * kFnv32Prime;
  return h;
}

template <typename T>
DS_DEVICE T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

template <typename T>
DS_DEVICE T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

DS_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async global->shared copy (LDGSTS), L2-only caching.
DS_DEVICE void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
DS_DEVICE void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  const int src = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src));
}
DS_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
DS_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

DS_DEVICE uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ldmatrix wrappers (8x8 b16 tiles).
DS_DEVICE void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
DS_DEVICE void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D (fp32).
DS_DEVICE void mma_bf16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

DS_DEVICE float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA/ALU pipes (offloads the MUFU): x = n + f with n = rint(x)
// (1.5 * 2^23 shifter), f in [-0.5, 0.5], 2^f by a degree-3 polynomial
// (relative error < 5e-4, under the bf16 rounding of P), then n added to the
// exponent field.  x is clamped at -126 (masked scores: -inf -> ~0).
DS_DEVICE float poly_exp2(float x) {
  x = fmaxf(x, -126.f);
  const float r = __fadd_rn(x, 12582912.f);
  const float f = __fsub_rn(x, __fsub_rn(r, 12582912.f));
  float p = fmaf(f, 0.0555041087f, 0.2402265070f);
  p = fmaf(p, f, 0.6931471806f);
  p = fmaf(p, f, 1.0f);
  const int n = __float_as_int(r) - 0x4B400000;
  return __int_as_float(__float_as_int(p) + (n << 23));
}

}  // namespace ds

// ---------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA engine, non-tensor) helpers
// ---------------------------------------------------------------------------
namespace ds {

DS_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
DS_DEVICE void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
DS_DEVICE void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
DS_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
DS_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy on the async (TMA) engine; completes tx bytes on bar
DS_DEVICE void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
DS_DEVICE void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

}  // namespace ds

// ---------------------------------------------------------------------------
// Programmatic dependent launch: every forward kernel is launched with
// programmatic stream serialization; it waits for its predecessor's memory
// (griddepcontrol.wait) only where it first consumes it, and lets the next
// kernel launch early (launch_dependents) so its prologue - e.g. the skinny
// GEMM's first weight loads, which do not depend on activations - overlaps.
// ---------------------------------------------------------------------------
namespace ds {
DS_DEVICE void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
DS_DEVICE void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Up to two byte ranges to pull into L2 while a latency-bound kernel leaves
// HBM idle (the attention pulls the next projections' weights): CTA `cta` of
// `n_cta` prefetches its equal share of the two ranges laid end to end.
struct L2Hint {
  const char* p[2];
  int64_t n[2];
};
DS_DEVICE void l2_prefetch_share(const L2Hint& h, int64_t cta, int64_t n_cta) {
  const int64_t n0 = h.p[0] ? h.n[0] & ~15ll : 0, n1 = h.p[1] ? h.n[1] & ~15ll : 0;
  const int64_t total = n0 + n1;
  if (total <= 0) return;
  const int64_t share = ((total + n_cta - 1) / n_cta + 15) & ~15ll;
  const int64_t beg = share * cta, end = beg + share < total ? beg + share : total;
  for (int64_t off = beg; off < end;) {
    const bool first = off < n0;
    const int64_t lim = first ? (end < n0 ? end : n0) : end;
    const int64_t c = lim - off < 32768 ? lim - off : 32768;
    const char* src = first ? h.p[0] + off : h.p[1] + (off - n0);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(static_cast<uint32_t>(c))
                 : "memory");
    off += c;
  }
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// same, with thread-block clusters of `cluster` CTAs along z
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster_z(void (*kern)(KArgs...), dim3 grid, dim3 block,
                                        size_t smem, int cluster, cudaStream_t stream,
                                        Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = cluster;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- packed row argmax: one u64 max = (largest value, lowest index) ----
DS_DEVICE unsigned long long argmax_key(float v, int idx) {
  uint32_t u = __float_as_uint(v + 0.f);  // -0 -> +0 (equal values tie on the index)
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(idx));
}
DS_DEVICE int argmax_key_index(unsigned long long key) {
  return static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(key));
}

// ---- thread-block cluster / distributed shared memory ----
DS_DEVICE uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
DS_DEVICE void cluster_sync_all() {  // every thread of every CTA in the cluster
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" :::
                   "memory");
}
DS_DEVICE uint32_t dsmem_map(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
DS_DEVICE float dsmem_ld_f32(uint32_t cluster_addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];\n" : "=f"(v) : "r"(cluster_addr));
  return v;
}
DS_DEVICE float4 dsmem_ld_f32x4(uint32_t cluster_addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_addr));
  return v;
}
}  // namespace ds
