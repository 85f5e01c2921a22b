// Element-wise / row kernels of the Llama-shaped forward: embedding gather,
// RMSNorm, SwiGLU, and K5 (RoPE + KV store into the paged cell pool).
// All HBM-bound; 128-bit vectorised where the row is.
#include "../../include/deltaserve_b200.h"
#include "common.cuh"

namespace ds {

// out[r] = table[tok[r]] as bf16 (out_f32=0) or widened to fp32 (residual stream)
__global__ void embed_kernel(const int32_t* __restrict__ tok, const uint4* __restrict__ table,
                             int chunks, void* __restrict__ out, int out_f32) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const uint4* src = table + static_cast<int64_t>(tok[r]) * chunks;
  for (int j = threadIdx.x; j < chunks; j += blockDim.x) {
    const uint4 v = __ldg(src + j);
    if (out_f32) {
      const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
      float4* dst = reinterpret_cast<float4*>(out) + (static_cast<int64_t>(r) * chunks + j) * 2;
      const float2 a = __bfloat1622float2(p[0]), b = __bfloat1622float2(p[1]);
      const float2 c = __bfloat1622float2(p[2]), d = __bfloat1622float2(p[3]);
      dst[0] = make_float4(a.x, a.y, b.x, b.y);
      dst[1] = make_float4(c.x, c.y, d.x, d.y);
    } else {
      reinterpret_cast<uint4*>(out)[static_cast<int64_t>(r) * chunks + j] = v;
    }
  }
}

// out[r] = x[rows[r]] * rsqrt(mean(x^2) + eps) * w   (fp32 math, one rounding)
// x is the bf16 or fp32 residual stream; 8 elements per chunk.
DS_DEVICE void load8(const void* x, int64_t idx, bool f32, float* f) {
  if (f32) {
    const float4* p = reinterpret_cast<const float4*>(x) + idx * 2;
    const float4 a = __ldg(p), b = __ldg(p + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  } else {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(x) + idx);
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 t = __bfloat1622float2(p[q]);
      f[2 * q] = t.x;
      f[2 * q + 1] = t.y;
    }
  }
}

template <int BLOCK, int MAXC>
__global__ void __launch_bounds__(BLOCK) rmsnorm_kernel(const void* __restrict__ x,
                                                        const int32_t* __restrict__ rows,
                                                        int chunks, int x_f32,
                                                        const uint4* __restrict__ w, float eps,
                                                        uint4* __restrict__ out) {
  __shared__ float s_part[BLOCK / 32];
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const int64_t src = rows ? rows[r] : r;
  float v[MAXC][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < MAXC; ++k) {
    const int j = threadIdx.x + k * BLOCK;
    if (j < chunks) {
      load8(x, src * chunks + j, x_f32 != 0, v[k]);
#pragma unroll
      for (int q = 0; q < 8; ++q) ss += v[k][q] * v[k][q];
    }
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < BLOCK / 32 ? s_part[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) s_part[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(s_part[0] / static_cast<float>(chunks * 8) + eps);
  uint4* orow = out + static_cast<int64_t>(r) * chunks;
#pragma unroll
  for (int k = 0; k < MAXC; ++k) {
    const int j = threadIdx.x + k * BLOCK;
    if (j < chunks) {
      const uint4 wv = __ldg(w + j);
      const __nv_bfloat162* pw = reinterpret_cast<const __nv_bfloat162*>(&wv);
      uint4 o;
      uint32_t* po = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 g = __bfloat1622float2(pw[q]);
        po[q] = pack_bf16(v[k][2 * q] * inv * g.x, v[k][2 * q + 1] * inv * g.y);
      }
      orow[j] = o;
    }
  }
}

// out[r][f] = silu(gate f) * up f; gate|up rows interleaved in 8-unit blocks
// (ds_model.w_gate_up): 16-byte chunk j of the output reads chunks 2j, 2j+1
__global__ void silu_mul_kernel(const uint4* __restrict__ gu, int chunks, uint4* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= chunks) return;
  const uint4 g = __ldg(gu + static_cast<int64_t>(r) * 2 * chunks + 2 * j);
  const uint4 u = __ldg(gu + static_cast<int64_t>(r) * 2 * chunks + 2 * j + 1);
  const __nv_bfloat162* pg = reinterpret_cast<const __nv_bfloat162*>(&g);
  const __nv_bfloat162* pu = reinterpret_cast<const __nv_bfloat162*>(&u);
  uint4 o;
  uint32_t* po = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 a = __bfloat1622float2(pg[q]);
    const float2 b = __bfloat1622float2(pu[q]);
    const float sa = a.x / (1.f + expf(-a.x));
    const float sb = a.y / (1.f + expf(-a.y));
    po[q] = pack_bf16(sa * b.x, sb * b.y);
  }
  out[static_cast<int64_t>(r) * chunks + j] = o;
}

// K5: rotate-half RoPE on q (in place, written back in plain dim order) and k,
// store k and v rows into the head-major cell pool.  q/k head columns arrive
// RoPE-pair interleaved (ds_model.wqkv: column 16t+j = dim 8t+j or 64+8t+j-8),
// so the row's q/k part is staged in smem before the in-place rewrite.  One
// CTA per batch row.  (The decode forward folds this into the wqkv epilogue.)

__global__ void rope_kv_store_kernel(__nv_bfloat16* __restrict__ qkv, const int32_t* row_seq,
                                     const int32_t* row_pos, const int32_t* __restrict__ pos2cell,
                                     int64_t pos_stride, int nh, int nkv, int hd,
                                     const float* __restrict__ rope_cos,
                                     const float* __restrict__ rope_sin,
                                     __nv_bfloat16* __restrict__ k_pool,
                                     __nv_bfloat16* __restrict__ v_pool, int64_t head_stride) {
  extern __shared__ __align__(16) __nv_bfloat16 stage[];  // [(nh + nkv) * hd]
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const int pos = row_pos[r];
  const int64_t cell = pos2cell[static_cast<int64_t>(row_seq[r]) * pos_stride + pos];
  const int half = hd / 2;
  const int width = (nh + 2 * nkv) * hd;
  __nv_bfloat16* row = qkv + static_cast<int64_t>(r) * width;
  const int qk_chunks = (nh + nkv) * hd / 8;
  for (int j = threadIdx.x; j < qk_chunks; j += blockDim.x)
    reinterpret_cast<uint4*>(stage)[j] = reinterpret_cast<const uint4*>(row)[j];
  __syncthreads();
  // pair block t of a head (dims 8t..8t+7 and 64+8t..64+8t+7) is the one
  // contiguous 32-byte column chunk [16t, 16t+16): one thread per block reads
  // it from the staged copy and writes two 16-byte rows of rotated output
  // (in place for q and k, and k into the pool) - vector stores, not bf16
  // scalars
  const float* cs = rope_cos + static_cast<int64_t>(pos) * half;
  const float* sn = rope_sin + static_cast<int64_t>(pos) * half;
  const int blocks_per_head = half / 8;
  const int n_blocks = (nh + nkv) * blocks_per_head;
  for (int idx = threadIdx.x; idx < n_blocks; idx += blockDim.x) {
    const int head = idx / blocks_per_head;
    const int t = idx - head * blocks_per_head;
    const uint4* xs = reinterpret_cast<const uint4*>(stage + head * hd) + 2 * t;
    const uint4 lo = xs[0], hi = xs[1];
    const __nv_bfloat162* pl = reinterpret_cast<const __nv_bfloat162*>(&lo);
    const __nv_bfloat162* ph = reinterpret_cast<const __nv_bfloat162*>(&hi);
    const float4 c0 = __ldg(reinterpret_cast<const float4*>(cs + 8 * t));
    const float4 c1 = __ldg(reinterpret_cast<const float4*>(cs + 8 * t) + 1);
    const float4 s0 = __ldg(reinterpret_cast<const float4*>(sn + 8 * t));
    const float4 s1 = __ldg(reinterpret_cast<const float4*>(sn + 8 * t) + 1);
    const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const float ss[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    uint4 o1, o2;
    uint32_t* p1 = reinterpret_cast<uint32_t*>(&o1);
    uint32_t* p2 = reinterpret_cast<uint32_t*>(&o2);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 a = __bfloat1622float2(pl[q]), b = __bfloat1622float2(ph[q]);
      const int j = 2 * q;
      // y1 = x1 c - x2 s (dim i), y2 = x2 c + x1 s (dim i + 64), each rounded
      p1[q] = pack_bf16(a.x * cc[j] - b.x * ss[j], a.y * cc[j + 1] - b.y * ss[j + 1]);
      p2[q] = pack_bf16(b.x * cc[j] + a.x * ss[j], b.y * cc[j + 1] + a.y * ss[j + 1]);
    }
    __nv_bfloat16* x = row + head * hd;
    reinterpret_cast<uint4*>(x + 8 * t)[0] = o1;
    reinterpret_cast<uint4*>(x + half + 8 * t)[0] = o2;
    if (head >= nh) {
      __nv_bfloat16* kd = k_pool + ((head - nh) * head_stride + cell) * hd;
      reinterpret_cast<uint4*>(kd + 8 * t)[0] = o1;
      reinterpret_cast<uint4*>(kd + half + 8 * t)[0] = o2;
    }
  }
  // v: 16-byte chunks, head-major pool ([kv_head][cell][hd])
  const int per_head = hd / 8;
  const uint4* vsrc = reinterpret_cast<const uint4*>(row + (nh + nkv) * hd);
  for (int j = threadIdx.x; j < nkv * per_head; j += blockDim.x) {
    const int kh = j / per_head;
    reinterpret_cast<uint4*>(v_pool + (kh * head_stride + cell) * hd)[j - kh * per_head] = vsrc[j];
  }
}

}  // namespace ds

extern "C" {

int ds_embed(const int32_t* tokens, int n_rows, const void* table, int hidden, void* out,
             int out_f32, ds_stream_t stream) {
  if (n_rows < 0 || hidden % 8) return DS_EINVAL;
  if (n_rows == 0) return DS_OK;
  ds::launch_pdl(ds::embed_kernel, dim3(n_rows), dim3(128), 0, (cudaStream_t)stream, tokens,
                 static_cast<const uint4*>(table), hidden / 8, out, out_f32);
  return (int)cudaGetLastError();
}

int ds_rmsnorm(const void* x, int x_f32, const int32_t* rows, int n_rows, int hidden,
               const void* w, float eps, void* out, ds_stream_t stream) {
  if (n_rows < 0 || hidden % 8 || hidden > 8 * 256 * 4) return DS_EINVAL;
  if (n_rows == 0) return DS_OK;
  ds::launch_pdl(ds::rmsnorm_kernel<256, 4>, dim3(n_rows), dim3(256), 0, (cudaStream_t)stream, x,
                 rows, hidden / 8, x_f32, static_cast<const uint4*>(w), eps,
                 static_cast<uint4*>(out));
  return (int)cudaGetLastError();
}

int ds_silu_mul(const void* gate_up, int n_rows, int ffn, void* out, ds_stream_t stream) {
  if (n_rows < 0 || ffn % 8) return DS_EINVAL;
  if (n_rows == 0) return DS_OK;
  const int chunks = ffn / 8;
  dim3 grid((chunks + 127) / 128, n_rows);
  ds::launch_pdl(ds::silu_mul_kernel, grid, dim3(128), 0, (cudaStream_t)stream,
                 static_cast<const uint4*>(gate_up), chunks, static_cast<uint4*>(out));
  return (int)cudaGetLastError();
}

int ds_rope_kv_store(void* qkv, int n_rows, const int32_t* row_seq, const int32_t* row_pos,
                     const int32_t* pos2cell, int64_t pos_stride, int n_heads, int n_kv_heads,
                     int head_dim, const float* rope_cos, const float* rope_sin, void* k_pool_l,
                     void* v_pool_l, int64_t kv_head_stride, ds_stream_t stream) {
  if (n_rows < 0 || head_dim != 128) return DS_EINVAL;
  if (n_rows == 0) return DS_OK;
  const int smem = (n_heads + n_kv_heads) * head_dim * 2;
  if (smem > 48 * 1024) return DS_EUNSUPPORTED;
  ds::launch_pdl(ds::rope_kv_store_kernel, dim3(n_rows), dim3(256), smem, (cudaStream_t)stream,
                 static_cast<__nv_bfloat16*>(qkv), row_seq, row_pos, pos2cell, pos_stride, n_heads,
                 n_kv_heads, head_dim, rope_cos, rope_sin, static_cast<__nv_bfloat16*>(k_pool_l),
                 static_cast<__nv_bfloat16*>(v_pool_l), kv_head_stride);
  return (int)cudaGetLastError();
}

}  // extern "C"
