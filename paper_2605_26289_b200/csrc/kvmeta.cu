// K4: paged KV store metadata - metadata-only aliasing (0 KV bytes moved).
//
// The host UnifiedKvCache mirror (kvcache.py:116-286 semantics: first-fit
// allocator, spans, refcounts) records one op per page-table mutation; a
// flush applies the whole op list here, strictly in order, inside one CTA
// (ops are short and few per iteration; ordering matters because a trimmed
// cell can be re-allocated to the same sequence in the same flush).
#include "../../include/deltaserve_b200.h"
#include "common.cuh"

namespace ds {

// Sequences outside [0, n_seqs) (host-only pressure in tests) are not
// mirrored; positions beyond pos_stride are never written.
//
// Order only matters between ops of the same sequence (its page-table row,
// its membership bits; a trimmed cell can be re-mapped to the same sequence in
// the same flush): warp w of the grid applies, in list order, every op of the
// sequences s with s % n_warps == w; membership words (32 sequences each) are
// updated with atomics, and the commutative counters - map_ref (exact
// mappings per cell, also when a sequence maps a cell twice, which one bit
// cannot represent) and trie_ref - with atomic adds from any warp.  Each CTA
// stages the op list through shared memory in 256-op chunks; a warp finds its
// ops with one ballot per 32.
constexpr int kApplyThreads = 256, kApplyChunk = 256;
__global__ void __launch_bounds__(kApplyThreads) kv_apply_kernel(
    const ds_kv_op* __restrict__ ops, int n_ops, int32_t* pos2cell, int64_t pos_stride, int n_seqs,
    uint32_t* member, int mask_words, int32_t* trie_ref, int32_t* map_ref) {
  __shared__ ds_kv_op s_ops[kApplyChunk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = gridDim.x * (kApplyThreads / 32), gw = blockIdx.x * (kApplyThreads / 32) + warp;
  for (int base = 0; base < n_ops; base += kApplyChunk) {
    const int nc = min(kApplyChunk, n_ops - base);
    __syncthreads();  // the previous chunk is consumed
    for (int i = threadIdx.x; i < nc; i += kApplyThreads) s_ops[i] = ops[base + i];
    __syncthreads();
    for (int b0 = 0; b0 < nc; b0 += 32) {
      bool mine = false;
      if (b0 + lane < nc) {
        const ds_kv_op& op = s_ops[b0 + lane];
        if (op.kind == DS_KV_TRIE_INC || op.kind == DS_KV_TRIE_DEC)
          mine = (base + b0 + lane) % nw == gw;
        else
          mine = op.seq >= 0 && op.seq < n_seqs && op.seq % nw == gw;
      }
      uint32_t m = __ballot_sync(0xffffffffu, mine);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const ds_kv_op op = s_ops[b0 + src];
        const uint32_t bit = 1u << (op.seq & 31);
        const int word = op.seq >> 5;
        switch (op.kind) {
          case DS_KV_MAP: {
            int32_t* row = pos2cell + static_cast<int64_t>(op.seq) * pos_stride + op.pos;
            for (int j = lane; j < op.len; j += 32) {
              const int32_t c = op.cell + j;
              if (op.pos + j < pos_stride) row[j] = c;
              atomicOr(member + static_cast<int64_t>(c) * mask_words + word, bit);
              if (map_ref) atomicAdd(map_ref + c, 1);
            }
            break;
          }
          case DS_KV_UNMAP:
            for (int j = lane; j < op.len; j += 32) {
              atomicAnd(member + static_cast<int64_t>(op.cell + j) * mask_words + word, ~bit);
              if (map_ref) atomicSub(map_ref + op.cell + j, 1);
            }
            break;
          case DS_KV_TRIE_INC:
            for (int j = lane; j < op.len; j += 32) atomicAdd(trie_ref + op.cell + j, 1);
            break;
          case DS_KV_TRIE_DEC:
            for (int j = lane; j < op.len; j += 32) atomicSub(trie_ref + op.cell + j, 1);
            break;
          case DS_KV_MAP_SCRATCH: {
            int32_t* row = pos2cell + static_cast<int64_t>(op.seq) * pos_stride + op.pos;
            for (int j = lane; j < op.len; j += 32)
              if (op.pos + j < pos_stride) row[j] = op.cell + j;
            break;
          }
          default:
            break;
        }
        __syncwarp();  // the next op of this warp's sequences sees these writes
      }
    }
  }
}

__global__ void kv_refcount_kernel(const uint32_t* __restrict__ member, int mask_words,
                                   const int32_t* __restrict__ trie_ref,
                                   const int32_t* __restrict__ map_ref, int64_t capacity,
                                   int32_t* refcnt, int32_t* occupancy) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int live = 0;
  if (c < capacity) {
    int r = trie_ref[c];
    if (map_ref) {
      r += map_ref[c];
    } else {
      const uint32_t* m = member + c * mask_words;
      for (int w = 0; w < mask_words; ++w) r += __popc(m[w]);
    }
    refcnt[c] = r;
    live = r > 0;
  }
  live = __syncthreads_count(live);
  if (threadIdx.x == 0 && live) atomicAdd(occupancy, live);
}

// Token-history writes (prompt uploads at admit, pending tokens before the
// n-gram matcher): segment i = {seq, start, len, src_offset}.
__global__ void hist_write_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ segs,
                                  int32_t* hist, int64_t pos_stride) {
  const int32_t* sg = segs + 4 * blockIdx.x;
  int32_t* dst = hist + static_cast<int64_t>(sg[0]) * pos_stride + sg[1];
  const int32_t* s = src + sg[3];
  for (int j = threadIdx.x; j < sg[2]; j += blockDim.x) dst[j] = s[j];
}

// one CTA per (pair, layer): K and V rows of every KV head (2 * nkv * hd bf16)
__global__ void kv_copy_cells_kernel(__nv_bfloat16* k_pool, __nv_bfloat16* v_pool, int nkv,
                                     int64_t head_stride, int hd, const int32_t* pairs) {
  const int i = blockIdx.x, l = blockIdx.y;
  const int64_t src = pairs[2 * i], dst = pairs[2 * i + 1];
  const int per_head = hd / 8;
  const int64_t layer = static_cast<int64_t>(l) * nkv * head_stride * hd;
  for (int j = threadIdx.x; j < 2 * nkv * per_head; j += blockDim.x) {
    const int kv = j / (nkv * per_head);
    const int rem = j - kv * nkv * per_head;
    const int h = rem / per_head, c = rem - h * per_head;
    __nv_bfloat16* pool = kv ? v_pool : k_pool;
    uint4* d = reinterpret_cast<uint4*>(pool + layer + (h * head_stride + dst) * hd) + c;
    const uint4* s = reinterpret_cast<const uint4*>(pool + layer + (h * head_stride + src) * hd) + c;
    *d = *s;
  }
}

// Prefix migration payload (dist.py): the K and V rows of n cells, all
// layers, packed as buf[L][2][nkv][n][hd] - one contiguous message per
// migrated prefix.  unpack = 1 scatters a received buffer straight into the
// freshly allocated cells (head-major pool [L][nkv][head_stride][hd]).
__global__ void kv_pack_cells_kernel(__nv_bfloat16* k_pool, __nv_bfloat16* v_pool, int nkv,
                                     int64_t head_stride, int hd, const int32_t* cells, int n,
                                     __nv_bfloat16* buf, int unpack) {
  const int i = blockIdx.x, l = blockIdx.y;
  const int64_t cell = cells[i];
  const int per_head = hd / 8;
  const int64_t layer = static_cast<int64_t>(l) * nkv * head_stride * hd;
  for (int j = threadIdx.x; j < 2 * nkv * per_head; j += blockDim.x) {
    const int kv = j / (nkv * per_head);
    const int rem = j - kv * nkv * per_head;
    const int h = rem / per_head, c = rem - h * per_head;
    __nv_bfloat16* pool = kv ? v_pool : k_pool;
    uint4* p = reinterpret_cast<uint4*>(pool + layer + (h * head_stride + cell) * hd) + c;
    uint4* b = reinterpret_cast<uint4*>(
                   buf + ((((static_cast<int64_t>(l) * 2 + kv) * nkv + h) * n + i) * hd)) + c;
    if (unpack)
      *p = *b;
    else
      *b = *p;
  }
}

}  // namespace ds

extern "C" {

int ds_kv_pack_cells(void* k_pool, void* v_pool, int layers, int n_kv_heads, int64_t head_stride,
                     int head_dim, const int32_t* cells, int n, void* buf, int unpack,
                     ds_stream_t stream) {
  if (n < 0 || head_dim % 8 || layers <= 0 || n_kv_heads <= 0) return DS_EINVAL;
  if (n == 0) return DS_OK;
  ds::kv_pack_cells_kernel<<<dim3(n, layers), 256, 0, (cudaStream_t)stream>>>(
      static_cast<__nv_bfloat16*>(k_pool), static_cast<__nv_bfloat16*>(v_pool), n_kv_heads,
      head_stride, head_dim, cells, n, static_cast<__nv_bfloat16*>(buf), unpack);
  return (int)cudaGetLastError();
}

int ds_kv_copy_cells(void* k_pool, void* v_pool, int layers, int n_kv_heads, int64_t head_stride,
                     int head_dim, const int32_t* pairs, int n, ds_stream_t stream) {
  if (n < 0 || head_dim % 8) return DS_EINVAL;
  if (n == 0) return DS_OK;
  ds::kv_copy_cells_kernel<<<dim3(n, layers), 256, 0, (cudaStream_t)stream>>>(
      static_cast<__nv_bfloat16*>(k_pool), static_cast<__nv_bfloat16*>(v_pool), n_kv_heads,
      head_stride, head_dim, pairs);
  return (int)cudaGetLastError();
}

int ds_kv_apply(const ds_kv_op* ops_dev, int n_ops, int32_t* pos2cell, int64_t pos_stride,
                int n_seqs, uint32_t* member, int mask_words, int32_t* trie_ref,
                int32_t* map_ref, ds_stream_t stream) {
  if (n_ops < 0 || mask_words <= 0 || n_seqs > 32 * mask_words) return DS_EINVAL;
  if (n_ops == 0) return DS_OK;
  // one warp per sequence up to 148 CTAs (8 warps each); at least one CTA
  // for the radix-only op lists of host-only sequences
  constexpr int kWarps = ds::kApplyThreads / 32;
  int blocks = (n_seqs + kWarps - 1) / kWarps;
  blocks = blocks < 1 ? 1 : blocks > 148 ? 148 : blocks;
  ds::kv_apply_kernel<<<blocks, ds::kApplyThreads, 0, (cudaStream_t)stream>>>(
      ops_dev, n_ops, pos2cell, pos_stride, n_seqs, member, mask_words, trie_ref, map_ref);
  return (int)cudaGetLastError();
}

int ds_hist_write(const int32_t* src, const int32_t* segs, int n_segs, int32_t* hist,
                  int64_t pos_stride, ds_stream_t stream) {
  if (n_segs < 0) return DS_EINVAL;
  if (n_segs == 0) return DS_OK;
  ds::hist_write_kernel<<<n_segs, 256, 0, (cudaStream_t)stream>>>(src, segs, hist, pos_stride);
  return (int)cudaGetLastError();
}

int ds_kv_refcount(const uint32_t* member, int mask_words, const int32_t* trie_ref,
                   const int32_t* map_ref, int64_t capacity, int32_t* refcnt_out,
                   int32_t* occupancy_out, ds_stream_t stream) {
  if (capacity <= 0 || mask_words <= 0) return DS_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t err = cudaMemsetAsync(occupancy_out, 0, sizeof(int32_t), s);
  if (err != cudaSuccess) return (int)err;
  const int blocks = static_cast<int>((capacity + 255) / 256);
  ds::kv_refcount_kernel<<<blocks, 256, 0, s>>>(member, mask_words, trie_ref, map_ref, capacity,
                                                refcnt_out, occupancy_out);
  return (int)cudaGetLastError();
}

}  // extern "C"
