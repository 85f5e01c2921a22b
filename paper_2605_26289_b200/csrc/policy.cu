// Integer hot kernels: FNV-1a, copy-model continuation scan (K2), prompt-lookup
// n-gram matcher (K1), row argmax + verify accept (K8).
//
// Reference semantics: deltaserve/_kernels/_native.pyx:18-119,
// engine.py:146-216, speculator.py:52-65 and 99-112.
#include "../../include/deltaserve_b200.h"
#include "common.cuh"
#include "internal.h"

namespace ds {

// ---------------------------------------------------------------------------
// FNV-1a over tokens / bytes: one thread per sequence (the recurrence is
// inherently sequential; sequences are independent).
// ---------------------------------------------------------------------------
__global__ void fnv_tokens_kernel(const int32_t* __restrict__ base, const int64_t* offsets,
                                  const int32_t* lengths, int n, int bits,
                                  const uint64_t* states_in, uint64_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t* p = base + offsets[i];
  const int len = lengths[i];
  if (bits == 64) {
    uint64_t h = states_in ? states_in[i] : kFnv64Offset;
    for (int j = 0; j < len; ++j) h = fnv64_token(h, __ldg(p + j));
    out[i] = h;
  } else {
    uint32_t h = states_in ? static_cast<uint32_t>(states_in[i]) : kFnv32Offset;
    for (int j = 0; j < len; ++j) h = fnv32_token(h, __ldg(p + j));
    out[i] = h;
  }
}

__global__ void fnv_bytes_kernel(const uint8_t* __restrict__ base, const int64_t* offsets,
                                 const int32_t* lengths, int n, int bits, uint64_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t* p = base + offsets[i];
  const int len = lengths[i];
  if (bits == 64) {
    uint64_t h = kFnv64Offset;
    for (int j = 0; j < len; ++j) h = (h ^ p[j]) * kFnv64Prime;
    out[i] = h;
  } else {
    uint32_t h = kFnv32Offset;
    for (int j = 0; j < len; ++j) h = (h ^ p[j]) * kFnv32Prime;
    out[i] = h;
  }
}

// ---------------------------------------------------------------------------
// K2 core: most recent earlier occurrence of the trailing mm-gram of
// tok[0:n].  Block-parallel right-to-left sweep in chunks of 4*blockDim
// candidate starts; the first chunk with a hit holds the answer (its max).
// Called by one whole CTA; returns e (or -1) to every thread.
// ---------------------------------------------------------------------------
template <int BLOCK>
DS_DEVICE int block_copy_continuation(const int32_t* __restrict__ tok, int n, int mm,
                                      int* s_best) {
  if (n <= mm || mm <= 0) return -1;
  const int g = n - mm;
  const int32_t first = __ldg(tok + g);
  constexpr int PER = 4;
  constexpr int CHUNK = BLOCK * PER;
  if (threadIdx.x == 0) *s_best = -1;
  __syncthreads();
  for (int hi = n - mm - 1; hi >= 0; hi -= CHUNK) {
    int found = -1;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int s = hi - (k * BLOCK + static_cast<int>(threadIdx.x));
      if (s >= 0 && found < 0 && __ldg(tok + s) == first) {
        int j = 1;
        while (j < mm && __ldg(tok + s + j) == __ldg(tok + g + j)) ++j;
        if (j == mm) found = s;  // k ascends => s descends: first hit is this thread's max
      }
    }
    if (found >= 0) atomicMax(s_best, found);
    __syncthreads();
    const int best = *s_best;
    if (best >= 0) return best + mm;
    __syncthreads();  // keep every thread's read of s_best before the next chunk
  }
  return -1;
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) copy_continuation_kernel(const int32_t* __restrict__ base,
                                                                  const int64_t* offsets,
                                                                  const int32_t* lengths, int mm,
                                                                  int32_t* e_out) {
  __shared__ int s_best;
  const int i = blockIdx.x;
  const int e = block_copy_continuation<BLOCK>(base + offsets[i], lengths[i], mm, &s_best);
  if (threadIdx.x == 0) e_out[i] = e;
}

// ---------------------------------------------------------------------------
// K1: longest suffix-anchored match (+ draft extraction), one CTA per slot.
// Candidate key = (length << 32) | e ; the max key is the reference's answer
// (longest first, then most recent, _native.pyx:104-117).
// ---------------------------------------------------------------------------
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) suffix_match_kernel(
    const int32_t* __restrict__ ring_base, const int64_t* ring_off, const int32_t* ring_len,
    const int32_t* __restrict__ tail_base, const int64_t* tail_off, const int32_t* tail_len,
    int min_len, const int32_t* caps, int max_draft, int32_t* e_out, int32_t* len_out,
    int32_t* draft_out, int32_t* draft_len_out) {
  __shared__ unsigned long long s_key[BLOCK / 32];
  const int slot = blockIdx.x;
  const int32_t* ring = ring_base + ring_off[slot];
  const int32_t* tail = tail_base + tail_off[slot];
  const int n = ring_len[slot];
  const int t = tail_len[slot];
  unsigned long long key = 0;
  if (!(t < min_len || n <= min_len || min_len <= 0)) {
    const int gs = t - min_len;
    const int32_t first = __ldg(tail + gs);
    for (int start = n - min_len - 1 - static_cast<int>(threadIdx.x); start >= 0; start -= BLOCK) {
      if (__ldg(ring + start) != first) continue;
      int j = 1;
      while (j < min_len && __ldg(ring + start + j) == __ldg(tail + gs + j)) ++j;
      if (j < min_len) continue;
      const int e = start + min_len;
      const int max_len = t < e ? t : e;
      int len = min_len;
      while (len < max_len && __ldg(ring + e - len - 1) == __ldg(tail + t - len - 1)) ++len;
      const unsigned long long k =
          (static_cast<unsigned long long>(len) << 32) | static_cast<unsigned int>(e);
      key = k > key ? k : key;
    }
  }
  key = warp_max(key);
  if ((threadIdx.x & 31) == 0) s_key[threadIdx.x >> 5] = key;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long k = threadIdx.x < BLOCK / 32 ? s_key[threadIdx.x] : 0ull;
    k = warp_max(k);
    const int e = k ? static_cast<int>(k & 0xFFFFFFFFull) : -1;
    const int len = k ? static_cast<int>(k >> 32) : 0;
    if (threadIdx.x == 0) {
      e_out[slot] = e;
      len_out[slot] = len;
    }
    if (caps) {
      int take = 0;
      if (e >= 0 && len >= min_len) {
        take = caps[slot];
        take = take < max_draft ? take : max_draft;
        take = take < n - e ? take : n - e;
        take = take > 0 ? take : 0;
      }
      for (int j = threadIdx.x; j < take; j += 32) draft_out[slot * max_draft + j] = ring[e + j];
      if (threadIdx.x == 0) draft_len_out[slot] = take;
    }
  }
}

// ---------------------------------------------------------------------------
// K8: argmax over fp32 rows, lowest index wins ties (np.argmax semantics).
// ---------------------------------------------------------------------------
DS_DEVICE void argmax_merge(float& v, int& i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

template <int BLOCK>
DS_DEVICE int block_argmax(const float* __restrict__ row, int vocab) {
  __shared__ float s_v[BLOCK / 32];
  __shared__ int s_i[BLOCK / 32];
  float best = -INFINITY;
  int bi = 0x7fffffff;
  const bool vec = (vocab % 4 == 0) && ((reinterpret_cast<uintptr_t>(row) & 15) == 0);
  if (vec) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    for (int j = threadIdx.x; j < vocab / 4; j += BLOCK) {
      const float4 v = __ldg(r4 + j);
      argmax_merge(best, bi, v.x, 4 * j);
      argmax_merge(best, bi, v.y, 4 * j + 1);
      argmax_merge(best, bi, v.z, 4 * j + 2);
      argmax_merge(best, bi, v.w, 4 * j + 3);
    }
  } else {
    for (int j = threadIdx.x; j < vocab; j += BLOCK) argmax_merge(best, bi, __ldg(row + j), j);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    argmax_merge(best, bi, v2, i2);
  }
  if ((threadIdx.x & 31) == 0) {
    s_v[threadIdx.x >> 5] = best;
    s_i[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < BLOCK / 32 ? s_v[threadIdx.x] : -INFINITY;
    bi = threadIdx.x < BLOCK / 32 ? s_i[threadIdx.x] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_merge(best, bi, v2, i2);
    }
  }
  return bi;  // valid in warp 0
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) argmax_kernel(const float* __restrict__ logits, int vocab,
                                                       int32_t* out) {
  const int r = blockIdx.x;
  const int bi = block_argmax<BLOCK>(logits + static_cast<size_t>(r) * vocab, vocab);
  if (threadIdx.x == 0) out[r] = bi;
}

// ---------------------------------------------------------------------------
// Forward-time token policy.
//   row hashes: FNV-1a64 of hist[:upto] for each sampled row, extended from
//   the entry's committed-prefix state (hash_in covers hist[:past]).
//   policy:     copy rule over the full preceding sequence, else hash mod V
//               (engine.py:205-213); or argmax of the real logits.
//   accept:     first mismatch against the drafts (speculator.py:104-112).
// ---------------------------------------------------------------------------
__global__ void row_hash_kernel(const ds_entry* entries, int n_entries, const int32_t* hist,
                                int64_t stride, uint64_t* row_hash) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_entries) return;
  const ds_entry en = entries[e];
  const int32_t* h = hist + static_cast<int64_t>(en.seq) * stride;
  uint64_t st = en.hash_in;
  // sampled row r (0-based within the entry's outputs) has preceding length
  // upto = past + q_len - n_out + r + 1
  const int first_upto = en.past + en.q_len - en.n_out + 1;
  int pos = en.past;
  for (int r = 0; r < en.n_out; ++r) {
    const int upto = first_upto + r;
    for (; pos < upto; ++pos) st = fnv64_token(st, __ldg(h + pos));
    row_hash[en.out_start + r] = st;
  }
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) token_policy_kernel(
    const ds_entry* entries, int n_entries, const int32_t* hist, int64_t stride,
    const uint64_t* row_hash, const float* logits, unsigned long long* amax, int model_vocab,
    int policy, int mm, int policy_vocab, int32_t* out_tok, int32_t* out_src) {
  __shared__ int s_best;
  pdl_wait();
  pdl_trigger();
  const int o = blockIdx.x;
  int ei = 0;
  while (ei + 1 < n_entries && entries[ei + 1].out_start <= o) ++ei;
  const ds_entry en = entries[ei];
  const int r = o - en.out_start;
  const int upto = en.past + en.q_len - en.n_out + r + 1;
  if (policy == DS_POLICY_COPY) {
    const int32_t* h = hist + static_cast<int64_t>(en.seq) * stride;
    const int e = block_copy_continuation<BLOCK>(h, upto, mm, &s_best);
    if (threadIdx.x == 0) {
      if (e >= 0) {
        out_tok[o] = __ldg(h + e);
        out_src[o] = e;
      } else {
        out_tok[o] = static_cast<int32_t>(row_hash[o] % static_cast<uint64_t>(policy_vocab));
        out_src[o] = -1;
      }
    }
  } else if (amax) {  // argmax fused into the LM head's epilogue
    if (threadIdx.x == 0) {
      out_tok[o] = argmax_key_index(amax[o]);
      out_src[o] = -1;
    }
  } else {
    const int bi = block_argmax<BLOCK>(logits + static_cast<size_t>(o) * model_vocab, model_vocab);
    if (threadIdx.x == 0) {
      out_tok[o] = bi;
      out_src[o] = -1;
    }
  }
  if (amax && threadIdx.x == 0) amax[o] = 0;  // re-arm for the next forward
}

__global__ void verify_accept_kernel(const ds_entry* entries, int n_entries, const int32_t* hist,
                                     int64_t stride, const int32_t* out_tok, int32_t* out_accept) {
  pdl_wait();
  pdl_trigger();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_entries) return;
  const ds_entry en = entries[e];
  int acc = 0;
  if (en.kind == DS_ENTRY_VERIFY) {
    // drafts d_s sit at batch rows 1..k, i.e. hist[past + 1 + s]
    const int32_t* h = hist + static_cast<int64_t>(en.seq) * stride + en.past + 1;
    while (acc < en.n_draft && out_tok[en.out_start + acc] == h[acc]) ++acc;
  }
  out_accept[e] = acc;
}

void launch_token_policy(const ds_forward_args* a, const ds_kv_store* kv, uint64_t* row_hash,
                         uint64_t* amax, int model_vocab, cudaStream_t hash_stream,
                         cudaStream_t stream) {
  (void)hash_stream;
  constexpr int B = 256;
  launch_pdl(token_policy_kernel<B>, dim3(a->n_out), dim3(B), 0, stream, a->entries,
             a->n_entries, kv->hist, kv->pos_stride, (const uint64_t*)row_hash,
             (const float*)a->logits, (unsigned long long*)amax, model_vocab, a->policy, a->copy_min_match, a->policy_vocab,
             a->out_tok, a->out_src);
  launch_pdl(verify_accept_kernel, dim3((a->n_entries + 63) / 64), dim3(64), 0, stream,
             a->entries, a->n_entries, (const int32_t*)kv->hist, kv->pos_stride,
             (const int32_t*)a->out_tok, a->out_accept);
}

// next proposal, fused into the forward: the bonus token into the history and
// the suffix-match ring of every decode / verify entry as the scheduler will
// hold it after committing (accepted drafts + bonus)
__global__ void next_draft_prep_kernel(const ds_entry* __restrict__ entries, int n_entries,
                                       const int32_t* __restrict__ out_tok,
                                       const int32_t* __restrict__ out_accept, int32_t* hist,
                                       int64_t pos_stride, int window, int cap, int64_t* ring_off,
                                       int32_t* ring_len, int32_t* caps) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_entries) return;
  const ds_entry en = entries[e];
  int n = 0;
  if (en.kind == DS_ENTRY_DECODE || en.kind == DS_ENTRY_VERIFY) {
    const int acc = en.kind == DS_ENTRY_VERIFY ? out_accept[e] : 0;
    n = en.past + acc + 2;  // committed tokens incl. the pending bonus
    hist[static_cast<int64_t>(en.seq) * pos_stride + n - 1] = out_tok[en.out_start + acc];
  } else if (en.kind == DS_ENTRY_PREFILL && en.n_draft < 0) {
    // the chunk that ends the prompt: the first decode step's proposal
    n = en.past + en.q_len + 1;  // the prompt + its sampled token
    hist[static_cast<int64_t>(en.seq) * pos_stride + n - 1] = out_tok[en.out_start];
  }
  const int ln = n < window ? n : window;
  ring_off[e] = static_cast<int64_t>(en.seq) * pos_stride + n - ln;
  ring_len[e] = ln;
  caps[e] = cap;
}

void launch_next_draft(const ds_forward_args* a, const ds_kv_store* kv, cudaStream_t stream) {
  const int n = a->n_entries, cap = a->next_cap;
  int32_t* base = a->next_out;
  int32_t* e_out = base;
  int32_t* len_out = base + n;
  int32_t* dlen_out = base + 2 * n;
  int32_t* draft_out = base + 3 * n;
  int32_t* scratch = base + 3 * n + n * cap;
  int64_t* ring_off = reinterpret_cast<int64_t*>(scratch + (reinterpret_cast<uintptr_t>(scratch) & 4 ? 1 : 0));
  int32_t* ring_len = reinterpret_cast<int32_t*>(ring_off + n);
  int32_t* caps = ring_len + n;
  next_draft_prep_kernel<<<(n + 63) / 64, 64, 0, stream>>>(
      a->entries, n, a->out_tok, a->out_accept, kv->hist, kv->pos_stride, a->next_window, cap,
      ring_off, ring_len, caps);
  suffix_match_kernel<128><<<n, 128, 0, stream>>>(kv->hist, ring_off, ring_len, kv->hist, ring_off,
                                                  ring_len, a->next_min_match, caps, cap, e_out,
                                                  len_out, draft_out, dlen_out);
}

void launch_row_hash(const ds_forward_args* a, const ds_kv_store* kv, uint64_t* row_hash,
                     cudaStream_t stream) {
  row_hash_kernel<<<(a->n_entries + 31) / 32, 32, 0, stream>>>(a->entries, a->n_entries, kv->hist,
                                                                kv->pos_stride, row_hash);
}

}  // namespace ds

using namespace ds;

extern "C" {

int ds_fnv1a_tokens(const int32_t* base, const int64_t* offsets, const int32_t* lengths, int n,
                    int bits, const uint64_t* states_in, uint64_t* out, ds_stream_t stream) {
  if (n < 0 || (bits != 32 && bits != 64)) return DS_EINVAL;
  if (n == 0) return DS_OK;
  fnv_tokens_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(base, offsets, lengths, n,
                                                                       bits, states_in, out);
  return (int)cudaGetLastError();
}

int ds_fnv1a_bytes(const uint8_t* base, const int64_t* offsets, const int32_t* lengths, int n,
                   int bits, uint64_t* out, ds_stream_t stream) {
  if (n < 0 || (bits != 32 && bits != 64)) return DS_EINVAL;
  if (n == 0) return DS_OK;
  fnv_bytes_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(base, offsets, lengths, n,
                                                                      bits, out);
  return (int)cudaGetLastError();
}

int ds_copy_continuation(const int32_t* base, const int64_t* offsets, const int32_t* lengths,
                         int n, int min_match, int32_t* e_out, ds_stream_t stream) {
  if (n < 0) return DS_EINVAL;
  if (n == 0) return DS_OK;
  copy_continuation_kernel<256>
      <<<n, 256, 0, (cudaStream_t)stream>>>(base, offsets, lengths, min_match, e_out);
  return (int)cudaGetLastError();
}

int ds_longest_suffix_match(const int32_t* ring_base, const int64_t* ring_off,
                            const int32_t* ring_len, const int32_t* tail_base,
                            const int64_t* tail_off, const int32_t* tail_len, int n, int min_len,
                            const int32_t* caps, int max_draft, int32_t* e_out, int32_t* len_out,
                            int32_t* draft_out, int32_t* draft_len_out, ds_stream_t stream) {
  if (n < 0) return DS_EINVAL;
  if (caps && (!draft_out || !draft_len_out || max_draft <= 0)) return DS_EINVAL;
  if (n == 0) return DS_OK;
  suffix_match_kernel<128><<<n, 128, 0, (cudaStream_t)stream>>>(
      ring_base, ring_off, ring_len, tail_base, tail_off, tail_len, min_len, caps, max_draft,
      e_out, len_out, draft_out, draft_len_out);
  return (int)cudaGetLastError();
}

int ds_argmax(const float* logits, int n_rows, int vocab, int32_t* out, ds_stream_t stream) {
  if (n_rows < 0 || vocab <= 0) return DS_EINVAL;
  if (n_rows == 0) return DS_OK;
  argmax_kernel<512><<<n_rows, 512, 0, (cudaStream_t)stream>>>(logits, vocab, out);
  return (int)cudaGetLastError();
}

uint64_t ds_host_fnv1a64_tokens(const int32_t* tokens, int64_t n, uint64_t state) {
  uint64_t h = state;
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t t = static_cast<uint32_t>(tokens[i]);
    h = (h ^ (t & 0xFFu)) * kFnv64Prime;
    h = (h ^ ((t >> 8) & 0xFFu)) * kFnv64Prime;
    h = (h ^ ((t >> 16) & 0xFFu)) * kFnv64Prime;
    h = (h ^ (t >> 24)) * kFnv64Prime;
  }
  return h;
}

uint32_t ds_host_fnv1a32_tokens(const int32_t* tokens, int64_t n, uint32_t state) {
  uint32_t h = state;
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t t = static_cast<uint32_t>(tokens[i]);
    h = (h ^ (t & 0xFFu)) * kFnv32Prime;
    h = (h ^ ((t >> 8) & 0xFFu)) * kFnv32Prime;
    h = (h ^ ((t >> 16) & 0xFFu)) * kFnv32Prime;
    h = (h ^ (t >> 24)) * kFnv32Prime;
  }
  return h;
}

}  // extern "C"
