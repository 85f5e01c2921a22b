/*
 * deltaserve_b200 - C ABI of the B200-native delta-only inference hot path.
 *
 * Plain pointers and sizes only (no torch types).  Every device pointer is a
 * CUDA global-memory address; `stream` is a cudaStream_t (NULL = legacy).
 * Return value: 0 = ok, < 0 = argument error (DS_E*), > 0 = cudaError_t or
 * (1000 + cublasStatus_t).  Kernels never allocate and are stream ordered;
 * capacity checks stay on the host (reference kvcache.py:116-118) so no
 * kernel fails for capacity.
 *
 * Each entry point cites the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/deltaserve/).
 */
#ifndef DELTASERVE_B200_H
#define DELTASERVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* ds_stream_t;

#define DS_OK 0
#define DS_EINVAL (-1)
#define DS_EUNSUPPORTED (-2)
#define DS_EWORKSPACE (-3)

int ds_abi_version(void);
const char* ds_status_string(int status);

/* ------------------------------------------------------------------------
 * Integer kernels: batched device versions of deltaserve._kernels
 * (_kernels/__init__.py:21-73, _native.pyx:18-119).  Sequence i lives at
 * base + offsets[i] with lengths[i] int32 tokens.
 * ---------------------------------------------------------------------- */

/* fnv1a32_tokens / fnv1a64_tokens (_native.pyx:36-59), tokens hashed as 4 LE
 * bytes; states_in (nullable) seeds each sequence (the `state=` argument).
 * bits = 32 or 64; out[i] holds the hash (32-bit results zero-extended). */
int ds_fnv1a_tokens(const int32_t* base, const int64_t* offsets, const int32_t* lengths, int n,
                    int bits, const uint64_t* states_in, uint64_t* out, ds_stream_t stream);

/* fnv1a32_bytes / fnv1a64_bytes (_native.pyx:18-33). */
int ds_fnv1a_bytes(const uint8_t* base, const int64_t* offsets, const int32_t* lengths, int n,
                   int bits, uint64_t* out, ds_stream_t stream);

/* copy_continuation (_native.pyx:62-81): e_out[i] = index after the most
 * recent earlier occurrence of the trailing min_match-gram, or -1. */
int ds_copy_continuation(const int32_t* base, const int64_t* offsets, const int32_t* lengths,
                         int n, int min_match, int32_t* e_out, ds_stream_t stream);

/* K1 prompt-lookup n-gram matcher: longest_suffix_match (_native.pyx:84-119)
 * for n slots at once, optionally fused with lookup_ngram's draft extraction
 * (speculator.py:52-65): when caps != NULL, draft_out[i*max_draft + j] =
 * ring[e + j] for j < draft_len_out[i] = min(caps[i], max_draft, len - e)
 * (0 when no match or caps[i] <= 0). tail_base may equal ring_base. */
int ds_longest_suffix_match(const int32_t* ring_base, const int64_t* ring_off,
                            const int32_t* ring_len, const int32_t* tail_base,
                            const int64_t* tail_off, const int32_t* tail_len, int n, int min_len,
                            const int32_t* caps, int max_draft, int32_t* e_out, int32_t* len_out,
                            int32_t* draft_out, int32_t* draft_len_out, ds_stream_t stream);

/* Host-side FNV-1a used by the scheduler's own bookkeeping (Slot.prefix_hash
 * scheduler.py:237/687/715 and _window_hash :489-490) - the same host work the
 * reference scheduler does; not part of the device compute path. */
uint64_t ds_host_fnv1a64_tokens(const int32_t* tokens, int64_t n, uint64_t state);
uint32_t ds_host_fnv1a32_tokens(const int32_t* tokens, int64_t n, uint32_t state);

/* ------------------------------------------------------------------------
 * K4: paged KV store metadata (UnifiedKvCache kvcache.py:116-286).
 * pos2cell[seq*pos_stride + p] = physical cell of logical position p;
 * member[cell*mask_words + seq/32] bit seq%32 = sequence membership;
 * trie_ref[cell] = references held by radix nodes (radix.py:158-159, 184);
 * map_ref[cell] (optional) = page-table mappings of the cell, exact also when
 * a sequence maps one cell twice (one membership bit cannot count that).
 * Ops of one sequence apply in list order (one warp per sequence, across the
 * grid); 0 KV bytes move.
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t kind; /* DS_KV_MAP: pos2cell[seq][pos+i] = cell+i, set member bit;
                   DS_KV_UNMAP: clear member bit `seq` on cells [cell, cell+len);
                   DS_KV_TRIE_INC / DS_KV_TRIE_DEC: trie_ref[cell+i] += / -= 1 */
  int32_t seq;
  int32_t pos;
  int32_t cell;
  int32_t len;
} ds_kv_op;
#define DS_KV_MAP 0
#define DS_KV_UNMAP 1
#define DS_KV_TRIE_INC 2
#define DS_KV_TRIE_DEC 3
#define DS_KV_MAP_SCRATCH 4 /* pos2cell only (batched verify rows live in scratch cells
                               until the host knows the accept count) */

int ds_kv_apply(const ds_kv_op* ops_dev, int n_ops, int32_t* pos2cell, int64_t pos_stride,
                int n_seqs, uint32_t* member, int mask_words, int32_t* trie_ref,
                int32_t* map_ref /* nullable */, ds_stream_t stream);

/* Token-history writes: segment i = {seq, start, len, src_offset} copies
 * src[src_offset : src_offset+len] to hist[seq*pos_stride + start ...]
 * (prompt upload at admission; pending tokens before the n-gram matcher). */
int ds_hist_write(const int32_t* src, const int32_t* segs, int n_segs, int32_t* hist,
                  int64_t pos_stride, ds_stream_t stream);

/* Copy all layers' K and V rows of cell src[i] to cell dst[i] (pairs int32
 * [n][2]) in a head-major pool; used to move accepted verify rows from scratch
 * cells into the cells the reference allocator assigns. */
int ds_kv_copy_cells(void* k_pool, void* v_pool, int layers, int n_kv_heads, int64_t head_stride,
                     int head_dim, const int32_t* pairs, int n, ds_stream_t stream);

/* Prefix migration payload (multi-GPU): pack the K and V rows of
 * n cells (all layers) into buf [L][2][nkv][n][hd] bf16 (unpack = 0), or
 * scatter a received buffer into the cells (unpack = 1).  The reference is
 * single-GPU; the receiving side replaces the re-prefill a
 * radix miss would cost (scheduler.py:422-480 _admit). */
int ds_kv_pack_cells(void* k_pool, void* v_pool, int layers, int n_kv_heads, int64_t head_stride,
                     int head_dim, const int32_t* cells, int n, void* buf, int unpack,
                     ds_stream_t stream);

/* Derived refcount (map_ref + trie_ref, or popcount(member) + trie_ref when
 * map_ref is NULL) and occupancy (cells with refcount > 0) - the device view
 * of kvcache.py:91-100, 185-187. */
int ds_kv_refcount(const uint32_t* member, int mask_words, const int32_t* trie_ref,
                   const int32_t* map_ref, int64_t capacity, int32_t* refcnt_out,
                   int32_t* occupancy_out, ds_stream_t stream);

/* ------------------------------------------------------------------------
 * Model forward: the device realisation of MockEngine.forward
 * (engine.py:268-281) + LogitsBatch argmax/copy_source (engine.py:196-216)
 * + the verify accept loop (speculator.py:99-112), for a whole batch of plan
 * entries (scheduler.py:674-772) in one call.
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab;
  float rms_eps;
  const void* embed;      /* bf16 [vocab][hidden] */
  const void* attn_norm;  /* bf16 [L][hidden] */
  const void* wqkv;       /* bf16 [L][(nh+2nkv)*hd][hidden]; inside each q and k head
                           * the rows are RoPE-pair interleaved (hd = 128): row
                           * 16t+j is dim 8t+j (j<8) or 64+8t+j-8 (j>=8), so a
                           * 16-row tile holds 8 rotation pairs; v rows in order */
  const void* wo;         /* bf16 [L][hidden][nh*hd] */
  const void* mlp_norm;   /* bf16 [L][hidden] */
  const void* w_gate_up;  /* bf16 [L][2*ffn][hidden]: 8-row blocks, gate units 8b..8b+7
                           * then up units 8b..8b+7 (row 16b+j: j<8 gate, else up) */
  const void* w_down;     /* bf16 [L][hidden][ffn] */
  const void* final_norm; /* bf16 [hidden] */
  const void* lm_head;    /* bf16 [vocab][hidden] */
  const float* rope_cos;  /* f32 [rope_max_pos][hd/2] */
  const float* rope_sin;
  int32_t rope_max_pos;
} ds_model;

typedef struct {
  void* k_pool; /* bf16 [L][nkv][capacity][hd] (head-major: a run of cells is contiguous) */
  void* v_pool;
  int64_t capacity;
  int32_t* pos2cell; /* [n_seqs][pos_stride] */
  int32_t* hist;     /* [n_seqs][pos_stride] token history */
  int64_t pos_stride;
  int32_t n_seqs;
} ds_kv_store;

#define DS_ENTRY_PREFILL 0 /* sample the last row (scheduler.py:721-723) */
#define DS_ENTRY_DECODE 1  /* one row (scheduler.py:762-772) */
#define DS_ENTRY_VERIFY 2  /* rows [last, d0..dk-1]; accept + bonus (speculator.py:77-113) */

typedef struct {
  int32_t seq;       /* sequence id (row of pos2cell / hist) */
  int32_t past;      /* cells already resident before this batch (context length) */
  int32_t q_len;     /* batch rows */
  int32_t q_start;   /* first packed row */
  int32_t kind;      /* DS_ENTRY_* */
  int32_t n_draft;   /* k for VERIFY; -1 on the PREFILL chunk that ends a prompt: the
                        next proposal (ds_forward_args.next_*) follows its sampled token */
  int32_t out_start; /* first output (sampled) row */
  int32_t n_out;     /* sampled rows: 1 (prefill/decode) or k+1 (verify) */
  uint64_t hash_in;  /* FNV-1a64 of the sequence's first `past` tokens */
} ds_entry;

#define DS_POLICY_COPY 0   /* reference copy-model token rule (engine.py:196-216) */
#define DS_POLICY_ARGMAX 1 /* greedy argmax of the real logits, lowest id on ties */

typedef struct {
  int32_t n_entries, n_rows, n_out;
  int32_t policy, copy_min_match, policy_vocab;
  const ds_entry* entries_host; /* host copy (launch shapes) */
  const ds_entry* entries;      /* device copy */
  const int32_t* tokens;        /* device [n_rows] packed batch tokens */
  const int32_t* row_seq;       /* device [n_rows] */
  const int32_t* row_pos;       /* device [n_rows] absolute positions */
  const int32_t* out_rows;      /* device [n_out] packed row of each sampled row */
  int32_t* out_tok;             /* device [n_out] */
  int32_t* out_src;             /* device [n_out] copy source or -1 */
  int32_t* out_accept;          /* device [n_entries] accepted drafts (VERIFY) */
  float* logits;                /* device [n_out][vocab] fp32 */
  void* workspace;               /* zero-initialised once, then reused across calls */
  size_t workspace_bytes;
  /* Next prompt-lookup proposal computed in the same launch (0 = off).  For
   * every DECODE / VERIFY entry the sampled bonus token is written to the
   * history at its position past + accepted + 1, and the longest-suffix match
   * (speculator.py:52-65) runs over the last next_window tokens of the
   * history as the scheduler will hold it after committing: next_out[n_entries
   * x (3 + next_cap)] = e[n], len[n], draft_len[n], drafts[n][next_cap], then
   * int32 scratch[4n + 2].  A later proposal with cap <= next_cap is its prefix. */
  int32_t next_window, next_min_match, next_cap;
  int32_t* next_out;
  /* 1: store the fp32 logits [n_out][vocab]; 0: no logits materialisation -
   * when n_out <= 32 the LM head's epilogue reduces each row to its argmax
   * (DS_POLICY_ARGMAX reads that, the copy policy ignores it); larger n_out
   * still use `logits` as scratch.  The argmax policy's result is the same
   * either way (lowest id on ties). */
  int32_t logits_out;
} ds_forward_args;

size_t ds_forward_workspace_bytes(const ds_model* model, int max_rows, int max_out,
                                  int max_entries);
int ds_model_forward(const ds_model* model, const ds_kv_store* kv, const ds_forward_args* args,
                     ds_stream_t stream);

/* ------------------------------------------------------------------------
 * Individual layer kernels (exported for parity tests and microbenchmarks).
 * ---------------------------------------------------------------------- */

/* K5: RoPE (rotate-half, cos/sin table) on q (in place in qkv, written back in
 * plain dim order) and k; store k,v rows into the layer's head-major cell pool
 * ([kv_head][cell][head_dim], kv_head_stride = cells per head) at
 * pos2cell[row_seq][row_pos].  q/k head columns of qkv arrive in the wqkv
 * RoPE-pair interleaved order (ds_model); head_dim 128. */
int ds_rope_kv_store(void* qkv, int n_rows, const int32_t* row_seq, const int32_t* row_pos,
                     const int32_t* pos2cell, int64_t pos_stride, int n_heads, int n_kv_heads,
                     int head_dim, const float* rope_cos, const float* rope_sin, void* k_pool_l,
                     void* v_pool_l, int64_t kv_head_stride, ds_stream_t stream);

/* K6/K7 attention over the paged store for a batch of entries.  q is the
 * roped qkv buffer ([n_rows][(nh+2nkv)*hd], q heads first), out is
 * [n_rows][nh*hd] bf16.  Causal over absolute positions. impl: 0 = auto,
 * 1 = split-KV decode/verify kernel (K7), 2 = tcgen05 delta-prefill (K6). */
size_t ds_attention_workspace_bytes(int n_rows, int n_entries, int n_heads, int head_dim);
int ds_attention(const void* qkv, const ds_entry* entries_host, const ds_entry* entries_dev,
                 int n_entries, int n_rows, const void* k_pool_l, const void* v_pool_l,
                 int64_t kv_head_stride, const int32_t* pos2cell, int64_t pos_stride,
                 int n_heads, int n_kv_heads,
                 int head_dim, float scale, void* out, void* workspace, size_t workspace_bytes,
                 int impl, ds_stream_t stream);

/* RMSNorm of rows (nullable = identity) of the bf16 (x_f32=0) or fp32 residual
 * stream -> bf16: out = x * rsqrt(mean(x^2) + eps) * w, fp32 math. */
int ds_rmsnorm(const void* x, int x_f32, const int32_t* rows, int n_rows, int hidden,
               const void* w, float eps, void* out, ds_stream_t stream);
/* act[r][f] = silu(gate f) * up f from a gate|up row in the interleaved
 * w_gate_up layout (ds_model). */
int ds_silu_mul(const void* gate_up, int n_rows, int ffn, void* out, ds_stream_t stream);
int ds_embed(const int32_t* tokens, int n_rows, const void* table, int hidden, void* out,
             int out_f32, ds_stream_t stream);
/* Skinny GEMM for decode/verify row counts (M <= 32): Y[M][N] (+)= X[M][K] .
 * W[N][K]^T, bf16 in, fp32 accumulate, Y bf16 (y_f32=0) or fp32; accumulate=1
 * adds into Y (fused residual).  N % 16 == 0, K % 256 == 0.  Weight-streaming,
 * HBM-bound; replaces cuBLAS for the engine's decode/verify projections. */
int ds_gemm_skinny(const void* X, const void* W, void* Y, int M, int N, int K, int y_f32,
                   int accumulate, ds_stream_t stream);

/* Epilogue fusions of the skinny GEMM (the decode forward's elementwise
 * kernels folded into the projections; see gemm_skinny.cu).  An "ss buffer"
 * is uint64 [32]: per-row sums of squares in 2^-24 fixed point (integer
 * atomics, so the sum is independent of CTA order).
 *  ss_out/h_out/h_w: residual producer (y_f32 = 1) - adds the rows' sums of
 *      y^2 into ss_out (which must start at zero); h_out[m][n] =
 *      bf16(y[m][n] * h_w[n]) (optional).
 *  ss_zero: an ss buffer to clear (after the kernel's dependency wait) - the
 *      forward alternates two buffers, each producer clearing the other.
 *  row_ss/eps: norm consumer - row m of the product is scaled by
 *      rsqrt(row_ss[m] * 2^-24 / K + eps) (X holds bf16(x * norm_w)).
 *  swiglu: W rows are gate/up interleaved in 8-row blocks (see ds_model);
 *      Y = bf16 silu(gate) * up [M][N/2].
 *  rope: W = wqkv (pair-interleaved q/k rows, see ds_model; head_dim 128):
 *      q heads are rotated into Y [M][N] (plain dim order, k/v columns of Y
 *      untouched), k heads rotated and v copied into the layer's head-major
 *      pools at cell pos2cell[row_seq[m]][row_pos[m]] - the K5 kernel folded
 *      into the projection. */
#define DS_SKINNY_SS_WORDS 32
typedef struct {
  const uint64_t* row_ss;
  float eps;
  uint64_t* ss_out;
  uint64_t* ss_zero;
  void* h_out;
  const void* h_w;
  int32_t swiglu;
  int32_t rope;
  int32_t n_heads, n_kv_heads;
  const int32_t* row_seq;
  const int32_t* row_pos;
  const int32_t* pos2cell;
  int64_t pos_stride;
  const float* rope_cos; /* f32 [max_pos][64] */
  const float* rope_sin;
  void* k_pool_l;
  void* v_pool_l;
  int64_t kv_head_stride;
  /* the next kernel's first weight bytes: the CTAs of the last wave pull
   * [l2_next, l2_next + l2_next_bytes) into L2 once their own weight stream
   * is issued, so HBM stays busy across the kernel boundary (0 = none) */
  const void* l2_next;
  int64_t l2_next_bytes;
  /* fused row argmax (the LM head): argmax_out[m] = max over the product's
   * columns n of (ordered(y[m][n]) << 32) | (0xFFFFFFFF - n), i.e. the largest
   * value and the lowest column on ties (np.argmax); the caller zeroes it
   * before the launch.  Y may then be NULL: no product is stored (needs
   * y_f32 = 1, accumulate = 0, no other fusion). */
  uint64_t* argmax_out;
  /* bytes every CTA pulls into L2 (its equal share) BEFORE the dependency
   * wait - for a projection launched early beside a latency-bound kernel
   * (the decode attention), whose HBM would otherwise idle (0 = none) */
  const void* l2_pre;
  int64_t l2_pre_bytes;
} ds_skinny_epi;

int ds_gemm_skinny_ex(const void* X, const void* W, void* Y, int M, int N, int K, int y_f32,
                      int accumulate, const ds_skinny_epi* epi, ds_stream_t stream);

/* K10: persistent stream-K projection GEMM on tcgen05/TMEM for prefill chunks
 * and batched plans (any T): Y[T][N] (+)= X[T][K] . W[N][K]^T with the
 * ds_skinny_epi fusions (norm consumer, residual producer + row sums,
 * SwiGLU, RoPE + KV store, LM-head argmax), row-indexed buffers sized for T
 * rows.  N % 128 == 0, K % 64 == 0.  Deterministic (fixed-order split
 * reduction).  Replaces the serial per-entry engine.forward of the reference
 * (scheduler.py:652-660) inside one varlen pass. */
int ds_gemm_stream(const void* X, const void* W, void* Y, int T, int N, int K, int y_f32,
                   int accumulate, const ds_skinny_epi* epi, ds_stream_t stream);

/* K11: projection GEMM on CTA pairs (tcgen05.mma.cta_group::2, 256 tokens x
 * 256 features per tile, persistent, double-buffered TMEM accumulator) for
 * the compute-bound row counts of prefill chunks and batched plans:
 * Y[T][N] (+)= X[T][K] . W[N][K]^T, tokens on the MMA M side so the fused
 * epilogues (epi, as ds_gemm_stream) run per token row.  N % 256 == 0,
 * K % 64 == 0.  Deterministic (no split-K).  Same boundary as K10
 * (scheduler.py:652-660). */
int ds_gemm_pair(const void* X, const void* W, void* Y, int T, int N, int K, int y_f32,
                 int accumulate, const ds_skinny_epi* epi, ds_stream_t stream);

/* K8: row argmax over fp32 logits (lowest index on ties, engine.py:146-159). */
int ds_argmax(const float* logits, int n_rows, int vocab, int32_t* out, ds_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* DELTASERVE_B200_H */
