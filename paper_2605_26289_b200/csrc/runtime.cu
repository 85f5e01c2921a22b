// Native forward runtime: one C call runs a whole plan batch through the
// Llama-shaped decoder (cuBLAS bf16 GEMMs for the plain projections, our
// kernels for everything else) and finishes with the token policy + verify
// accept on device.  Realises engine.forward (engine.py:268-281) for all
// entries of a BatchPlan (scheduler.py:652-772) without materialising the
// context on the host: the context is the resident paged KV store.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/deltaserve_b200.h"
#include "attn_plan.h"
#include "common.cuh"
#include "internal.h"

namespace ds {

void gemm_pair_reserve();  // gemm_pair.cu: K11's tail workspace
void set_attn_l2_prefetch(const void* ptr, int64_t bytes, const void* ptr2 = nullptr,
                          int64_t bytes2 = 0);
int launch_attn_split(const void* qkv, const ds_entry* entries_host, const ds_entry* entries_dev,
                      int n_entries, const void* k_pool, const void* v_pool, int64_t head_stride,
                      const int32_t* pos2cell, int64_t pos_stride, int nh, int nkv, int hd,
                      float scale, void* out, void* workspace, size_t ws_bytes,
                      cudaStream_t stream);
int launch_attn_prefill_sm100(const void* qkv, const ds_entry* entries_host,
                              const ds_entry* entries_dev, int n_entries, const void* k_pool,
                              const void* v_pool, int64_t head_stride, const int32_t* pos2cell,
                              int64_t pos_stride, int nh, int nkv, int hd, float scale, void* out,
                              void* workspace, size_t ws_bytes, cudaStream_t stream);

namespace {

constexpr size_t kAlign = 256;
constexpr size_t kCublasWs = 32u << 20;
// row bound of the fused norm / argmax scalars (two row-sum buffers + the
// LM-head argmax keys), kept at row-count-independent offsets: both GEMM
// paths (skinny M <= 32, stream-K above) share them and the clear/fill cycle
constexpr int kMaxSsRows = 16384;

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Runtime {
  cublasHandle_t blas = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  // graph capture/replay stream (the caller's may be the legacy default stream,
  // which cannot be captured), ordered against the caller's by two events
  cudaStream_t gs = nullptr;
  cudaEvent_t g_in = nullptr, g_out = nullptr;
  int device = -1;
};

Runtime& runtime() {
  static thread_local Runtime rt;
  int dev = 0;
  cudaGetDevice(&dev);
  if (rt.device != dev) {
    if (rt.blas) cublasDestroy(rt.blas);
    cublasCreate(&rt.blas);
    cublasSetMathMode(rt.blas, CUBLAS_DEFAULT_MATH);
    cudaStreamCreateWithFlags(&rt.side, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&rt.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&rt.join, cudaEventDisableTiming);
    cudaStreamCreateWithFlags(&rt.gs, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&rt.g_in, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&rt.g_out, cudaEventDisableTiming);
    gemm_pair_reserve();  // K11's tail workspace, before any graph capture
    rt.device = dev;
  }
  return rt;
}

struct Carve {
  uint8_t* p;
  size_t off = 0;
  template <typename T>
  T* take(size_t bytes) {
    T* r = reinterpret_cast<T*>(p + off);
    off += align_up(bytes);
    return r;
  }
};

struct Buffers {
  float* x;  // fp32 residual stream
  __nv_bfloat16 *h, *qkv, *attn, *gu, *act, *hf;
  uint64_t* ss;    // 2 x kMaxSsRows: fixed-point row sums of squares (GEMM epilogues)
  uint64_t* amax;  // kMaxSsRows: fused LM-head argmax keys (re-armed by the token policy)
  uint64_t* row_hash;
  void* attn_ws;
  size_t attn_ws_bytes;
  void* blas_ws;
};

size_t layout(const ds_model* m, int rows, int outs, Buffers* b, uint8_t* base) {
  Carve c{base};
  const size_t H = m->hidden, F = m->ffn;
  const size_t QKV = static_cast<size_t>(m->n_heads + 2 * m->n_kv_heads) * m->head_dim;
  const size_t A = static_cast<size_t>(m->n_heads) * m->head_dim;
  Buffers t{};
  // first, at row-count-independent offsets: the ss buffers and the attention
  // split-merge counters are zero between calls (self re-arming), which must
  // hold whatever the previous call's batch size was
  t.ss = c.take<uint64_t>(2 * kMaxSsRows * 8);
  t.amax = c.take<uint64_t>(kMaxSsRows * 8);
  t.attn_ws_bytes = attn_partial_bytes_bound();
  t.attn_ws = c.take<uint8_t>(t.attn_ws_bytes);
  t.x = c.take<float>(rows * H * 4);
  t.h = c.take<__nv_bfloat16>(rows * H * 2);
  t.qkv = c.take<__nv_bfloat16>(rows * QKV * 2);
  t.attn = c.take<__nv_bfloat16>(rows * A * 2);
  t.gu = c.take<__nv_bfloat16>(rows * 2 * F * 2);
  t.act = c.take<__nv_bfloat16>(rows * F * 2);
  t.hf = c.take<__nv_bfloat16>(static_cast<size_t>(outs) * H * 2);
  t.row_hash = c.take<uint64_t>(static_cast<size_t>(outs) * 8);
  t.blas_ws = c.take<uint8_t>(kCublasWs);
  if (b) *b = t;
  return c.off;
}

// Y[M][N] (row-major) = X[M][K] . W[N][K]^T  (+ beta*Y)
cublasStatus_t gemm(cublasHandle_t h, const void* X, const void* W, void* Y, int M, int N, int K,
                    float beta, cudaDataType_t ytype) {
  const float alpha = 1.f;
  return cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, &alpha, W, CUDA_R_16BF, K, X,
                      CUDA_R_16BF, K, &beta, Y, ytype, N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
}

}  // namespace
}  // namespace ds
extern "C" int ds_gemm_skinny(const void* X, const void* W, void* Y, int M, int N, int K,
                              int y_f32, int accumulate, ds_stream_t stream);
extern "C" int ds_gemm_skinny_ex(const void* X, const void* W, void* Y, int M, int N, int K,
                                 int y_f32, int accumulate, const ds_skinny_epi* epi,
                                 ds_stream_t stream);
namespace ds {
namespace {

// DS_GEMM_STREAM=1: K10 (stream-K / cluster split-K tcgen05 GEMM with the
// fused epilogues) for M > 32 rows.  Opt-in: it is correct, deterministic
// and fuses RMSNorm / RoPE+KV store / SwiGLU / the LM-head argmax, but its
// split-K reduction (partials through L2 or DSMEM) and 128 x NT single-CTA
// tiles still lose to cuBLAS + the unfused kernels
bool use_stream_gemm() {
  static const bool v = getenv("DS_GEMM_STREAM") && atoi(getenv("DS_GEMM_STREAM")) == 1;
  return v;
}
// the LM head of > 32 sampled rows (batched plans) on K10 with the fused
// argmax: no [rows][V] fp32 logits are materialised (263 MB at 512 rows) and
// the greedy id comes from the same epilogue key as on the skinny path.
// Default (unset / 2) and 1; DS_GEMM_STREAM=0 restores the library GEMM +
// fp32 logits + K8 argmax.  Measured at 512 rows: 12.59 vs 12.37 ms per
// batched verify forward (+1.8%), 128 rows 5.79 vs 5.75 ms.
bool use_stream_head() {
  static const bool v = !(getenv("DS_GEMM_STREAM") && atoi(getenv("DS_GEMM_STREAM")) == 0);
  return v;
}

// K11 (CTA-pair tcgen05 GEMM with the fused epilogues) from DS_PAIR_MIN_ROWS
// rows (opt-in, unset / 0: off).  Measured: a tie with
// the library GEMM + unfused kernels on whole 2k / 4k-row prefill forwards
// (26.56 vs 26.86 ms, 53.67 vs 53.79), 2% behind on C5's batched prefill
// (3,130-3,140 vs 3,080 ms per step), behind below ~1k rows
int pair_min_rows() {
  static const int v = getenv("DS_PAIR_MIN_ROWS") ? atoi(getenv("DS_PAIR_MIN_ROWS")) : 0;
  return v > 0 ? v : 1 << 30;
}
bool pair_ok(int M, int N, int K) { return M >= pair_min_rows() && N % 256 == 0 && K % 64 == 0; }
// the LM head of many sampled rows (batched verify plans) on K11 with the
// fused argmax from DS_PAIR_HEAD_MIN_ROWS rows (default 64; K10 below): whole
// batched verify forward at 64 / 128 / 256 / 512 / 1024 sampled rows 4.73 ->
// 4.68, 5.78 -> 5.74, 7.90 -> 7.80, 12.56 -> 12.39, 22.39 -> 22.10 ms
bool head_pair_ok(int M, int N, int K) {
  static const int v = getenv("DS_PAIR_HEAD_MIN_ROWS") ? atoi(getenv("DS_PAIR_HEAD_MIN_ROWS")) : 64;
  return v > 0 && M >= v && N % 256 == 0 && K % 64 == 0;
}

// decode / verify row counts stream the weights through our skinny GEMM;
// prefill chunks and batched plans through the stream-K tcgen05 GEMM (K10).
int project(cublasHandle_t h, const void* X, const void* W, void* Y, int M, int N, int K,
            bool y_f32, bool accumulate, cudaStream_t s) {
  if (M <= 32 && N % 16 == 0 && K % 256 == 0)
    return ds_gemm_skinny(X, W, Y, M, N, K, y_f32, accumulate, s);
  if (pair_ok(M, N, K)) return ds_gemm_pair(X, W, Y, M, N, K, y_f32, accumulate, nullptr, s);
  if (use_stream_gemm() && N % 128 == 0 && K % 64 == 0)
    return ds_gemm_stream(X, W, Y, M, N, K, y_f32, accumulate, nullptr, s);
  const cublasStatus_t st = gemm(h, X, W, Y, M, N, K, accumulate ? 1.f : 0.f,
                                 y_f32 ? CUDA_R_32F : CUDA_R_16BF);
  return st == CUBLAS_STATUS_SUCCESS ? 0 : 1000 + static_cast<int>(st);
}

__global__ void scatter_tokens_kernel(const int32_t* tok, const int32_t* row_seq,
                                      const int32_t* row_pos, int n, int32_t* hist,
                                      int64_t stride) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) hist[static_cast<int64_t>(row_seq[r]) * stride + row_pos[r]] = tok[r];
}

}  // namespace
}  // namespace ds

using namespace ds;

#define DS_CUDA(x)                                 \
  do {                                             \
    cudaError_t e_ = (x);                          \
    if (e_ != cudaSuccess) return static_cast<int>(e_); \
  } while (0)
#define DS_BLAS(x)                                              \
  do {                                                          \
    cublasStatus_t s_ = (x);                                    \
    if (s_ != CUBLAS_STATUS_SUCCESS) return 1000 + static_cast<int>(s_); \
  } while (0)
#define DS_CHECK(x)        \
  do {                     \
    int r_ = (x);          \
    if (r_ != 0) return r_; \
  } while (0)

extern "C" {

int ds_abi_version(void) { return 1; }

const char* ds_status_string(int status) {
  if (status == DS_OK) return "ok";
  if (status == DS_EINVAL) return "invalid argument";
  if (status == DS_EUNSUPPORTED) return "unsupported shape";
  if (status == DS_EWORKSPACE) return "workspace too small";
  if (status >= 1000) return "cublas error";
  return cudaGetErrorString(static_cast<cudaError_t>(status));
}

size_t ds_attention_workspace_bytes(int n_rows, int n_entries, int n_heads, int head_dim) {
  (void)n_rows;
  (void)n_entries;
  (void)n_heads;
  (void)head_dim;
  return attn_partial_bytes_bound();
}

int ds_attention(const void* qkv, const ds_entry* entries_host, const ds_entry* entries_dev,
                 int n_entries, int n_rows, const void* k_pool_l, const void* v_pool_l,
                 int64_t kv_head_stride, const int32_t* pos2cell, int64_t pos_stride,
                 int n_heads, int n_kv_heads,
                 int head_dim, float scale, void* out, void* workspace, size_t workspace_bytes,
                 int impl, ds_stream_t stream) {
  (void)n_rows;
  if (n_entries <= 0 || n_kv_heads <= 0 || n_heads % n_kv_heads) return DS_EINVAL;
  int max_q = 0;
  for (int e = 0; e < n_entries; ++e) max_q = entries_host[e].q_len > max_q ? entries_host[e].q_len : max_q;
  // auto: decode / verify rows (R <= kDecodeMaxRows) -> K7; delta prefill -> tcgen05 K6
  if (impl == 0) impl = max_q * (n_heads / n_kv_heads) > kDecodeMaxRows ? 2 : 1;
  if (impl == 2)
    return launch_attn_prefill_sm100(qkv, entries_host, entries_dev, n_entries, k_pool_l, v_pool_l,
                                     kv_head_stride, pos2cell, pos_stride, n_heads, n_kv_heads,
                                     head_dim, scale, out, workspace, workspace_bytes,
                                     (cudaStream_t)stream);
  return launch_attn_split(qkv, entries_host, entries_dev, n_entries, k_pool_l, v_pool_l,
                           kv_head_stride, pos2cell, pos_stride, n_heads, n_kv_heads, head_dim,
                           scale, out, workspace, workspace_bytes, (cudaStream_t)stream);
}

size_t ds_forward_workspace_bytes(const ds_model* model, int max_rows, int max_out,
                                  int max_entries) {
  (void)max_entries;
  return layout(model, max_rows, max_out, nullptr, nullptr) + kAlign;
}

static int forward_body(const ds_model* m, const ds_kv_store* kv, const ds_forward_args* a,
                        cudaStream_t stream);

// ---- CUDA graphs for the decode / verify forward ----
// A single-entry forward of <= 32 rows launches ~165 kernels whose launch
// parameters depend only on the argument pointers/counts and, through the
// attention split plan, on (q_len, n_splits, split_len, >= 4k keys).  The
// second time a signature is seen its launch sequence is captured (PDL edges,
// the side-stream fork/join and the cluster launches included) and replayed
// with one cudaGraphLaunch from then on; the first sighting runs eagerly (it
// also performs every one-time attribute / tensor-map setup outside capture).
// Every pointer the graph bakes in is part of the key, so a moved buffer is a
// new signature.  DS_GRAPHS=0 disables.
namespace {
struct GraphEntry {
  int seen = 0;
  cudaGraphExec_t exec = nullptr;
};

std::string graph_key(const ds_model* m, const ds_kv_store* kv, const ds_forward_args* a) {
  std::string k;
  k.append(reinterpret_cast<const char*>(m), sizeof(*m));
  k.append(reinterpret_cast<const char*>(kv), sizeof(*kv));
  k.append(reinterpret_cast<const char*>(a), sizeof(*a));
  const int G = m->n_heads / m->n_kv_heads;
  for (int e = 0; e < a->n_entries; ++e) {
    const ds_entry& en = a->entries_host[e];
    const int kv_len = en.past + en.q_len;
    const AttnSplitPlan p =
        attn_split_plan(1, kv_len, m->n_kv_heads, a->n_entries, 1, en.q_len * G);
    // decode / verify (K7): the split plan fixes every launch shape; prefill
    // chunks (K6 + library GEMMs): the exact (past, q_len)
    const bool k6 = en.q_len * G > kDecodeMaxRows;
    const int sig[5] = {en.q_len, k6 ? en.past : p.n_splits, k6 ? -1 : p.split_len,
                        kv_len >= kDecodeTcMinKeys ? 1 : 0, en.q_len * G};
    k.append(reinterpret_cast<const char*>(sig), sizeof(sig));
  }
  return k;
}
}  // namespace

int ds_model_forward(const ds_model* m, const ds_kv_store* kv, const ds_forward_args* a,
                     ds_stream_t stream_) {
  if (!m || !kv || !a || a->n_rows <= 0 || a->n_entries <= 0 || a->n_out <= 0) return DS_EINVAL;
  cudaStream_t stream = (cudaStream_t)stream_;
  static const bool graphs = !(getenv("DS_GRAPHS") && atoi(getenv("DS_GRAPHS")) == 0);
  // single-entry decode / verify forwards (<= 32 rows; the key is the split
  // plan, which repeats across prefix lengths).  DS_GRAPHS=3 also captures
  // prefill chunks, keyed by their exact (past, q_len): a real workload
  // rarely repeats one, so the capture + instantiate (~10 ms) lands on the
  // critical path (C4 prefill 691 -> 1077 ms per step) - A/B only.
  static const bool graph_prefill = getenv("DS_GRAPHS") && atoi(getenv("DS_GRAPHS")) == 3;
  if (graphs && a->n_entries == 1 && (a->n_rows <= 32 || graph_prefill)) {
    static thread_local std::unordered_map<std::string, GraphEntry> cache;
    if (cache.size() > 512) {  // bound: drop everything (rare - signatures repeat)
      for (auto& kv_ : cache)
        if (kv_.second.exec) cudaGraphExecDestroy(kv_.second.exec);
      cache.clear();
    }
    GraphEntry& ge = cache[graph_key(m, kv, a)];
    if (ge.exec || ge.seen >= 1) {
      Runtime& rt = runtime();
      const cudaStream_t gs = rt.gs;
      DS_CUDA(cudaEventRecord(rt.g_in, stream));
      DS_CUDA(cudaStreamWaitEvent(gs, rt.g_in, 0));
      if (!ge.exec) {
        DS_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeRelaxed));
        int rc = forward_body(m, kv, a, gs);
        const cudaError_t pe = cudaGetLastError();  // an unchecked call that refused capture
        if (rc == DS_OK && pe != cudaSuccess) rc = static_cast<int>(pe);
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(gs, &g);
        cudaError_t ie = cudaSuccess;
        if (rc == DS_OK && ce == cudaSuccess && g) ie = cudaGraphInstantiate(&ge.exec, g, 0);
        if (g) cudaGraphDestroy(g);
        if (rc != DS_OK || ce != cudaSuccess || !g || ie != cudaSuccess) {
          ge.exec = nullptr;
          ge.seen = -1000000;  // this signature is not capturable: stay eager
          cudaGetLastError();
          static bool warned = false;
          if (!warned) {
            warned = true;
            fprintf(stderr, "deltaserve_b200: forward graph capture failed (%d / %s / %s)\n",
                    rc, cudaGetErrorString(ce), cudaGetErrorString(ie));
          }
          DS_CUDA(cudaEventRecord(rt.g_out, gs));
          DS_CUDA(cudaStreamWaitEvent(stream, rt.g_out, 0));
          return forward_body(m, kv, a, stream);
        }
      }
      DS_CUDA(cudaGraphLaunch(ge.exec, gs));
      DS_CUDA(cudaEventRecord(rt.g_out, gs));
      DS_CUDA(cudaStreamWaitEvent(stream, rt.g_out, 0));
      return DS_OK;
    }
    ++ge.seen;
  }
  return forward_body(m, kv, a, stream);
}

static int forward_body(const ds_model* m, const ds_kv_store* kv, const ds_forward_args* a,
                        cudaStream_t stream) {
  Runtime& rt = runtime();
  uint8_t* base = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(a->workspace) + kAlign - 1) / kAlign * kAlign);
  Buffers b;
  const size_t need = layout(m, a->n_rows, a->n_out, &b, base);
  if (need + kAlign > a->workspace_bytes) return DS_EWORKSPACE;

  const int T = a->n_rows, H = m->hidden, L = m->layers, hd = m->head_dim;
  const int nh = m->n_heads, nkv = m->n_kv_heads, F = m->ffn;
  const int QKV = (nh + 2 * nkv) * hd;
  const float scale = 1.f / sqrtf(static_cast<float>(hd));
  const size_t kv_layer = static_cast<size_t>(kv->capacity) * nkv * hd;  // elements per layer
  int max_q = 0;
  for (int e = 0; e < a->n_entries; ++e)
    max_q = a->entries_host[e].q_len > max_q ? a->entries_host[e].q_len : max_q;
  const int attn_impl = 0;  // auto
  // entries ordered long (q*G > kDecodeMaxRows: tcgen05 K6) first, then short (K7)
  int n_long = 0;
  while (n_long < a->n_entries && a->entries_host[n_long].q_len * (nh / nkv) > kDecodeMaxRows)
    ++n_long;
  for (int e = n_long; e < a->n_entries; ++e)
    if (a->entries_host[e].q_len * (nh / nkv) > kDecodeMaxRows) n_long = 0;  // unsorted: auto

  if (T > 32) {  // the library GEMM serves only prefill chunks / batched plans
    DS_BLAS(cublasSetStream(rt.blas, stream));
    DS_BLAS(cublasSetWorkspace(rt.blas, b.blas_ws, kCublasWs));
  }

  // the embedding first (it depends only on the uploaded tokens): the first
  // node of a replayed graph starts at once; then batch tokens -> history (the
  // copy rule scans it) and the per-row FNV states on a side stream
  DS_CHECK(ds_embed(a->tokens, T, m->embed, H, b.x, 1, stream));
  DS_CUDA(launch_pdl(scatter_tokens_kernel, dim3((T + 127) / 128), dim3(128), 0, stream,
                     a->tokens, a->row_seq, a->row_pos, T, kv->hist, kv->pos_stride));
  DS_CUDA(cudaEventRecord(rt.fork, stream));
  DS_CUDA(cudaStreamWaitEvent(rt.side, rt.fork, 0));
  launch_row_hash(a, kv, b.row_hash, rt.side);
  DS_CUDA(cudaGetLastError());
  DS_CUDA(cudaEventRecord(rt.join, rt.side));

  const __nv_bfloat16* wqkv = static_cast<const __nv_bfloat16*>(m->wqkv);
  const __nv_bfloat16* wo = static_cast<const __nv_bfloat16*>(m->wo);
  const __nv_bfloat16* wgu = static_cast<const __nv_bfloat16*>(m->w_gate_up);
  const __nv_bfloat16* wd = static_cast<const __nv_bfloat16*>(m->w_down);
  const __nv_bfloat16* an = static_cast<const __nv_bfloat16*>(m->attn_norm);
  const __nv_bfloat16* mn = static_cast<const __nv_bfloat16*>(m->mlp_norm);
  __nv_bfloat16* kp = static_cast<__nv_bfloat16*>(kv->k_pool);
  __nv_bfloat16* vp = static_cast<__nv_bfloat16*>(kv->v_pool);
  // decode / verify row counts (T <= 32): the RMSNorms and the SwiGLU ride in
  // the skinny GEMM epilogues - wo / down (residual producers) emit
  // h = bf16(x * next norm weight) and per-CTA row sums of x^2, wqkv / gate_up
  // scale their rows by the inverse RMS; gate_up emits silu(g)*u directly.
  // bytes of the next projection's weights each skinny GEMM's last wave pulls
  // into L2 (DS_L2_NEXT_MB overrides for A/B measurements; 0 disables).  10 MB
  // since the balanced verify grids (m=1k q=5 forward: 0 / 4 / 8 / 10 / 12 /
  // 16 MB -> 2.83 / 2.795 / 2.785 / 2.784 / 2.806 / 2.842 ms; q=1 flat)
  static const int64_t l2_next_bytes = [] {
    const char* e = getenv("DS_L2_NEXT_MB");
    return static_cast<int64_t>(e ? atof(e) * 1048576.0 : 10.0 * 1048576.0);
  }();
  // the fused epilogues: skinny GEMM (T <= 32) or the stream-K tcgen05 GEMM
  // (K10, larger T) - the same ds_skinny_epi fusions either way
  const bool small = T <= 32;
  // M > 32: K11 from pair_min_rows() rows (every projection N % 256), else K10
  // when opted in, else the library GEMM + the unfused kernels
  const bool pair = !small && T >= pair_min_rows() && T <= kMaxSsRows && QKV % 256 == 0 &&
                    H % 256 == 0 && (2 * F) % 256 == 0 && (nh * hd) % 64 == 0 && F % 64 == 0;
  const bool fused = hd == 128 && QKV % 16 == 0 &&
                     (small ? (H % 256 == 0 && F % 256 == 0 && (nh * hd) % 256 == 0)
                            : pair || (use_stream_gemm() && T <= kMaxSsRows && QKV % 128 == 0 &&
                                       H % 128 == 0 && (2 * F) % 128 == 0 &&
                                       (nh * hd) % 64 == 0 && F % 64 == 0));
  auto gemm_ex = [&](const void* X, const void* W, void* Y, int N, int K, int y_f32, int acc,
                     const ds_skinny_epi* e) {
    return small ? ds_gemm_skinny_ex(X, W, Y, T, N, K, y_f32, acc, e, stream)
                 : pair ? ds_gemm_pair(X, W, Y, T, N, K, y_f32, acc, e, stream)
                        : ds_gemm_stream(X, W, Y, T, N, K, y_f32, acc, e, stream);
  };
  // two ss buffers, each producer clearing the one its consumer already read
  // (wo clears ss_attn, read by this layer's wqkv; down clears ss_mlp)
  uint64_t* ss_attn = b.ss;               // down -> next wqkv
  uint64_t* ss_mlp = b.ss + kMaxSsRows;  // wo -> gate_up
  for (int l = 0; l < L; ++l) {
    const __nv_bfloat16* wqkv_l = wqkv + static_cast<size_t>(l) * QKV * H;
    if (fused) {  // norm (row scale) + projection + RoPE + KV store in one launch
      ds_skinny_epi e{};
      if (l > 0) {
        e.row_ss = ss_attn;
        e.eps = m->rms_eps;
      } else {
        DS_CHECK(ds_rmsnorm(b.x, 1, nullptr, T, H, an, m->rms_eps, b.h, stream));
      }
      e.rope = 1;
      e.n_heads = nh;
      e.n_kv_heads = nkv;
      e.row_seq = a->row_seq;
      e.row_pos = a->row_pos;
      e.pos2cell = kv->pos2cell;
      e.pos_stride = kv->pos_stride;
      e.rope_cos = m->rope_cos;
      e.rope_sin = m->rope_sin;
      e.k_pool_l = kp + l * kv_layer;
      e.v_pool_l = vp + l * kv_layer;
      e.kv_head_stride = kv->capacity;
      DS_CHECK(gemm_ex(b.h, wqkv_l, b.qkv, QKV, H, 0, 0, &e));
    } else {
      DS_CHECK(ds_rmsnorm(b.x, 1, nullptr, T, H, an + static_cast<size_t>(l) * H, m->rms_eps, b.h,
                          stream));
      // wqkv on K11 with RoPE + the KV store in its epilogue from
      // DS_PAIR_QKV_MIN_ROWS rows (default 2048; with K11 gate_up: 2k / 4k rows
      // 26.7 -> 26.4, 53.6 -> 53.2 ms; at 1.5k rows it lost 21.41 -> 21.75)
      static const int qkv_min =
          getenv("DS_PAIR_QKV_MIN_ROWS") ? atoi(getenv("DS_PAIR_QKV_MIN_ROWS")) : 2048;
      if (qkv_min > 0 && T >= qkv_min && QKV % 256 == 0 && H % 64 == 0 && hd == 128) {
        ds_skinny_epi e{};
        e.rope = 1;
        e.n_heads = nh;
        e.n_kv_heads = nkv;
        e.row_seq = a->row_seq;
        e.row_pos = a->row_pos;
        e.pos2cell = kv->pos2cell;
        e.pos_stride = kv->pos_stride;
        e.rope_cos = m->rope_cos;
        e.rope_sin = m->rope_sin;
        e.k_pool_l = kp + l * kv_layer;
        e.v_pool_l = vp + l * kv_layer;
        e.kv_head_stride = kv->capacity;
        DS_CHECK(ds_gemm_pair(b.h, wqkv_l, b.qkv, T, QKV, H, 0, 0, &e, stream));
      } else {
        DS_CHECK(project(rt.blas, b.h, wqkv_l, b.qkv, T, QKV, H, false, false, stream));
        DS_CHECK(ds_rope_kv_store(b.qkv, T, a->row_seq, a->row_pos, kv->pos2cell,
                                  kv->pos_stride, nh, nkv, hd, m->rope_cos, m->rope_sin,
                                  kp + l * kv_layer, vp + l * kv_layer, kv->capacity, stream));
      }
    }
    // the attention leaves HBM mostly idle (short contexts): K7's producer
    // warps pull wo's weights into L2 for the next projection meanwhile
    // (and the head of gate_up's: DS_GU_L2_MB, continued by wo's own prefetch)
    // half of wo: the rest streams through the wo CTAs' rings (measured, sweep
    // of 0 / 0.25 / 0.5 / 1: m=300 q=1 forward 2.76 -> 2.67 ms, m=1k q=1 2.69 ->
    // 2.62, q=5 2.85 -> 2.84; C2 26.78 -> 26.92 turns/s - the whole of wo
    // crowded the short attention's own loads)
    static const double wo_l2_frac = getenv("DS_WO_L2_FRAC") ? atof(getenv("DS_WO_L2_FRAC")) : 0.5;
    static const int64_t gu_l2_bytes = static_cast<int64_t>(
        (getenv("DS_GU_L2_MB") ? atof(getenv("DS_GU_L2_MB")) : 0.0) * 1048576.0) & ~15ll;
    const int64_t gu_head = fused && small ? gu_l2_bytes : 0;
    if (fused && small && (wo_l2_frac > 0 || gu_head > 0))
      set_attn_l2_prefetch(wo + static_cast<size_t>(l) * H * nh * hd,
                           static_cast<int64_t>(wo_l2_frac * H * nh * hd * 2) & ~15ll,
                           wgu + static_cast<size_t>(l) * 2 * F * H, gu_head);
    if (n_long > 0 && n_long < a->n_entries) {  // mixed plan: K6 for prefill chunks, K7 rest
      DS_CHECK(ds_attention(b.qkv, a->entries_host, a->entries, n_long, T, kp + l * kv_layer,
                            vp + l * kv_layer, kv->capacity, kv->pos2cell, kv->pos_stride, nh,
                            nkv, hd, scale, b.attn, b.attn_ws, b.attn_ws_bytes, 2, stream));
      DS_CHECK(ds_attention(b.qkv, a->entries_host + n_long, a->entries + n_long,
                            a->n_entries - n_long, T, kp + l * kv_layer, vp + l * kv_layer,
                            kv->capacity, kv->pos2cell, kv->pos_stride, nh, nkv, hd, scale,
                            b.attn, b.attn_ws, b.attn_ws_bytes, 1, stream));
    } else {
      DS_CHECK(ds_attention(b.qkv, a->entries_host, a->entries, a->n_entries, T,
                            kp + l * kv_layer, vp + l * kv_layer, kv->capacity, kv->pos2cell,
                            kv->pos_stride, nh, nkv, hd, scale, b.attn, b.attn_ws,
                            b.attn_ws_bytes, attn_impl, stream));
    }
    const __nv_bfloat16* wo_l = wo + static_cast<size_t>(l) * H * nh * hd;
    const __nv_bfloat16* wgu_l = wgu + static_cast<size_t>(l) * 2 * F * H;
    const __nv_bfloat16* wd_l = wd + static_cast<size_t>(l) * H * F;
    if (fused) {
      ds_skinny_epi eo{};
      // wo's CTAs sit beside the attention (one-stage K7) waiting for it: they
      // pull the head of gate_up's weights meanwhile (DS_WO_PRE_MB)
      static const int64_t wo_pre_bytes = static_cast<int64_t>(
          (getenv("DS_WO_PRE_MB") ? atof(getenv("DS_WO_PRE_MB")) : 0.0) * 1048576.0) & ~15ll;
      const int64_t gu_pre = small ? wo_pre_bytes : 0;
      eo.l2_pre = gu_pre ? reinterpret_cast<const char*>(wgu_l) + gu_head : nullptr;
      eo.l2_pre_bytes = gu_pre;
      eo.l2_next = reinterpret_cast<const char*>(wgu_l) + gu_head + gu_pre;
      eo.l2_next_bytes = l2_next_bytes;
      eo.ss_out = ss_mlp;
      eo.ss_zero = ss_attn;
      eo.h_out = b.h;
      eo.h_w = mn + static_cast<size_t>(l) * H;
      DS_CHECK(gemm_ex(b.attn, wo_l, b.x, H, nh * hd, 1, 1, &eo));
      ds_skinny_epi eg{};
      eg.row_ss = ss_mlp;
      eg.eps = m->rms_eps;
      eg.swiglu = 1;
      eg.l2_next = wd_l;
      eg.l2_next_bytes = l2_next_bytes;
      DS_CHECK(gemm_ex(b.h, wgu_l, b.act, 2 * F, H, 0, 0, &eg));
      ds_skinny_epi ed{};
      ed.ss_out = ss_attn;  // (last layer: unused, keeps the clear/fill cycle uniform)
      ed.ss_zero = ss_mlp;
      ed.l2_next = l + 1 < L ? static_cast<const void*>(wqkv_l + static_cast<size_t>(QKV) * H)
                             : m->lm_head;
      ed.l2_next_bytes = l2_next_bytes;
      if (l + 1 < L) {
        ed.h_out = b.h;
        ed.h_w = an + static_cast<size_t>(l + 1) * H;
      }
      DS_CHECK(gemm_ex(b.act, wd_l, b.x, H, F, 1, 1, &ed));
    } else {
      DS_CHECK(project(rt.blas, b.attn, wo_l, b.x, T, H, nh * hd, true, true, stream));
      DS_CHECK(ds_rmsnorm(b.x, 1, nullptr, T, H, mn + static_cast<size_t>(l) * H, m->rms_eps,
                          b.h, stream));
      // gate_up on K11 with the SwiGLU in its epilogue from DS_PAIR_GU_MIN_ROWS
      // rows (default 1024; no [T][2F] intermediate, no SiLU launch): whole
      // forward at 1.5k / 2k / 4k rows 22.06 -> 21.41, 27.5 -> 26.7, 55.6 -> 53.6 ms
      static const int gu_min =
          getenv("DS_PAIR_GU_MIN_ROWS") ? atoi(getenv("DS_PAIR_GU_MIN_ROWS")) : 1024;
      if (gu_min > 0 && T >= gu_min && (2 * F) % 256 == 0 && H % 64 == 0 && hd == 128) {
        ds_skinny_epi eg{};
        eg.swiglu = 1;
        DS_CHECK(ds_gemm_pair(b.h, wgu_l, b.act, T, 2 * F, H, 0, 0, &eg, stream));
      } else {
        DS_CHECK(project(rt.blas, b.h, wgu_l, b.gu, T, 2 * F, H, false, false, stream));
        DS_CHECK(ds_silu_mul(b.gu, T, F, b.act, stream));
      }
      DS_CHECK(project(rt.blas, b.act, wd_l, b.x, T, H, F, true, true, stream));
    }
  }
  set_attn_l2_prefetch(nullptr, 0);  // a hint not consumed (K6-only layer) must not leak
  // final norm on sampled rows only, LM head in fp32
  DS_CHECK(ds_rmsnorm(b.x, 1, a->out_rows, a->n_out, H, m->final_norm, m->rms_eps, b.hf, stream));
  // LM head: <= 32 sampled rows reduce to their argmax in the GEMM epilogue
  // (logits stored only on request); more rows go through the library GEMM
  // and the K8 row argmax
  const bool fused_head = a->n_out <= 32 ||
                          (use_stream_head() && a->n_out <= kMaxSsRows && m->vocab % 128 == 0);
  if (fused_head) {
    ds_skinny_epi eh{};
    eh.argmax_out = b.amax;
    void* lg = a->logits_out ? a->logits : nullptr;
    if (a->n_out <= 32)
      DS_CHECK(ds_gemm_skinny_ex(b.hf, m->lm_head, lg, a->n_out, m->vocab, H, 1, 0, &eh, stream));
    else if (pair_ok(a->n_out, m->vocab, H) || head_pair_ok(a->n_out, m->vocab, H))
      DS_CHECK(ds_gemm_pair(b.hf, m->lm_head, lg, a->n_out, m->vocab, H, 1, 0, &eh, stream));
    else
      DS_CHECK(ds_gemm_stream(b.hf, m->lm_head, lg, a->n_out, m->vocab, H, 1, 0, &eh, stream));
  } else {
    DS_CHECK(project(rt.blas, b.hf, m->lm_head, a->logits, a->n_out, m->vocab, H, true, false,
                     stream));
  }

  DS_CUDA(cudaStreamWaitEvent(stream, rt.join, 0));
  launch_token_policy(a, kv, b.row_hash, fused_head ? b.amax : nullptr, m->vocab, rt.side, stream);
  DS_CUDA(cudaGetLastError());
  if (a->next_window > 0 && a->next_cap > 0 && a->next_out) {
    launch_next_draft(a, kv, stream);
    DS_CUDA(cudaGetLastError());
  }
  return DS_OK;
}

}  // extern "C"
