// sp_runtime.cu — C-ABI runtime: group construction (weight snapshot + TMA descriptors + HBM
// workspace) and the per-request launch sequence of the student-group forward.
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <unordered_set>
#include <tuple>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/studentpar_b200.h"
#include "sp_kernels.cuh"

namespace sp {
bool rowops_supported_hidden(int hidden);
}

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define SP_CUDA(expr)                                                                         \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) return fail(SP_ECUDA, "%s: %s", #expr, cudaGetErrorString(_e));   \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// fp16 row-major [rows, cols] viewed as a 2-D tensor map with a {64, box_rows} box, 128-B swizzle.
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

bool make_map(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  auto fn = encode_fn();
  if (fn == nullptr || ptr == nullptr || rows == 0) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct XMaps {
  CUtensorMap x64, x16;
};

bool make_xmaps(XMaps* m, const void* ptr, uint64_t rows, uint64_t cols) {
  return make_map(&m->x64, ptr, rows, cols, 64) && make_map(&m->x16, ptr, rows, cols, 16);
}

int choose_splits(int units, int nkb, int smax) {
  static const int policy = [] {  // 0: first split with >= 128 CTAs; 1 (default, -2 us at L=128-256): balance the SMs
    const char* v = getenv("SP_SPLIT_POLICY");
    return v ? atoi(v) : 1;
  }();
  if (policy == 1 && units < 148) {  // with >= 1 tile per SM the one-split persistent path wins
    // makespan in k-blocks of the busiest CTA slot: ceil(units * s / slots) waves of nkb / s each
    int best = 1;
    long long best_cost = 0x7fffffffffffll;
    for (int s = 1; s <= smax; ++s) {
      if (nkb % s || (s > 1 && nkb / s < 2)) continue;
      const long long ctas = (long long)units * s;
      // per-SM load: CTAs per SM (ceil over the 148 SMs) x k-blocks each, + partial-sum traffic
      const long long per_sm = (ctas + 147) / 148;
      const long long cost = per_sm * (nkb / s) * 4 + s;
      if (cost < best_cost) {
        best_cost = cost;
        best = s;
      }
    }
    return best;
  }
  int best = 1;
  for (int s = 1; s <= smax; ++s) {
    if (nkb % s) continue;
    if (s > 1 && nkb / s < 2) continue;
    best = s;
    if (units * s >= 128) break;
  }
  return best;
}

constexpr int kMaxSplits = 4;
static_assert(sp::kReqMaxSplit <= kMaxSplits, "request-kernel partials live in the split-K buffers");

}  // namespace

namespace sp {
void prefer_max_smem(const void* fn) {
  static const int carveout = env_int("SP_CARVEOUT", -1);
  static std::mutex mu;
  static std::unordered_set<const void*> done;
  if (carveout < 0) return;
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert(fn).second) cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
}
}  // namespace sp

struct sp_group {
  sp_config cfg;
  sp_weights w;
  int device = 0;
  int rows_cap = 0;  // max(max_tokens, max_seqs)
  // workspace
  float* x32 = nullptr;    // [S][max_tokens][H] residual stream (fp32)
  half* x16 = nullptr;     // [S][max_tokens][H] GEMM operand copy of x32
  half* qkv = nullptr;     // [S][max_tokens][3H]
  half* ctx = nullptr;     // [S][max_tokens][H]
  half* ffn = nullptr;     // [S][max_tokens][F]
  float* part = nullptr;   // [kMaxSplits][S][max_tokens][H] split-K partials
  half* cls16 = nullptr;   // [S][max_seqs][H] CLS rows
  float* final32 = nullptr;  // [S][rows_cap][H] per-student final representation
  half* xin = nullptr;     // dense: [max_tokens][d_in] staged input (host API)
  int32_t* d_ids = nullptr;   // staging block [cu_pad | ids]: d_cu = block, d_ids = block + cu_pad
  int32_t* d_cu = nullptr;
  int cu_pad = 0;             // max_seqs + 1 rounded up to 32 ints (128 B)
  int32_t* h_stage = nullptr;  // pinned mirror of the staging block: one H2D copy per request
  float* h_logits = nullptr;   // pinned logits landing buffer
  // batch-1 host path without a stream sync: the head kernel writes the logits into mapped pinned
  // memory, then the request's sequence number (staged with its ids) into a mapped flag the host
  // polls; the graph has no device-to-host copy node
  void* h_mapped = nullptr;     // [logits f32 x n_classes | pad | flag int]
  float* d_out = nullptr;       // device alias of the logits slot
  int* d_flag = nullptr;        // device alias of the flag
  int seq = 0;
  int* head_flag = nullptr;     // set while capturing a host-path graph
  const int* head_seq = nullptr;
  float* d_logits = nullptr;
  int* mlp_done = nullptr;  // fused FFN kernel: FFN1 tiles finished per student + exit counter
  // weight streamer (sp_stream.cu): [progress, base, finished CTAs], side stream + fork/join events
  unsigned long long* ws_state = nullptr;
  unsigned long long* ws_active = nullptr;  // = ws_state while a streamed forward is being launched
  cudaStream_t ws_stream = nullptr;
  cudaEvent_t ws_fork = nullptr, ws_join = nullptr;
  std::vector<void*> allocs;
  // tensor maps
  std::vector<CUtensorMap> m_qkv, m_o, m_f1, m_f2, m_layers;
  CUtensorMap m_pool, m_in;
  CUtensorMap m_qkv_attn;  // qkv buffer viewed with a {64, 128} box (tensor-core attention)
  CUtensorMap m_qkv_kv64;  // the same with a {64, 64} box (64-key chunks of the three-CTA kernel)
  // the two maps with their origin at student g0 (second chain of a student-split request)
  std::vector<CUtensorMap> m_qkv_attn_at, m_qkv_kv64_at;
  // student-split batch-1 requests: the second half of the students runs as its own kernel chain
  cudaStream_t chain_stream = nullptr;
  cudaEvent_t chain_fork = nullptr, chain_join = nullptr;
  XMaps xm_x16, xm_ctx, xm_ffn, xm_cls, xm_ha, xm_hb;
  int last_launches = 0;
  // CUDA graphs of the batch-1 host path, keyed by (16-token bucket, k_active, add_bias)
  std::map<std::tuple<int, int, int>, cudaGraphExec_t> graphs;
  // graphs of the device-buffer batch-1 path (sp_group_forward_graph), keyed also by the logits slot
  std::map<std::tuple<int, int, int, uintptr_t>, cudaGraphExec_t> dgraphs;
  cudaStream_t cap_stream = nullptr;
  int graph_launches = 0;  // kernels per graph replay
  double sum_len_sq = 0.0;  // sum_b L_b^2 of the current request (attention flops)
  // training-side evaluation outputs of the current sp_group_forward*_eval call (else null)
  float* eval_finals = nullptr;  // [k][rows][H]
  float* eval_prefix = nullptr;  // [k][rows][C]
  float* eval_scratch = nullptr;  // finals when the caller only asks for prefix logits
  // whole-request persistent kernel (sp_request.cu), allocated on first use
  bool req_ready = false;
  int* req_banks = nullptr;    // [2][kReqBankInts] dataflow counters
  int* req_epoch = nullptr;
  sp::ReqMaps req_maps;
  // per-launch profiling (CUDA events around every kernel of the last forward)
  bool profiling = false;
  struct Rec {
    int kind;
    double bytes, flops;
    cudaEvent_t e0, e1;
  };
  std::vector<Rec> recs;
  size_t n_recs = 0;
  cudaStream_t rec_stream = nullptr;
  void rec_reset(cudaStream_t st) {
    n_recs = 0;
    rec_stream = st;
  }
  void rec_begin(int kind, double bytes, double flops) {
    if (!profiling) return;
    if (n_recs == recs.size()) {
      Rec r{};
      cudaEventCreate(&r.e0);
      cudaEventCreate(&r.e1);
      recs.push_back(r);
    }
    Rec& r = recs[n_recs];
    r.kind = kind;
    r.bytes = bytes;
    r.flops = flops;
    cudaEventRecord(r.e0, rec_stream);
  }
  void rec_end() {
    if (!profiling) return;
    cudaEventRecord(recs[n_recs].e1, rec_stream);
    ++n_recs;
  }
};

namespace {

template <typename T>
int dev_alloc(sp_group* g, T** p, size_t count) {
  if (count == 0) count = 1;
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, count * sizeof(T));
  if (e != cudaSuccess) return fail(SP_ENOMEM, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
  g->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return SP_OK;
}

void free_all(sp_group* g) {
  for (auto& kv : g->graphs) cudaGraphExecDestroy(kv.second);
  for (auto& kv : g->dgraphs) cudaGraphExecDestroy(kv.second);
  if (g->ws_stream) cudaStreamDestroy(g->ws_stream);
  if (g->chain_stream) cudaStreamDestroy(g->chain_stream);
  if (g->chain_fork) cudaEventDestroy(g->chain_fork);
  if (g->chain_join) cudaEventDestroy(g->chain_join);
  if (g->ws_fork) cudaEventDestroy(g->ws_fork);
  if (g->ws_join) cudaEventDestroy(g->ws_join);
  g->graphs.clear();
  if (g->cap_stream) cudaStreamDestroy(g->cap_stream);
  g->cap_stream = nullptr;
  for (void* p : g->allocs) cudaFree(p);
  g->allocs.clear();
  if (g->h_stage) cudaFreeHost(g->h_stage);
  if (g->h_logits) cudaFreeHost(g->h_logits);
  if (g->h_mapped) cudaFreeHost(g->h_mapped);
  g->h_mapped = nullptr;
  g->h_stage = nullptr;
  g->h_logits = nullptr;
  for (auto& r : g->recs) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  g->recs.clear();
}

int validate_config(const sp_config& c) {
  if (c.kind != SP_KIND_DENSE && c.kind != SP_KIND_BERT) return fail(SP_EINVAL, "unknown student kind %d", c.kind);
  if (c.n_students < 1) return fail(SP_EINVAL, "n_students must be >= 1");
  if (c.hidden < 128 || c.hidden % 128 || c.hidden > 1024)
    return fail(SP_EINVAL, "hidden=%d must be a multiple of 128 in [128, 1024]", c.hidden);
  if (c.kind == SP_KIND_BERT && !sp::rowops_supported_hidden(c.hidden))
    return fail(SP_EINVAL, "BERT hidden=%d must be one of 128, 256, 512, 768, 1024", c.hidden);
  if (c.n_classes < 1) return fail(SP_EINVAL, "n_classes must be >= 1");
  if (c.max_tokens < 1 || c.max_seqs < 1) return fail(SP_EINVAL, "capacities must be >= 1");
  if (c.kind == SP_KIND_BERT) {
    if (c.n_layers < 1) return fail(SP_EINVAL, "BERT student needs n_layers >= 1");
    if (c.n_heads < 1 || c.hidden % c.n_heads) return fail(SP_EINVAL, "hidden must be divisible by n_heads");
    const int hd = c.hidden / c.n_heads;
    if (hd != 32 && hd != 64) return fail(SP_EINVAL, "head_dim=%d unsupported (32 or 64)", hd);
    if (c.ffn < 128 || c.ffn % 128) return fail(SP_EINVAL, "ffn must be a positive multiple of 128");
    if (c.vocab < 1 || c.max_pos < 1) return fail(SP_EINVAL, "vocab and max_pos must be >= 1");
  } else {
    if (c.n_layers < 2) return fail(SP_EINVAL, "student needs at least 2 layers");  // nnkernel.py:265-266
    if (c.d_in < 64 || c.d_in % 64) return fail(SP_EINVAL, "d_in must be a positive multiple of 64");
  }
  return SP_OK;
}

}  // namespace

extern "C" {

int sp_abi_version(void) { return SP_ABI_VERSION; }

const char* sp_last_error(void) { return g_err.c_str(); }

int sp_group_create(const sp_config* cfg, const sp_weights* weights, int device, sp_group** out) {
  if (cfg == nullptr || weights == nullptr || out == nullptr) return fail(SP_EINVAL, "null argument");
  *out = nullptr;
  int rc = validate_config(*cfg);
  if (rc) return rc;
  if (encode_fn() == nullptr) return fail(SP_ECUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  SP_CUDA(cudaSetDevice(device));
  sp_group* g = new sp_group();
  g->cfg = *cfg;
  g->w = *weights;
  g->device = device;
  const sp_config& c = g->cfg;
  const sp_weights& w = g->w;
  const size_t S = c.n_students, H = c.hidden, T = c.max_tokens, B = c.max_seqs, F = c.ffn;
  g->rows_cap = std::max(c.max_tokens, c.max_seqs);
  const size_t R = g->rows_cap;
  auto bail = [&](int code) {
    free_all(g);
    delete g;
    return code;
  };
  if ((rc = dev_alloc(g, &g->final32, (size_t)kMaxSplits * S * R * H))) return bail(rc);  // pooler split-K partials
  g->cu_pad = ((B + 1 + 31) / 32) * 32;
  if ((rc = dev_alloc(g, &g->d_cu, (size_t)g->cu_pad + T))) return bail(rc);
  g->d_ids = g->d_cu + g->cu_pad;
  if (cudaHostAlloc(reinterpret_cast<void**>(&g->h_stage), sizeof(int32_t) * ((size_t)g->cu_pad + T),
                    cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&g->h_logits), sizeof(float) * (size_t)R * c.n_classes,
                    cudaHostAllocDefault) != cudaSuccess)
    return bail(fail(SP_ENOMEM, "pinned staging buffers"));
  if ((rc = dev_alloc(g, &g->d_logits, R * c.n_classes))) return bail(rc);
  {
    const size_t flag_off = ((sizeof(float) * (size_t)c.n_classes + 127) / 128) * 128;
    void* dev = nullptr;
    if (cudaHostAlloc(&g->h_mapped, flag_off + 128, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&dev, g->h_mapped, 0) != cudaSuccess)
      return bail(fail(SP_ENOMEM, "mapped logits buffer"));
    memset(g->h_mapped, 0, flag_off + 128);
    g->d_out = static_cast<float*>(dev);
    g->d_flag = reinterpret_cast<int*>(static_cast<uint8_t*>(dev) + flag_off);
  }
  if ((rc = dev_alloc(g, &g->mlp_done, sp::kReqMaxStudents + 1))) return bail(rc);
  if (cudaMemset(g->mlp_done, 0, sizeof(int) * (sp::kReqMaxStudents + 1)) != cudaSuccess)
    return bail(fail(SP_ECUDA, "memset"));
  if ((rc = dev_alloc(g, &g->ws_state, 4))) return bail(rc);
  if (cudaMemset(g->ws_state, 0, 4 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&g->ws_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&g->ws_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&g->ws_join, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(SP_ECUDA, "weight streamer state"));

  if (c.kind == SP_KIND_BERT) {
    if (!w.word_emb || !w.pos_emb || !w.type_emb || !w.emb_ln_gamma || !w.emb_ln_beta || !w.w_qkv || !w.b_qkv ||
        !w.w_o || !w.b_o || !w.ln1_gamma || !w.ln1_beta || !w.w_ffn1 || !w.b_ffn1 || !w.w_ffn2 || !w.b_ffn2 ||
        !w.ln2_gamma || !w.ln2_beta || !w.w_pool || !w.b_pool || !w.alpha || !w.w_cls || !w.b_cls)
      return bail(fail(SP_EINVAL, "missing BERT weight pointer"));
    if ((rc = dev_alloc(g, &g->x32, S * T * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->x16, S * T * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->qkv, S * T * 3 * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->ctx, S * T * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->ffn, S * T * F))) return bail(rc);
    if ((rc = dev_alloc(g, &g->part, (size_t)kMaxSplits * S * T * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->cls16, S * B * H))) return bail(rc);
    const auto* wq = static_cast<const half*>(w.w_qkv);
    const auto* wo = static_cast<const half*>(w.w_o);
    const auto* w1 = static_cast<const half*>(w.w_ffn1);
    const auto* w2 = static_cast<const half*>(w.w_ffn2);
    g->m_qkv.resize(c.n_layers);
    g->m_o.resize(c.n_layers);
    g->m_f1.resize(c.n_layers);
    g->m_f2.resize(c.n_layers);
    bool ok = true;
    for (int l = 0; l < c.n_layers; ++l) {
      ok &= make_map(&g->m_qkv[l], wq + (size_t)l * S * 3 * H * H, S * 3 * H, H, 128);
      ok &= make_map(&g->m_o[l], wo + (size_t)l * S * H * H, S * H, H, 128);
      ok &= make_map(&g->m_f1[l], w1 + (size_t)l * S * F * H, S * F, H, 128);
      ok &= make_map(&g->m_f2[l], w2 + (size_t)l * S * H * F, S * H, F, 128);
    }
    ok &= make_map(&g->m_pool, w.w_pool, S * H, H, 128);
    ok &= make_xmaps(&g->xm_x16, g->x16, S * T, H);
    ok &= make_xmaps(&g->xm_ctx, g->ctx, S * T, H);
    ok &= make_xmaps(&g->xm_ffn, g->ffn, S * T, F);
    ok &= make_xmaps(&g->xm_cls, g->cls16, S * B, H);
    ok &= make_map(&g->m_qkv_attn, g->qkv, S * T, 3 * H, 128);
    ok &= make_map(&g->m_qkv_kv64, g->qkv, S * T, 3 * H, 64);
    g->m_qkv_attn_at.resize(S);
    g->m_qkv_kv64_at.resize(S);
    for (int s0 = 0; s0 < S; ++s0) {
      const half* base = g->qkv + (size_t)s0 * T * 3 * H;
      ok &= make_map(&g->m_qkv_attn_at[s0], base, (uint64_t)(S - s0) * T, 3 * H, 128);
      ok &= make_map(&g->m_qkv_kv64_at[s0], base, (uint64_t)(S - s0) * T, 3 * H, 64);
    }
    ok &= cudaStreamCreateWithFlags(&g->chain_stream, cudaStreamNonBlocking) == cudaSuccess &&
          cudaEventCreateWithFlags(&g->chain_fork, cudaEventDisableTiming) == cudaSuccess &&
          cudaEventCreateWithFlags(&g->chain_join, cudaEventDisableTiming) == cudaSuccess;
    // rows past a request's tokens are read (masked) by the attention tiles: keep them finite
    if (cudaMemset(g->qkv, 0, S * T * 3 * H * sizeof(half)) != cudaSuccess) ok = false;
    if (!ok) return bail(fail(SP_EINVAL, "tensor-map creation failed (pointer alignment / shape)"));
  } else {
    if (!w.w_in || !w.b_in || !w.w_layers || !w.b_layers || !w.alpha || !w.w_cls || !w.b_cls)
      return bail(fail(SP_EINVAL, "missing dense weight pointer"));
    half *ha = nullptr, *hb = nullptr;
    if ((rc = dev_alloc(g, &ha, S * T * H))) return bail(rc);
    if ((rc = dev_alloc(g, &hb, S * T * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->xin, T * (size_t)c.d_in))) return bail(rc);
    g->x16 = ha;
    g->ctx = hb;
    const auto* wl = static_cast<const half*>(w.w_layers);
    g->m_layers.resize(c.n_layers);
    bool ok = make_map(&g->m_in, w.w_in, S * H, c.d_in, 128);
    for (int l = 0; l < c.n_layers; ++l) ok &= make_map(&g->m_layers[l], wl + (size_t)l * S * H * H, S * H, H, 128);
    ok &= make_xmaps(&g->xm_ha, ha, S * T, H);
    ok &= make_xmaps(&g->xm_hb, hb, S * T, H);
    if (!ok) return bail(fail(SP_EINVAL, "tensor-map creation failed (pointer alignment / shape)"));
  }
  *out = g;
  return SP_OK;
}

int sp_group_destroy(sp_group* g) {
  if (g == nullptr) return SP_OK;
  cudaSetDevice(g->device);
  free_all(g);
  delete g;
  return SP_OK;
}

int sp_group_last_launches(const sp_group* g) { return g ? g->last_launches : 0; }


int sp_group_set_profiling(sp_group* g, int enable) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  cudaSetDevice(g->device);
  g->profiling = enable != 0;
  g->n_recs = 0;
  return SP_OK;
}

int sp_group_profile_read(sp_group* g, sp_launch_record* out, int max_records) {
  if (g == nullptr || (out == nullptr && max_records > 0)) return -fail(SP_EINVAL, "null argument");
  cudaSetDevice(g->device);
  const int n = static_cast<int>(std::min<size_t>(g->n_recs, max_records > 0 ? (size_t)max_records : 0));
  for (int i = 0; i < n; ++i) {
    const auto& r = g->recs[i];
    if (cudaEventSynchronize(r.e1) != cudaSuccess) return -fail(SP_ECUDA, "event sync failed");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.e0, r.e1);
    out[i].kind = r.kind;
    out[i].ms = ms;
    out[i].bytes = r.bytes;
    out[i].flops = r.flops;
  }
  return static_cast<int>(g->n_recs);
}

}  // extern "C"

namespace {

#define PF(x) (x).p, (x).n

// Tensor-core attention (head_dim 64, L <= 512) is opt-in (SP_ATTN_TC=1): it is correct but measured
// slower than the pipelined mma.sync kernel at every batch-1 length.
// tcgen05 attention (sp_attn_tc.cu) vs mma.sync attention (sp_attn.cu), by the measured crossover
// (tools/len_probe.py): tcgen05 wins up to 128 keys and beyond 384 (one CTA per SM: at 160-384 the
// mma.sync kernel's two CTAs per SM win). SP_ATTN_TC=0 / 1 forces either kernel.
// Attention kernel by length: 0 = mma.sync (sp_attn.cu), 1 = two-pass tcgen05 (sp_attn_tc.cu),
// 2 = single-pass tcgen05, two CTAs per SM, 3 = the same with 64-key chunks at three CTAs per SM
// (sp_attn_tc2.cu). SP_ATTN_TC forces one.
int attn_kind(int head_dim, int max_len) {
  static const int mode = [] {
    const char* v = getenv("SP_ATTN_TC");
    return v == nullptr ? -1 : atoi(v);
  }();
  if (head_dim != 64 || max_len > 512) return 0;
  if (mode >= 0) return mode;
  // measured in-graph (tools/len_probe.py): tc3 (fewest threads / TMEM columns: the shortest
  // latency chain) up to 64 tokens (-2 us), tc1 to 128, tc2 from 129; above 384 (4 query tiles per
  // head) tc3's one wave at three CTAs per SM beats tc2's two waves (-6..-10 us per request)
  if (max_len <= 64) return 3;
  return max_len <= 128 ? 1 : (max_len <= 384 ? 2 : 3);
}

void launch_attention_any(int kind, const CUtensorMap& map_qkv, const CUtensorMap& map_kv64, const half* qkv,
                          half* ctx, const int* cu, int n_seqs, int max_len, int groups, int n_heads, int head_dim,
                          int hidden, long long group_rows, cudaStream_t st) {
  if (kind == 3)
    sp::launch_attention_tc3(map_qkv, map_kv64, ctx, cu, n_seqs, max_len, groups, n_heads, hidden, group_rows, st);
  else if (kind == 2)
    sp::launch_attention_tc2(map_qkv, ctx, cu, n_seqs, max_len, groups, n_heads, hidden, group_rows, st);
  else if (kind == 1)
    sp::launch_attention_tc(map_qkv, ctx, cu, n_seqs, max_len, groups, n_heads, hidden, group_rows, st);
  else
    sp::launch_attention(qkv, ctx, cu, n_seqs, max_len, groups, n_heads, head_dim, hidden, group_rows, st);
}

// Launch one grouped projection. Returns the number of kernels launched (1).
int run_gemm(sp_group* grp, int kind, const CUtensorMap& wmap, const XMaps& xm, int groups, int n_out, int k_dim,
             int t_rows, int x_group_rows, const float* bias, int bias_gs, int act, void* out, long long out_gs,
             int out_f32, int splits, long long split_stride, cudaStream_t st, const int* t_dev = nullptr,
             int g0 = 0) {
  static const int persist_min_rows = [] {
    const char* v = getenv("SP_GEMM_PERSIST_MIN_ROWS");  // one-split projections from 17 tokens on: measured
    return v ? atoi(v) : 17;                                 // equal or 2-4 us faster than the small-T kernel
  }();
  static const int l2_prefetch = [] {
    const char* v = getenv("SP_GEMM_L2PREFETCH");  // measured neutral-to-slower: opt-in
    return v ? atoi(v) : 0;
  }();
  if (splits == 1 && t_rows >= persist_min_rows) {
    sp::GemmParams p{};
    p.g0 = g0;
    p.progress = grp ? grp->ws_active : nullptr;
    p.l2_prefetch = l2_prefetch;
    p.t_dev = t_dev;
    p.n_out = n_out;
    p.k_dim = k_dim;
    p.t_rows = t_rows;
    p.x_group_rows = x_group_rows;
    p.m_tiles = n_out / 128;
    p.splits = 1;
    p.kb_per_split = k_dim / 64;
    p.cluster = 1;
    static const int w_pol = [] {  // persistent path weight L2 policy: 0 evict_first, 1 normal, 2 evict_last
      const char* v = getenv("SP_PERSIST_WPOL");
      return v ? atoi(v) : -1;
    }();
    sp::gemm_configure_persistent(t_rows, out_f32 != 0, groups * p.m_tiles, sp::sm_count(),
                                  sp::gemm_persistent_pair(t_rows, p.m_tiles, groups), &p.bn, &p.n_tiles, &p.stages);
    // weights re-read by many token tiles stay in L2 (evict_last); streamed once or twice (batch-1)
    // they must not push the residual stream out (evict_first: -2% at L=512)
    p.w_keep = w_pol >= 0 ? w_pol : (p.n_tiles > 2 ? 2 : 0);
    static const int direct = [] {
      const char* v = getenv("SP_PERSIST_DIRECT_STORE");  // measured 2-4% slower than smem staging
      return v ? atoi(v) : 0;
    }();
    p.direct_store = direct;
    p.out = out;
    p.out_group_stride = out_gs;
    p.out_ld = n_out;
    p.bias = bias;
    p.bias_group_stride = bias_gs;
    p.act = act;
    p.out_f32 = out_f32;
    sp::GemmMaps maps;
    maps.w = wmap;
    maps.x64 = xm.x64;
    maps.x16 = xm.x16;
    if (grp) {
      const double G = groups, N = n_out, K = k_dim, T = t_rows;
      const double xin = (x_group_rows == 0 ? 1.0 : G) * T * K * 2.0;
      grp->rec_begin(kind, G * N * K * 2.0 + xin + G * T * N * (out_f32 ? 4.0 : 2.0) + (bias ? G * N * 4.0 : 0.0),
                     2.0 * G * N * K * T);
    }
    sp::launch_gemm_persistent(maps, p, groups, st);
    if (grp) grp->rec_end();
    return 1;
  }
  sp::GemmParams p{};
  p.g0 = g0;
  p.progress = grp ? grp->ws_active : nullptr;
  p.l2_prefetch = l2_prefetch;
  p.t_dev = t_dev;
  p.n_out = n_out;
  p.k_dim = k_dim;
  p.t_rows = t_rows;
  p.x_group_rows = x_group_rows;
  p.m_tiles = n_out / 128;
  static const bool cluster_on = [] {
    const char* v = getenv("SP_GEMM_CLUSTER");
    return v != nullptr && atoi(v) != 0;  // measured slower at every length: off by default
  }();
  p.cluster = (cluster_on && p.m_tiles % 2 == 0 && t_rows > 16) ? 2 : 1;
  static const int w_keep = [] {
    const char* v = getenv("SP_GEMM_WKEEP");  // evict_last weights when token tiles re-read them:
    return v == nullptr ? 0 : atoi(v);          // measured 1-4 us slower at 160-256 tokens (default off)
  }();
  p.w_keep = w_keep;
  sp::gemm_configure_tiles(t_rows, p.cluster == 2, &p.bn, &p.n_tiles, &p.stages);
  p.epi_warps = sp::gemm_epi_warps(p.bn, p.n_tiles);
  p.splits = splits;
  p.kb_per_split = (k_dim / 64) / splits;
  p.out = out;
  p.out_group_stride = out_gs;
  p.out_split_stride = split_stride;
  p.out_ld = n_out;
  p.bias = bias;
  p.bias_group_stride = bias_gs;
  p.act = act;
  p.out_f32 = out_f32;
  sp::GemmMaps maps;
  maps.w = wmap;
  maps.x64 = xm.x64;
  maps.x16 = xm.x16;
  if (grp) {
    const double G = groups, N = n_out, K = k_dim, T = t_rows;
    const double xin = (x_group_rows == 0 ? 1.0 : G) * T * K * 2.0;
    const double outb = G * T * N * (splits > 1 ? 4.0 * splits : (out_f32 ? 4.0 : 2.0));
    grp->rec_begin(kind, G * N * K * 2.0 + xin + outb + (bias ? G * N * 4.0 : 0.0), 2.0 * G * N * K * T);
  }
  sp::launch_gemm(maps, p, groups, st);
  if (grp) grp->rec_end();
  return 1;
}

// Fused projection + bias + residual + LayerNorm (sp_gemm_ln.cu). Returns 1 (launches).
int run_gemm_ln(sp_group* grp, int kind, const CUtensorMap& wmap, const XMaps& xm, int groups, int n_out, int k_dim,
                int t_rows, int x_group_rows, const sp::LnParams& ln, const int* t_dev, cudaStream_t st) {
  sp::GemmParams p{};
  p.t_dev = t_dev;
  p.n_out = n_out;
  p.k_dim = k_dim;
  p.t_rows = t_rows;
  p.x_group_rows = x_group_rows;
  p.m_tiles = n_out / 128;
  p.splits = 1;
  p.kb_per_split = k_dim / 64;
  p.cluster = 1;
  sp::gemm_configure_tiles(t_rows, false, &p.bn, &p.n_tiles, &p.stages);
  // the row buffer (bn x 129 fp32) reuses the ring after the main loop
  while ((size_t)p.stages * (16384 + p.bn * 128) < (size_t)p.bn * 129 * 4) ++p.stages;
  sp::GemmMaps maps;
  maps.w = wmap;
  maps.x64 = xm.x64;
  maps.x16 = xm.x16;
  if (grp) {
    const double G = groups, N = n_out, K = k_dim, T = t_rows;
    grp->rec_begin(kind, G * N * K * 2.0 + G * T * K * 2.0 + G * T * N * (4.0 + 4.0 + 2.0), 2.0 * G * N * K * T);
  }
  sp::launch_gemm_ln(maps, p, ln, groups, st);
  if (grp) grp->rec_end();
  return 1;
}

// Fused LayerNorm epilogue for a projection: opt-in (SP_LN_FUSE=1). Measured slower at every
// batch-1 length on B200 — one CTA per feature tile with full K leaves only 48-96 CTAs streaming
// weights, while split-K + reduce_ln keeps 144+ streams in flight.
bool use_ln_fused(int m_tiles, int n_tiles, int groups, int k_dim, int hidden) {
  static const int mode = [] {
    const char* v = getenv("SP_LN_FUSE");
    return v ? atoi(v) : 0;
  }();
  static const int min_ctas_long_k = [] {
    const char* v = getenv("SP_LN_FUSE_MIN_CTAS");
    return v ? atoi(v) : 96;
  }();
  if (mode == 0 || m_tiles > 8) return false;
  if (k_dim <= hidden) return true;
  return m_tiles * n_tiles * groups >= min_ctas_long_k;
}

unsigned long long* g_req_trace = nullptr;  // sp_debug_set_request_trace

bool fused_enabled() {  // measured slower than the PDL-chained kernels: opt-in
  static const bool on = [] {
    const char* v = getenv("SP_FUSED");
    return v != nullptr && atoi(v) != 0;
  }();
  return on;
}

// Can this request run as ONE persistent kernel (sp_request.cu)? Short requests only: the
// activations of all tokens must fit one TMEM accumulator column block (<= 128 tokens).
bool fused_ok(const sp_group* g, int n_seqs, int n_tokens_bound, int k) {
  const sp_config& c = g->cfg;
  if (!fused_enabled() || c.kind != SP_KIND_BERT || g->profiling || g->eval_finals || g->eval_prefix) return false;
  if (k < 1 || k > sp::kReqMaxStudents || c.n_layers > sp::kReqMaxLayers) return false;
  if (n_tokens_bound > sp::kReqMaxTokens || n_seqs > n_tokens_bound) return false;
  const int H = c.hidden, F = c.ffn;
  if (F % 128 || k * std::max(3 * H, F) / 128 > sp::kReqMaxTiles) return false;
  const int nc = H / 128, d = H / c.n_heads;
  return (nc == 6 && d == 64) || (nc == 8 && d == 64) || (nc == 1 && d == 32) || (nc == 2 && d == 64);
}

int fused_prepare(sp_group* g) {
  if (g->req_ready) return SP_OK;
  const sp_config& c = g->cfg;
  const int G = sp::sm_count();
  (void)G;
  int rc;
  if ((rc = dev_alloc(g, &g->req_banks, 2 * (size_t)sp::kReqBankInts))) return rc;
  if ((rc = dev_alloc(g, &g->req_epoch, 1))) return rc;
  SP_CUDA(cudaMemset(g->req_banks, 0, 2 * sizeof(int) * sp::kReqBankInts));
  SP_CUDA(cudaMemset(g->req_epoch, 0, sizeof(int)));
  sp::ReqMaps& m = g->req_maps;
  memset(&m, 0, sizeof(m));
  for (int l = 0; l < c.n_layers; ++l) {
    m.w[l][0] = g->m_qkv[l];
    m.w[l][1] = g->m_o[l];
    m.w[l][2] = g->m_f1[l];
    m.w[l][3] = g->m_f2[l];
  }
  m.w_pool = g->m_pool;
  m.x16_64 = g->xm_x16.x64;
  m.x16_16 = g->xm_x16.x16;
  m.ctx_64 = g->xm_ctx.x64;
  m.ctx_16 = g->xm_ctx.x16;
  m.ffn_64 = g->xm_ffn.x64;
  m.ffn_16 = g->xm_ffn.x16;
  m.cls_64 = g->xm_cls.x64;
  m.cls_16 = g->xm_cls.x16;
  g->req_ready = true;
  return SP_OK;
}

int fused_forward(sp_group* g, const int32_t* ids, const int32_t* cu, int n_seqs, int k, float* rep, float* logits,
                  int add_bias, cudaStream_t st) {
  int rc = fused_prepare(g);
  if (rc) return rc;
  const sp_config& c = g->cfg;
  const sp_weights& w = g->w;
  sp::ReqParams p;
  memset(&p, 0, sizeof(p));
  p.ids = ids;
  p.cu = cu;
  p.n_seqs = n_seqs;
  p.k = k;
  p.s_total = c.n_students;
  p.hidden = c.hidden;
  p.ffn = c.ffn;
  p.n_heads = c.n_heads;
  p.n_layers = c.n_layers;
  p.t_cap = c.max_tokens;
  p.b_cap = c.max_seqs;
  p.rows_cap = g->rows_cap;
  p.n_classes = c.n_classes;
  p.add_bias = add_bias;
  p.part_ss = (long long)c.n_students * c.max_tokens * c.hidden;  // g->part: [split][S][T][H]
  p.pool_ss = (long long)c.n_students * g->rows_cap * c.hidden;   // g->final32: [split][S][R][H]
  p.eps = c.ln_eps;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(c.hidden / c.n_heads));
  p.word = static_cast<const half*>(w.word_emb);
  p.pos = static_cast<const half*>(w.pos_emb);
  p.type = static_cast<const half*>(w.type_emb);
  p.word_gs = (long long)c.vocab * c.hidden;
  p.pos_gs = (long long)c.max_pos * c.hidden;
  p.emb_g = w.emb_ln_gamma;
  p.emb_b = w.emb_ln_beta;
  p.b_qkv = w.b_qkv;
  p.b_o = w.b_o;
  p.ln1_g = w.ln1_gamma;
  p.ln1_b = w.ln1_beta;
  p.b_f1 = w.b_ffn1;
  p.b_f2 = w.b_ffn2;
  p.ln2_g = w.ln2_gamma;
  p.ln2_b = w.ln2_beta;
  p.b_pool = w.b_pool;
  p.alpha = w.alpha;
  p.w_cls = w.w_cls;
  p.b_cls = w.b_cls;
  p.x32 = g->x32;
  p.x16 = g->x16;
  p.qkv = g->qkv;
  p.ctx = g->ctx;
  p.ffn_act = g->ffn;
  p.pre = g->part;
  p.cls16 = g->cls16;
  p.pool_part = g->final32;
  p.logits = logits;
  p.rep = rep;
  p.banks = g->req_banks;
  p.epoch = g->req_epoch;
  p.trace = g_req_trace;
  if (!sp::launch_request(g->req_maps, p, sp::sm_count(), st))
    return fail(SP_ECUDA, "request kernel launch: %s", cudaGetErrorString(cudaGetLastError()));
  g->last_launches = 1;
  return SP_OK;
}

bool mlp_fusion_enabled() {  // SP_MLP_FUSE=0 falls back to two launches
  static const bool on = [] {
    const char* v = getenv("SP_MLP_FUSE");
    return v == nullptr || atoi(v) != 0;
  }();
  return on;
}

// FFN1 (+GELU) and FFN2 of layer l as one persistent kernel (sp_mlp.cu); FFN2's raw projection
// lands in g->part (one split) for the LayerNorm kernel.
int run_mlp(sp_group* g, int l, int k, int n_tokens, const int* t_dev, cudaStream_t st, int* splits_b) {
  const sp_config& c = g->cfg;
  const sp_weights& w = g->w;
  const int H = c.hidden, F = c.ffn, T = c.max_tokens;
  const size_t lS = (size_t)l * c.n_students;
  sp::MlpParams p{};
  p.n_a = F;
  p.k_a = H;
  p.n_b = H;
  p.k_b = F;
  int stages = 0;
  sp::gemm_configure_persistent(n_tokens, false, k * (F / 128), sp::sm_count(), false, &p.bn_a, &p.n_tiles_a, &stages);
  sp::gemm_configure_persistent(n_tokens, true, k * (H / 128), sp::sm_count(), false, &p.bn_b, &p.n_tiles_b, &stages);
  sp::mlp_smem_bytes(std::max(p.bn_a, p.bn_b), &p.stages);
  p.groups = k;
  p.t_rows = n_tokens;
  p.x_group_rows = T;
  p.t_dev = t_dev;
  p.out_a = g->ffn;
  p.out_a_gs = (long long)T * F;
  p.out_a_ld = F;
  p.bias_a = w.b_ffn1 + lS * F;
  p.bias_a_gs = F;
  p.out_b = g->part;
  p.out_b_gs = (long long)T * H;
  p.out_b_ld = H;
  p.out_b_ss = (long long)c.n_students * T * H;
  // FFN2 split-K (opt-in SP_MLP_SPLITS=n, 0 = until two units per SM): measured +5..18 us at
  // L = 384..512 — phase B already fills one round (144 deep units at bn = 192), and the static
  // reverse-order dealing puts the extra split units on the CTAs that also ran three FFN1 tiles
  static const int split_env = env_int("SP_MLP_SPLITS", 1);
  const int units_b = k * (H / 128) * p.n_tiles_b;
  int sb = 1;
  if (split_env > 0) {
    sb = split_env;
  } else {
    while (sb < kMaxSplits && units_b * sb < 2 * sp::sm_count() && (F / 64) % (sb + 1) == 0) ++sb;
  }
  if ((F / 64) % sb != 0 || sb > kMaxSplits) sb = 1;
  p.splits_b = sb;
  *splits_b = sb;
  p.done = g->mlp_done;
  sp::MlpMaps m;
  m.w_a = g->m_f1[l];
  m.xa64 = g->xm_x16.x64;
  m.xa16 = g->xm_x16.x16;
  m.w_b = g->m_f2[l];
  m.xb64 = g->xm_ffn.x64;
  m.xb16 = g->xm_ffn.x16;
  const double G = k, Tt = n_tokens;
  g->rec_begin(SP_LAUNCH_GEMM_FFN1, G * 2.0 * F * H * 2.0 + G * Tt * (H * 2.0 + F * 2.0 * 2.0 + H * 4.0),
               2.0 * 2.0 * G * F * H * Tt);
  sp::launch_mlp(m, p, st);
  g->rec_end();
  return 1;
}

// dyn = true (graph capture): n_tokens / max_len are bucket bounds used for grids and tiles; every
// kernel reads the live token count from cu_seqlens[n_seqs] on the device.
// Weight streamer for short requests (see sp_stream.cu). Only where every projection of the request
// reports its progress: the small-T and persistent GEMMs (not the fused MLP / LN / request kernels).
bool weight_stream_on(const sp_group* g, int n_tokens, int k) {
  static const int max_tokens = env_int("SP_WS_MAX_TOKENS", 0);
  static const bool ln_fused = env_int("SP_LN_FUSE", 0) != 0;
  return k > 0 && n_tokens <= max_tokens && n_tokens <= 128 && !ln_fused && !fused_enabled() &&
         4 * g->cfg.n_layers + 1 <= sp::kStreamMaxSegs;
}

int weight_stream_begin(sp_group* g, int k, cudaStream_t st) {
  static const unsigned long long window = (unsigned long long)env_int("SP_WS_WINDOW_MB", 64) << 20;
  static const unsigned long long chunk = (unsigned long long)env_int("SP_WS_CHUNK_KB", 64) << 10;
  static const int ctas = env_int("SP_WS_CTAS", 16);
  static const bool skip_first = env_int("SP_WS_SKIP_FIRST", 1) != 0;
  const sp_config& c = g->cfg;
  const sp_weights& w = g->w;
  const size_t S = c.n_students, H = c.hidden, F = c.ffn;
  sp::StreamPlan plan{};
  auto seg = [&](const void* base, size_t layer_elems, size_t l, size_t per_student) {
    plan.ptr[plan.n] = static_cast<const half*>(base) + l * layer_elems;
    plan.bytes[plan.n] = (unsigned long long)k * per_student * 2;
    plan.total += plan.bytes[plan.n];
    ++plan.n;
  };
  for (int l = 0; l < c.n_layers; ++l) {
    seg(w.w_qkv, S * 3 * H * H, l, 3 * H * H);
    seg(w.w_o, S * H * H, l, H * H);
    seg(w.w_ffn1, S * F * H, l, F * H);
    seg(w.w_ffn2, S * H * F, l, H * F);
  }
  seg(w.w_pool, 0, 0, H * H);
  plan.skip = skip_first ? plan.bytes[0] : 0;
  plan.window = window;
  plan.chunk = chunk;
  plan.max_wait_ns = 2000000ull;
  SP_CUDA(cudaEventRecord(g->ws_fork, st));
  SP_CUDA(cudaStreamWaitEvent(g->ws_stream, g->ws_fork, 0));
  sp::launch_weight_stream(plan, g->ws_state, ctas, g->ws_stream);
  SP_CUDA(cudaEventRecord(g->ws_join, g->ws_stream));
  g->ws_active = g->ws_state;
  return SP_OK;
}

int weight_stream_end(sp_group* g, cudaStream_t st) {
  g->ws_active = nullptr;
  SP_CUDA(cudaStreamWaitEvent(st, g->ws_join, 0));
  return SP_OK;
}

// Kernel chains per request (see bert_forward): opt-in SP_CHAINS=2 for 17..112-token requests.
// Measured: in graph replay -2..-5.5 us at 32..96 tokens, equal at 16, +2.5..8 us at 112..128; in the
// eager launch path (twice the host launches) -1.7% req/s on the bench mix, so off by default.
int request_chains(const sp_group* g, int n_tokens, int k) {
  static const int chains = env_int("SP_CHAINS", 1);
  static const int min_tokens = env_int("SP_CHAINS_MIN_TOKENS", 17);
  static const int max_tokens = env_int("SP_CHAINS_MAX_TOKENS", 112);
  static const bool ln_fused = env_int("SP_LN_FUSE", 0) != 0;
  if (chains < 2 || k < 2 || n_tokens < min_tokens || n_tokens > max_tokens || n_tokens > 128 || ln_fused ||
      g->profiling || g->ws_active)
    return 1;
  return 2;
}

int bert_forward(sp_group* g, const int32_t* ids, const int32_t* cu, int n_seqs, int n_tokens, int max_len, int k,
                 float* rep, float* logits, int add_bias, cudaStream_t st, bool dyn = false) {
  const int n_rows_arg = dyn ? -n_tokens : n_tokens;  // row kernels: negative = live count on device
  const int* t_dev = dyn ? cu + n_seqs : nullptr;
  const sp_config& c = g->cfg;
  const sp_weights& w = g->w;
  const int S = c.n_students, H = c.hidden, F = c.ffn, T = c.max_tokens, B = c.max_seqs;
  const long long xgs = (long long)T * H;
  int launches = 0;
  int pool_splits = 1;
  const half* wq = static_cast<const half*>(w.w_qkv);
  const half* wo = static_cast<const half*>(w.w_o);
  const half* w1 = static_cast<const half*>(w.w_ffn1);
  static const bool pf_on = [] {
    const char* v = getenv("SP_L2_PREFETCH_NEXT");  // measured slower (latency-bound chain): opt-in
    return v != nullptr && atoi(v) != 0;
  }();
  // (ptr, bytes) of fp16 weights the next projection will stream: pulled into L2 by the kernel in between
  struct Pf {
    const void* p;
    unsigned long long n;
  };
  auto pf = [&](const void* p, size_t elems) { return pf_on ? Pf{p, (unsigned long long)elems * 2} : Pf{nullptr, 0}; };
  if (k > 0 && fused_ok(g, n_seqs, n_tokens, k)) {  // short request: one persistent kernel
    g->rec_reset(st);
    return fused_forward(g, ids, cu, n_seqs, k, rep, logits, add_bias, st);
  }
  g->rec_reset(st);
  const double GTH = (double)k * n_tokens * H;
  const bool ws = weight_stream_on(g, n_tokens, k);
  if (ws) {
    const int rc = weight_stream_begin(g, k, st);
    if (rc) return rc;
  }
  if (k > 0) {
    g->rec_begin(SP_LAUNCH_EMBED_LN, GTH * 10.0, 0.0);
    sp::launch_embed_ln(ids, cu, n_seqs, n_rows_arg, k, static_cast<const half*>(w.word_emb),
                        static_cast<const half*>(w.pos_emb), static_cast<const half*>(w.type_emb),
                        (long long)c.vocab * H, (long long)c.max_pos * H, w.emb_ln_gamma, w.emb_ln_beta, H, c.ln_eps,
                        g->x32, g->x16, xgs, st, PF(pf(w.w_qkv, (size_t)k * 3 * H * H)));
    g->rec_end();
    ++launches;
    int bn, n_tiles, stages;
    sp::gemm_configure_tiles(n_tokens, false, &bn, &n_tiles, &stages);
    const long long part_ss = (long long)S * xgs;
    // Student-split request (short requests, SP_CHAINS=2): the students' second half runs as its own
    // kernel chain on a second stream, one projection behind the first, so each chain's latency-bound
    // stages (attention, LayerNorm, fills and drains) overlap the other's weight streaming. Students
    // are independent until the head, which sums them in order after the join.
    const int n_chains = request_chains(g, n_tokens, k);
    const int kc0 = n_chains == 2 ? (k + 1) / 2 : k;
    struct Chain {
      int g0, kc;
      cudaStream_t cs;
    } chains[2] = {{0, kc0, st}, {kc0, k - kc0, g->chain_stream}};
    auto layer = [&](const Chain& ch, int l, bool fork_after_qkv) {
      const int g0 = ch.g0, kc = ch.kc;
      cudaStream_t cs = ch.cs;
      const double GTHc = (double)kc * n_tokens * H;
      const int s_o = choose_splits(kc * (H / 128) * n_tiles, H / 64, kMaxSplits);
      const int s_f = choose_splits(kc * (H / 128) * n_tiles, F / 64, kMaxSplits);
      const size_t lS = (size_t)l * S;
      const long long o16 = (long long)g0 * xgs;  // activation offset of the chain's first student
      launches += run_gemm(g, SP_LAUNCH_GEMM_QKV, g->m_qkv[l], g->xm_x16, kc, 3 * H, H, n_tokens, T, w.b_qkv + lS * 3 * H,
                           3 * H, sp::ACT_NONE, g->qkv, (long long)T * 3 * H, 0, 1, 0, cs, t_dev, g0);
      if (fork_after_qkv) cudaEventRecord(g->chain_fork, cs);
      g->rec_begin(SP_LAUNCH_ATTENTION, GTHc * 8.0, 4.0 * kc * H * g->sum_len_sq);
      launch_attention_any(attn_kind(H / c.n_heads, max_len), g->m_qkv_attn_at[g0], g->m_qkv_kv64_at[g0],
                           g->qkv + (size_t)g0 * T * 3 * H, g->ctx + o16, cu, n_seqs, max_len, kc, c.n_heads,
                           H / c.n_heads, H, T, cs);
      g->rec_end();
      ++launches;
      // O and FFN2 write raw partial sums; the reduce+LN kernel owns bias, residual and LayerNorm
      if (use_ln_fused(H / 128, n_tiles, kc, H, H)) {
        sp::LnParams ln{w.b_o + lS * H, w.ln1_gamma + lS * H, w.ln1_beta + lS * H, c.ln_eps, g->x32, g->x16, xgs,
                        nullptr, 0, cu, n_seqs, H};
        launches += run_gemm_ln(g, SP_LAUNCH_GEMM_O, g->m_o[l], g->xm_ctx, kc, H, H, n_tokens, T, ln, t_dev, cs);
      } else {
        launches += run_gemm(g, SP_LAUNCH_GEMM_O, g->m_o[l], g->xm_ctx, kc, H, H, n_tokens, T, nullptr, H,
                             sp::ACT_NONE, g->part, xgs, 1, s_o, part_ss, cs, t_dev, g0);
        g->rec_begin(SP_LAUNCH_REDUCE_LN, GTHc * (4.0 * s_o + 10.0), 0.0);
        sp::launch_reduce_ln(g->part + o16, s_o, part_ss, w.b_o + (lS + g0) * H, w.ln1_gamma + (lS + g0) * H,
                             w.ln1_beta + (lS + g0) * H, H, c.ln_eps, g->x32 + o16, g->x16 + o16, xgs, n_rows_arg, kc,
                             cu, n_seqs, nullptr, 0, cs, PF(pf(w1 + lS * F * H, (size_t)k * F * H)));
        g->rec_end();
        ++launches;
      }
      // FFN1 + FFN2 as one persistent kernel where both would take the (single-CTA) persistent path
      // (only where FFN2 itself would be a one-split persistent GEMM: measured -2% at L=512, but
      // +3% at L=256 where FFN2's split-K tiles beat the fused kernel's 96-token phase-B tiles)
      const bool mlp = mlp_fusion_enabled() && s_f == 1 && n_tokens >= 129 &&
                       !sp::gemm_persistent_pair(n_tokens, F / 128, kc) &&
                       !sp::gemm_persistent_pair(n_tokens, H / 128, kc) && !use_ln_fused(H / 128, n_tiles, kc, F, H);
      int mlp_splits = 1;
      if (mlp) {
        launches += run_mlp(g, l, kc, n_tokens, t_dev, cs, &mlp_splits);  // (single-chain: >= 129 tokens)
      } else {
        launches += run_gemm(g, SP_LAUNCH_GEMM_FFN1, g->m_f1[l], g->xm_x16, kc, F, H, n_tokens, T, w.b_ffn1 + lS * F,
                             F, sp::ACT_GELU, g->ffn, (long long)T * F, 0, 1, 0, cs, t_dev, g0);
      }
      const bool last = (l == c.n_layers - 1);
      if (!mlp && use_ln_fused(H / 128, n_tiles, kc, F, H)) {
        sp::LnParams ln{w.b_ffn2 + lS * H, w.ln2_gamma + lS * H, w.ln2_beta + lS * H, c.ln_eps, g->x32, g->x16, xgs,
                        last ? g->cls16 : nullptr, (long long)B * H, cu, n_seqs, H};
        launches += run_gemm_ln(g, SP_LAUNCH_GEMM_FFN2, g->m_f2[l], g->xm_ffn, kc, H, F, n_tokens, T, ln, t_dev, cs);
      } else {
        if (!mlp)
          launches += run_gemm(g, SP_LAUNCH_GEMM_FFN2, g->m_f2[l], g->xm_ffn, kc, H, F, n_tokens, T, nullptr, H,
                               sp::ACT_NONE, g->part, xgs, 1, s_f, part_ss, cs, t_dev, g0);
        const int s_ln2 = mlp ? mlp_splits : s_f;  // the fused MLP kernel's FFN2 split-K partials
        g->rec_begin(SP_LAUNCH_REDUCE_LN, GTHc * (4.0 * s_ln2 + 10.0), 0.0);
        sp::launch_reduce_ln(g->part + o16, s_ln2, part_ss, w.b_ffn2 + (lS + g0) * H, w.ln2_gamma + (lS + g0) * H,
                             w.ln2_beta + (lS + g0) * H, H, c.ln_eps, g->x32 + o16, g->x16 + o16, xgs, n_rows_arg,
                             kc, cu, n_seqs, last ? g->cls16 + (long long)g0 * B * H : nullptr, (long long)B * H, cs,
                             PF(last ? pf(w.w_pool, (size_t)k * H * H)
                                     : pf(wq + (lS + S) * 3 * H * H, (size_t)k * 3 * H * H)));
        g->rec_end();
        ++launches;
      }
    };
    // pooler on the CLS rows: tanh(W_p h_CLS + b_p). Few rows: split-K partials (more CTAs stream the
    // pooler weights), finished by the head kernel (one split count for both chains); many rows: one
    // pass with the tanh epilogue.
    const int s_p = n_seqs <= 128 ? choose_splits(k * (H / 128), H / 64, kMaxSplits) : 1;
    pool_splits = s_p;
    auto pool = [&](const Chain& ch) {
      launches += run_gemm(g, SP_LAUNCH_GEMM_POOL, g->m_pool, g->xm_cls, ch.kc, H, H, n_seqs, B,
                           s_p > 1 ? nullptr : w.b_pool, H, sp::ACT_TANH, g->final32, (long long)g->rows_cap * H, 1,
                           s_p, (long long)S * g->rows_cap * H, ch.cs, nullptr, ch.g0);
    };
    for (int l = 0; l < c.n_layers; ++l) {
      layer(chains[0], l, n_chains == 2 && l == 0);
      if (n_chains == 2) {
        if (l == 0) SP_CUDA(cudaStreamWaitEvent(g->chain_stream, g->chain_fork, 0));
        layer(chains[1], l, false);
      }
    }
    pool(chains[0]);
    if (n_chains == 2) {
      pool(chains[1]);
      SP_CUDA(cudaEventRecord(g->chain_join, g->chain_stream));
      SP_CUDA(cudaStreamWaitEvent(st, g->chain_join, 0));
    }
  }
  g->rec_begin(SP_LAUNCH_HEAD, (double)k * n_seqs * H * 4.0 * (pool_splits > 1 ? pool_splits : 1) +
                                   (double)c.n_classes * H * 4.0 + n_seqs * H * 4.0, 0.0);
  sp::launch_head(g->final32, (long long)g->rows_cap * H, (long long)S * g->rows_cap * H,
                  pool_splits > 1 ? pool_splits : 0, w.b_pool, k, w.alpha, w.w_cls, w.b_cls, c.n_classes, H, n_seqs,
                  add_bias, rep, logits, st, g->eval_finals, g->head_flag, g->head_seq);
  g->rec_end();
  ++launches;
  if (ws) {
    const int rc = weight_stream_end(g, st);
    if (rc) return rc;
    ++launches;
  }
  if (g->eval_prefix) {
    sp::launch_prefix_logits(g->eval_finals, k, w.alpha, w.w_cls, w.b_cls, c.n_classes, H, n_seqs, add_bias,
                             g->eval_prefix, st);
    ++launches;
  }
  g->last_launches = launches;
  return SP_OK;
}

bool graphs_enabled() {
  static const bool on = [] {
    const char* v = getenv("SP_GRAPHS");
    return v == nullptr || atoi(v) != 0;
  }();
  return on;
}

// Batch-1 host path: one instantiated graph per 16-token bucket replays the whole forward
// (17 PDL-chained kernels) with a single launch; kernels read the live length from d_cu.
int get_graph(sp_group* g, int n_tokens, int k, int add_bias, cudaGraphExec_t* out) {
  const int bucket = std::min(((n_tokens + 15) / 16) * 16, std::max(16, g->cfg.max_tokens));
  const auto key = std::make_tuple(bucket, k, add_bias);
  auto it = g->graphs.find(key);
  if (it != g->graphs.end()) {
    *out = it->second;
    return SP_OK;
  }
  if (g->cap_stream == nullptr) SP_CUDA(cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking));
  SP_CUDA(cudaStreamBeginCapture(g->cap_stream, cudaStreamCaptureModeThreadLocal));
  const int max_len = std::min(bucket, g->cfg.max_pos);
  // the request's copies are graph nodes too: pinned [cu | ids] staging -> device (bucket size; the
  // kernels read the live length from cu), forward, logits -> pinned
  cudaMemcpyAsync(g->d_cu, g->h_stage, sizeof(int32_t) * ((size_t)g->cu_pad + std::min(bucket, g->cfg.max_tokens)),
                  cudaMemcpyHostToDevice, g->cap_stream);
  g->head_flag = g->d_flag;  // the head kernel publishes the request's sequence number (staged in
  g->head_seq = g->d_cu + g->cu_pad - 1;  // the last cu slot) after writing the mapped logits
  int rc = bert_forward(g, g->d_ids, g->d_cu, 1, bucket, max_len, k, nullptr, g->d_out, add_bias, g->cap_stream, true);
  g->head_flag = nullptr;
  g->head_seq = nullptr;
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(g->cap_stream, &graph);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(SP_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(SP_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  g->graph_launches = g->last_launches;
  g->graphs[key] = exec;
  *out = exec;
  return SP_OK;
}

// Device-buffer batch-1 path: the same bucket graphs without the host copies; the forward reads
// the group's own device staging (filled by two device-to-device copies) and writes `logits`.
int get_graph_dev(sp_group* g, int n_tokens, int k, int add_bias, float* logits, cudaGraphExec_t* out) {
  const int bucket = std::min(((n_tokens + 15) / 16) * 16, std::max(16, g->cfg.max_tokens));
  const auto key = std::make_tuple(bucket, k, add_bias, reinterpret_cast<uintptr_t>(logits));
  auto it = g->dgraphs.find(key);
  if (it != g->dgraphs.end()) {
    *out = it->second;
    return SP_OK;
  }
  if (g->cap_stream == nullptr) SP_CUDA(cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking));
  SP_CUDA(cudaStreamBeginCapture(g->cap_stream, cudaStreamCaptureModeThreadLocal));
  const int max_len = std::min(bucket, g->cfg.max_pos);
  int rc = bert_forward(g, g->d_ids, g->d_cu, 1, bucket, max_len, k, nullptr, logits, add_bias, g->cap_stream, true);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(g->cap_stream, &graph);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(SP_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(SP_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  g->graph_launches = g->last_launches;
  g->dgraphs[key] = exec;
  *out = exec;
  return SP_OK;
}

int dense_forward(sp_group* g, const half* x, int n_rows, int k, float* rep, float* logits, int add_bias,
                  cudaStream_t st, const XMaps& xin_maps) {
  const sp_config& c = g->cfg;
  const sp_weights& w = g->w;
  const int S = c.n_students, H = c.hidden, T = c.max_tokens;
  const long long hgs = (long long)T * H;
  const long long fgs = (long long)g->rows_cap * H;
  int launches = 0;
  g->rec_reset(st);
  if (k > 0) {
    // input_proj: every student reads the same rows (x_group_rows = 0)
    half* bufs[2] = {g->x16, g->ctx};
    const XMaps* maps[2] = {&g->xm_ha, &g->xm_hb};
    launches += run_gemm(g, SP_LAUNCH_GEMM_DENSE, g->m_in, xin_maps, k, H, c.d_in, n_rows, 0, w.b_in, H, sp::ACT_TANH, bufs[0], hgs, 0, 1, 0, st);
    int cur = 0;
    for (int l = 0; l < c.n_layers; ++l) {
      const bool last = (l == c.n_layers - 1);
      const size_t lS = (size_t)l * S;
      void* out = last ? static_cast<void*>(g->final32) : static_cast<void*>(bufs[cur ^ 1]);
      launches += run_gemm(g, SP_LAUNCH_GEMM_DENSE, g->m_layers[l], *maps[cur], k, H, H, n_rows, T, w.b_layers + lS * H, H, sp::ACT_TANH, out,
                           last ? fgs : hgs, last ? 1 : 0, 1, 0, st);
      cur ^= 1;
    }
  }
  g->rec_begin(SP_LAUNCH_HEAD, (double)k * n_rows * H * 4.0 + (double)c.n_classes * H * 4.0, 0.0);
  sp::launch_head(g->final32, fgs, 0, 0, nullptr, k, w.alpha, w.w_cls, w.b_cls, c.n_classes, H, n_rows, add_bias, rep,
                  logits, st, g->eval_finals);
  g->rec_end();
  ++launches;
  if (g->eval_prefix) {
    sp::launch_prefix_logits(g->eval_finals, k, w.alpha, w.w_cls, w.b_cls, c.n_classes, H, n_rows, add_bias,
                             g->eval_prefix, st);
    ++launches;
  }
  g->last_launches = launches;
  (void)x;
  return SP_OK;
}

}  // namespace

extern "C" {

int sp_group_forward(sp_group* g, const int32_t* ids, const int32_t* cu_seqlens, int32_t n_seqs, int32_t n_tokens,
                     int32_t max_seq_len, int32_t k_active, float* rep_out, float* logits_out, int32_t add_bias,
                     void* stream) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  const sp_config& c = g->cfg;
  if (c.kind != SP_KIND_BERT) return fail(SP_EINVAL, "sp_group_forward needs a BERT-kind group");
  if (k_active < 0 || k_active > c.n_students)
    return fail(SP_EINVAL, "k=%d out of range 0..%d", k_active, c.n_students);
  if (n_seqs < 1 || n_seqs > c.max_seqs) return fail(SP_EINVAL, "n_seqs=%d outside 1..%d", n_seqs, c.max_seqs);
  if (n_tokens < n_seqs || n_tokens > c.max_tokens)
    return fail(SP_EINVAL, "n_tokens=%d outside %d..%d", n_tokens, n_seqs, c.max_tokens);
  if (max_seq_len < 1 || max_seq_len > c.max_pos || max_seq_len > n_tokens)
    return fail(SP_EINVAL, "max_seq_len=%d outside 1..%d", max_seq_len, c.max_pos);
  if (!ids || !cu_seqlens || !logits_out) return fail(SP_EINVAL, "null buffer");
  cudaSetDevice(g->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (g->profiling) {  // exact attention flops need the lengths (profiling already perturbs timing)
    std::vector<int32_t> h(n_seqs + 1);
    SP_CUDA(cudaMemcpyAsync(h.data(), cu_seqlens, sizeof(int32_t) * (n_seqs + 1), cudaMemcpyDeviceToHost, st));
    SP_CUDA(cudaStreamSynchronize(st));
    g->sum_len_sq = 0.0;
    for (int b = 0; b < n_seqs; ++b) g->sum_len_sq += double(h[b + 1] - h[b]) * double(h[b + 1] - h[b]);
  }
  int rc = bert_forward(g, ids, cu_seqlens, n_seqs, n_tokens, max_seq_len, k_active, rep_out, logits_out, add_bias, st);
  if (rc) return rc;
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_group_forward_dense(sp_group* g, const void* x, int32_t n_rows, int32_t k_active, float* rep_out,
                           float* logits_out, int32_t add_bias, void* stream) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  const sp_config& c = g->cfg;
  if (c.kind != SP_KIND_DENSE) return fail(SP_EINVAL, "sp_group_forward_dense needs a dense-kind group");
  if (k_active < 0 || k_active > c.n_students)
    return fail(SP_EINVAL, "k=%d out of range 0..%d", k_active, c.n_students);
  if (n_rows < 1 || n_rows > c.max_tokens) return fail(SP_EINVAL, "n_rows=%d outside 1..%d", n_rows, c.max_tokens);
  if (!x || !logits_out) return fail(SP_EINVAL, "null buffer");
  cudaSetDevice(g->device);
  XMaps xm;
  if (!make_xmaps(&xm, x, (uint64_t)n_rows, (uint64_t)c.d_in))
    return fail(SP_EINVAL, "input tensor map failed (x must be 16-byte aligned fp16 [n_rows][d_in])");
  int rc = dense_forward(g, static_cast<const half*>(x), n_rows, k_active, rep_out, logits_out, add_bias,
                         static_cast<cudaStream_t>(stream), xm);
  if (rc) return rc;
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

// Training-side evaluation: route the per-student finals / prefix logits of one forward call.
static int eval_begin(sp_group* g, float* finals_out, float* prefix_out) {
  if (!finals_out && !prefix_out) return fail(SP_EINVAL, "finals_out and prefix_logits_out are both null");
  if (!finals_out && g->eval_scratch == nullptr) {
    int rc = dev_alloc(g, &g->eval_scratch, (size_t)g->cfg.n_students * g->rows_cap * g->cfg.hidden);
    if (rc) return rc;
  }
  g->eval_finals = finals_out ? finals_out : g->eval_scratch;
  g->eval_prefix = prefix_out;
  return SP_OK;
}
static void eval_end(sp_group* g) {
  g->eval_finals = nullptr;
  g->eval_prefix = nullptr;
}

int sp_group_forward_eval(sp_group* g, const int32_t* ids, const int32_t* cu_seqlens, int32_t n_seqs,
                          int32_t n_tokens, int32_t max_seq_len, int32_t k_active, float* finals_out,
                          float* prefix_logits_out, void* stream) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  if (k_active < 1 || k_active > g->cfg.n_students)
    return fail(SP_EINVAL, "k=%d out of range 1..%d", k_active, g->cfg.n_students);
  cudaSetDevice(g->device);
  int rc = eval_begin(g, finals_out, prefix_logits_out);
  if (rc) return rc;
  rc = sp_group_forward(g, ids, cu_seqlens, n_seqs, n_tokens, max_seq_len, k_active, nullptr, g->d_logits, 1, stream);
  eval_end(g);
  return rc;
}

int sp_group_forward_dense_eval(sp_group* g, const void* x, int32_t n_rows, int32_t k_active, float* finals_out,
                                float* prefix_logits_out, void* stream) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  if (k_active < 1 || k_active > g->cfg.n_students)
    return fail(SP_EINVAL, "k=%d out of range 1..%d", k_active, g->cfg.n_students);
  cudaSetDevice(g->device);
  int rc = eval_begin(g, finals_out, prefix_logits_out);
  if (rc) return rc;
  rc = sp_group_forward_dense(g, x, n_rows, k_active, nullptr, g->d_logits, 1, stream);
  eval_end(g);
  return rc;
}

int sp_group_forward_host(sp_group* g, const int32_t* ids, const int32_t* cu, int32_t n_seqs, int32_t n_tokens,
                          int32_t k_active, float* logits_out, int32_t add_bias, void* stream) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  const sp_config& c = g->cfg;
  if (c.kind != SP_KIND_BERT) return fail(SP_EINVAL, "sp_group_forward_host needs a BERT-kind group");
  if (!ids || !cu || !logits_out) return fail(SP_EINVAL, "null buffer");
  if (n_seqs < 1 || n_seqs > c.max_seqs) return fail(SP_EINVAL, "n_seqs=%d outside 1..%d", n_seqs, c.max_seqs);
  if (cu[0] != 0) return fail(SP_EINVAL, "cu_seqlens[0] must be 0");
  int max_len = 0;
  g->sum_len_sq = 0.0;
  for (int b = 0; b < n_seqs; ++b) {
    const int len = cu[b + 1] - cu[b];
    g->sum_len_sq += double(len) * double(len);
    if (len < 1) return fail(SP_EINVAL, "sequence %d is empty or cu_seqlens decreases", b);
    if (len > c.max_pos) return fail(SP_EINVAL, "sequence %d has %d tokens > max_pos %d", b, len, c.max_pos);
    max_len = std::max(max_len, len);
  }
  if (cu[n_seqs] != n_tokens) return fail(SP_EINVAL, "cu_seqlens[-1]=%d != n_tokens=%d", cu[n_seqs], n_tokens);
  if (n_tokens > c.max_tokens) return fail(SP_EINVAL, "n_tokens=%d > capacity %d", n_tokens, c.max_tokens);
  for (int t = 0; t < n_tokens; ++t)
    if (ids[t] < 0 || ids[t] >= c.vocab) return fail(SP_EINVAL, "token id %d at %d outside vocab", ids[t], t);
  cudaSetDevice(g->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // short requests run as one persistent kernel (no graph needed); longer ones replay a graph
  const bool use_graph = graphs_enabled() && n_seqs == 1 && !g->profiling && !fused_ok(g, n_seqs, n_tokens, k_active);
  cudaGraphExec_t exec = nullptr;
  if (use_graph) {
    int rc = get_graph(g, n_tokens, k_active, add_bias, &exec);
    if (rc) return rc;
  }
  // pinned staging ([cu | ids] block; the caller's buffers may be pageable). Every call ends with a
  // stream sync, so the previous request no longer reads h_stage.
  memcpy(g->h_stage, cu, sizeof(int32_t) * (n_seqs + 1));
  memcpy(g->h_stage + g->cu_pad, ids, sizeof(int32_t) * n_tokens);
  if (use_graph) {  // H2D copy and forward are nodes of the bucket's graph; logits land in mapped memory
    const int seq = (g->seq = g->seq == 0x7fffffff ? 1 : g->seq + 1);
    g->h_stage[g->cu_pad - 1] = seq;
    SP_CUDA(cudaGraphLaunch(exec, st));
    g->last_launches = g->graph_launches;
    const size_t flag_off = ((sizeof(float) * (size_t)c.n_classes + 127) / 128) * 128;
    volatile int* flag = reinterpret_cast<volatile int*>(static_cast<uint8_t*>(g->h_mapped) + flag_off);
    for (unsigned spins = 1; *flag != seq; ++spins) {
      if ((spins & 0xfff) == 0) {  // every few microseconds: surface a failed launch instead of spinning
        const cudaError_t e = cudaStreamQuery(st);
        if (e != cudaSuccess && e != cudaErrorNotReady) return fail(SP_ECUDA, "forward: %s", cudaGetErrorString(e));
        if (e == cudaSuccess && *flag != seq) return fail(SP_ECUDA, "forward finished without publishing its logits");
      }
    }
    const volatile float* out = static_cast<const volatile float*>(g->h_mapped);
    for (int i = 0; i < c.n_classes; ++i) logits_out[i] = out[i];
    return SP_OK;
  }
  SP_CUDA(cudaMemcpyAsync(g->d_cu, g->h_stage, sizeof(int32_t) * ((size_t)g->cu_pad + n_tokens),
                          cudaMemcpyHostToDevice, st));
  {
    int rc = bert_forward(g, g->d_ids, g->d_cu, n_seqs, n_tokens, max_len, k_active, nullptr, g->d_logits, add_bias, st);
    if (rc) return rc;
  }
  SP_CUDA(cudaGetLastError());
  SP_CUDA(cudaMemcpyAsync(g->h_logits, g->d_logits, sizeof(float) * n_seqs * c.n_classes, cudaMemcpyDeviceToHost,
                          st));
  SP_CUDA(cudaStreamSynchronize(st));
  memcpy(logits_out, g->h_logits, sizeof(float) * n_seqs * c.n_classes);
  return SP_OK;
}

int sp_op_gemm(const void* w, const void* x, int32_t groups, int32_t n_out, int32_t k_dim, int32_t t_rows,
               int32_t x_group_rows, int32_t x_rows_total, const float* bias, int32_t act, void* out, int32_t out_f32,
               int32_t splits, void* stream) {
  if (!w || !x || !out) return fail(SP_EINVAL, "null buffer");
  if (groups < 1 || n_out < 128 || n_out % 128 || k_dim < 64 || k_dim % 64 || t_rows < 1)
    return fail(SP_EINVAL, "bad gemm shape groups=%d n_out=%d k=%d t=%d", groups, n_out, k_dim, t_rows);
  if (splits < 1 || (k_dim / 64) % splits) return fail(SP_EINVAL, "splits=%d must divide k/64", splits);
  if (act < 0 || act > 2) return fail(SP_EINVAL, "unknown activation %d", act);
  CUtensorMap wm;
  XMaps xm;
  if (!make_map(&wm, w, (uint64_t)groups * n_out, k_dim, 128) || !make_xmaps(&xm, x, x_rows_total, k_dim))
    return fail(SP_EINVAL, "tensor-map creation failed");
  const long long ogs = (long long)t_rows * n_out;
  run_gemm(nullptr, 0, wm, xm, groups, n_out, k_dim, t_rows, x_group_rows, bias, n_out, act, out, ogs, splits > 1 ? 1 : out_f32,
           splits, ogs * groups, static_cast<cudaStream_t>(stream));
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_debug_set_gemm_trace(void* device_buf) {
  sp::set_gemm_trace(static_cast<unsigned long long*>(device_buf));
  return SP_OK;
}

int sp_debug_set_attn_trace(void* device_buf) {
  sp::set_attn_trace(static_cast<unsigned long long*>(device_buf));
  return SP_OK;
}

int sp_debug_gemm_trace_launches(int32_t* ctas_per_launch, int32_t max_launches) {
  return sp::gemm_trace_counts(ctas_per_launch, max_launches);
}

int sp_op_attention(const void* qkv, void* ctx, const int32_t* cu_seqlens, int32_t n_seqs, int32_t max_seq_len,
                    int32_t groups, int32_t n_heads, int32_t head_dim, int32_t group_rows, void* stream) {
  if (!qkv || !ctx || !cu_seqlens) return fail(SP_EINVAL, "null buffer");
  if (head_dim != 32 && head_dim != 64) return fail(SP_EINVAL, "head_dim must be 32 or 64");
  if (n_seqs < 1 || groups < 1 || n_heads < 1 || max_seq_len < 1) return fail(SP_EINVAL, "bad attention shape");
  const int hidden = n_heads * head_dim;
  const int kind = attn_kind(head_dim, max_seq_len);
  CUtensorMap m{}, m64{};
  if (kind != 0 && (!make_map(&m, qkv, (uint64_t)groups * group_rows, 3 * hidden, 128) ||
                    !make_map(&m64, qkv, (uint64_t)groups * group_rows, 3 * hidden, 64)))
    return fail(SP_EINVAL, "attention tensor map failed");
  launch_attention_any(kind, m, m64, static_cast<const half*>(qkv), static_cast<half*>(ctx), cu_seqlens, n_seqs,
                       max_seq_len, groups, n_heads, head_dim, hidden, group_rows, static_cast<cudaStream_t>(stream));
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

}  // extern "C"

extern "C" int sp_debug_set_request_trace(void* buf) {
  g_req_trace = static_cast<unsigned long long*>(buf);
  return SP_OK;
}

extern "C" int sp_group_forward_graph(sp_group* g, const int32_t* ids, const int32_t* cu_seqlens, int32_t n_tokens,
                                      int32_t k_active, float* logits_out, int32_t add_bias, void* stream) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  const sp_config& c = g->cfg;
  if (c.kind != SP_KIND_BERT) return fail(SP_EINVAL, "sp_group_forward_graph needs a BERT-kind group");
  if (!ids || !cu_seqlens || !logits_out) return fail(SP_EINVAL, "null buffer");
  if (k_active < 1 || k_active > c.n_students) return fail(SP_EINVAL, "k=%d out of range 1..%d", k_active, c.n_students);
  if (n_tokens < 1 || n_tokens > c.max_tokens || n_tokens > c.max_pos)
    return fail(SP_EINVAL, "n_tokens=%d outside 1..%d", n_tokens, std::min(c.max_tokens, c.max_pos));
  if (g->profiling || !graphs_enabled() || fused_ok(g, 1, n_tokens, k_active))
    return sp_group_forward(g, ids, cu_seqlens, 1, n_tokens, n_tokens, k_active, nullptr, logits_out, add_bias, stream);
  cudaSetDevice(g->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaGraphExec_t exec = nullptr;
  int rc = get_graph_dev(g, n_tokens, k_active, add_bias, logits_out, &exec);
  if (rc) return rc;
  SP_CUDA(cudaMemcpyAsync(g->d_cu, cu_seqlens, 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  SP_CUDA(cudaMemcpyAsync(g->d_ids, ids, sizeof(int32_t) * n_tokens, cudaMemcpyDeviceToDevice, st));
  SP_CUDA(cudaGraphLaunch(exec, st));
  g->last_launches = g->graph_launches;
  return SP_OK;
}

extern "C" int sp_group_prepare_graphs(sp_group* g, int32_t max_tokens, int32_t k_active, int32_t add_bias) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  if (g->cfg.kind != SP_KIND_BERT) return fail(SP_EINVAL, "graphs serve BERT-kind groups");
  if (k_active < 0 || k_active > g->cfg.n_students) return fail(SP_EINVAL, "k out of range");
  if (!graphs_enabled()) return SP_OK;
  cudaSetDevice(g->device);
  const int top = std::min(max_tokens, g->cfg.max_tokens);
  for (int t = 16; t - 15 <= top; t += 16) {
    if (k_active > 0 && fused_ok(g, 1, t, k_active)) {  // served by the persistent kernel
      int rc = fused_prepare(g);
      if (rc) return rc;
      continue;
    }
    cudaGraphExec_t exec;
    int rc = get_graph(g, t, k_active, add_bias, &exec);
    if (rc) return rc;
  }
  return SP_OK;
}

