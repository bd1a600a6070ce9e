// sp_runtime.cu — C-ABI runtime: group construction (weight snapshot + TMA descriptors + HBM
// workspace) and the per-request launch sequence of the student-group forward.
//
// Every activation a projection reads (LayerNorm outputs, attention context, GELU output, the CLS
// rows, the dense kind's hidden states) lives in HBM as an fp16 (hi, lo) pair — two equal-shaped
// planes of one allocation, lo = fp16(x - hi) — and the GEMMs issue one tcgen05 MMA per term into
// the same fp32 accumulator (sp_device.cuh split_half2). Weights are fp16 and exact on both sides
// (weights.py), so the operands carry ~22 significant bits and the logits meet the north star's
// 1e-3 bar on every seed.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
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
// box_cols 64 (128-byte rows, SWIZZLE_128B) or 32 (64-byte rows, SWIZZLE_64B: head_dim-32 attention)
bool make_map(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows,
              uint32_t box_cols = 64) {
  auto fn = encode_fn();
  if (fn == nullptr || ptr == nullptr || rows == 0) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Token-side operand of a projection: hi term (and lo term, when hilo) as {64, 64} / {64, 16} boxes.
struct XMaps {
  CUtensorMap x64, x16, xl64, xl16;
  bool hilo = false;
};

bool make_xmaps(XMaps* m, const void* hi, const void* lo, uint64_t rows, uint64_t cols) {
  m->hilo = lo != nullptr;
  bool ok = make_map(&m->x64, hi, rows, cols, 64) && make_map(&m->x16, hi, rows, cols, 16);
  if (lo) ok = ok && make_map(&m->xl64, lo, rows, cols, 64) && make_map(&m->xl16, lo, rows, cols, 16);
  else {
    m->xl64 = m->x64;
    m->xl16 = m->x16;
  }
  return ok;
}

// Split-K count of a projection with few output tiles: balance the CTAs over the SMs (the makespan
// in k-blocks of the busiest slot, plus a small cost per extra partial). Two small-kernel CTAs
// (<= 110 KiB smem each) share an SM and stream concurrently, so the slots are 2 x 148: a
// single-token-tile projection takes 4 splits / 192 CTAs rather than 3 / 144 (-1.5..-3 us per
// request at every length, measured) — for token tiles of <= 64 columns, where the weights
// dominate the traffic; wider tiles keep one slot per SM (two 112-column CTAs per SM measured
// slower at 320-384 tokens). With >= 1 tile per SM the one-split persistent path wins.
int choose_splits(int units, int nkb, int smax, int bn) {
  if (units >= 148) return 1;
  const int slots = bn <= 64 ? 296 : 148;
  int best = 1;
  long long best_cost = 0x7fffffffffffll;
  for (int s = 1; s <= smax; ++s) {
    if (nkb % s || (s > 1 && nkb / s < 2)) continue;
    const long long ctas = (long long)units * s;
    const long long per_sm = (ctas + slots - 1) / slots;
    const long long cost = per_sm * (nkb / s) * 4 + s;
    if (cost < best_cost) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

constexpr int kMaxSplits = 4;

}  // namespace

namespace sp {
int report_error(int code, const char* msg) { return fail(code, "%s", msg); }
}  // namespace sp

struct sp_group {
  sp_config cfg;
  sp_weights w;
  int device = 0;
  int rows_cap = 0;  // max(max_tokens, max_seqs)
  // workspace; "[2]" planes are the (hi, lo) terms of a GEMM operand, lo at +*_lo elements
  half* x16 = nullptr;     // [2][S][max_tokens][H] LayerNorm output (QKV / FFN1 operand)
  half* qkv = nullptr;     // [2][S][max_tokens][3H]: hi plane, then the lo plane at qkv_lo
  long long qkv_lo = 0;
  half* ctx = nullptr;     // [2][S][max_tokens][H] attention context (O operand)
  half* ffn = nullptr;     // [2][S][max_tokens][F] GELU output (FFN2 operand)
  float* part = nullptr;   // [kMaxSplits][S][max_tokens][H] split-K partials
  half* cls16 = nullptr;   // [2][S][max_seqs][H] CLS rows (pooler operand)
  // the last layer on the CLS rows only (B = max_seqs rows per student)
  float* xc32 = nullptr;   // [S][B][H] residual stream of the CLS rows
  half* cln = nullptr;     // [2][S][B][H] LayerNorm-1 output of the CLS rows (FFN1 operand)
  half* ctxc = nullptr;    // [2][S][B][H] CLS-query attention context (O operand)
  half* ffnc = nullptr;    // [2][S][B][F] GELU output of the CLS rows (FFN2 operand)
  float* partc = nullptr;  // [kMaxSplits][S][B][H] split-K partials of the CLS-row projections
  half* qc = nullptr;      // [S][B][H] last-layer query of the CLS rows (long requests)
  long long x_lo = 0, ctx_lo = 0, ffn_lo = 0, cls_lo = 0, cf_lo = 0;  // cf_lo: lo offset of ffnc
  float* final32 = nullptr;  // [kMaxSplits][S][rows_cap][H] per-student final representation / pooler partials
  int32_t* d_ids = nullptr;  // staging block [cu_pad | ids]: d_cu = block, d_ids = block + cu_pad
  int32_t* d_cu = nullptr;
  int cu_pad = 0;              // max_seqs + 1 rounded up to 32 ints (128 B)
  int32_t* h_stage = nullptr;  // pinned mirror of the staging block: one H2D copy per request
  float* h_logits = nullptr;   // pinned logits landing buffer
  // batch-1 host path without a stream sync: the head kernel writes the logits into mapped pinned
  // memory, then the request's sequence number (staged with its ids) into a mapped flag the host
  // polls; the graph has no device-to-host copy node
  void* h_mapped = nullptr;  // [logits f32 x n_classes | pad | flag int]
  float* d_out = nullptr;    // device alias of the logits slot
  int* d_flag = nullptr;     // device alias of the flag
  int seq = 0;
  int* head_flag = nullptr;  // set while capturing a host-path graph
  const int* head_seq = nullptr;
  float* d_logits = nullptr;  // [rows_cap][C] device logits (eager host path, eval, device-graph slot)
  int* mlp_done = nullptr;    // fused FFN kernel: FFN1 tiles finished per student + exit counter
  std::vector<void*> allocs;
  // tensor maps
  std::vector<CUtensorMap> m_qkv, m_o, m_f1, m_f2, m_layers, m_layers_lo;
  CUtensorMap m_pool, m_in, m_in_lo;
  bool dense_whilo = false;  // dense weights carry their lo terms (w_in_lo / w_layers_lo)
  CUtensorMap m_qkv_attn;  // qkv buffer viewed with a {64, 128} box (tensor-core attention)
  CUtensorMap m_qkv_kv64;  // the same with a {64, 64} box (64-key chunks of the three-CTA kernel)
  XMaps xm_x16, xm_ctx, xm_ffn, xm_cls, xm_ha, xm_hb, xm_cln, xm_ctxc, xm_ffnc;
  half* ha = nullptr;  // dense kind: hidden-state ping-pong [2][S][T][H] each
  half* hb = nullptr;
  long long h_lo = 0;
  int last_launches = 0;
  // CUDA graphs of the batch-1 paths, keyed by (16-token bucket, k_active, add_bias)
  std::map<std::tuple<int, int, int>, cudaGraphExec_t> graphs;   // host path (mapped logits + flag)
  std::map<std::tuple<int, int, int>, cudaGraphExec_t> dgraphs;  // device path (logits in d_logits)
  cudaStream_t cap_stream = nullptr;
  int graph_launches = 0;    // kernels per graph replay
  double sum_len_sq = 0.0;   // sum_b L_b^2 of the current request (attention flops)
  // training-side evaluation outputs of the current sp_group_forward*_eval call (else null)
  float* eval_finals = nullptr;   // [k][rows][H]
  float* eval_prefix = nullptr;   // [k][rows][C]
  float* eval_scratch = nullptr;  // finals when the caller only asks for prefix logits
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
  int tok_cap() const { return std::min(cfg.max_tokens, cfg.kind == SP_KIND_BERT ? cfg.max_pos : cfg.max_tokens); }
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
  g->graphs.clear();
  g->dgraphs.clear();
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
  if ((rc = dev_alloc(g, &g->mlp_done, sp::kMlpMaxStudents + 1))) return bail(rc);
  if (cudaMemset(g->mlp_done, 0, sizeof(int) * (sp::kMlpMaxStudents + 1)) != cudaSuccess)
    return bail(fail(SP_ECUDA, "memset"));

  if (c.kind == SP_KIND_BERT) {
    if (!w.word_emb || !w.pos_emb || !w.type_emb || !w.emb_ln_gamma || !w.emb_ln_beta || !w.w_qkv || !w.b_qkv ||
        !w.w_o || !w.b_o || !w.ln1_gamma || !w.ln1_beta || !w.w_ffn1 || !w.b_ffn1 || !w.w_ffn2 || !w.b_ffn2 ||
        !w.ln2_gamma || !w.ln2_beta || !w.w_pool || !w.b_pool || !w.alpha || !w.w_cls || !w.b_cls)
      return bail(fail(SP_EINVAL, "missing BERT weight pointer"));
    g->x_lo = (long long)(S * T * H);
    g->ctx_lo = g->x_lo;
    g->ffn_lo = (long long)(S * T * F);
    g->cls_lo = (long long)(S * B * H);
    if ((rc = dev_alloc(g, &g->x16, 2 * S * T * H))) return bail(rc);
    g->qkv_lo = (long long)S * T * 3 * H;
    if ((rc = dev_alloc(g, &g->qkv, 2 * S * T * 3 * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->ctx, 2 * S * T * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->ffn, 2 * S * T * F))) return bail(rc);
    if ((rc = dev_alloc(g, &g->part, (size_t)kMaxSplits * S * T * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->cls16, 2 * S * B * H))) return bail(rc);
    g->cf_lo = (long long)(S * B * F);
    if ((rc = dev_alloc(g, &g->xc32, S * B * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->cln, 2 * S * B * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->ctxc, 2 * S * B * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->ffnc, 2 * S * B * F))) return bail(rc);
    if ((rc = dev_alloc(g, &g->partc, (size_t)kMaxSplits * S * B * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->qc, 2 * S * B * H))) return bail(rc);  // (hi, lo)

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
    ok &= make_xmaps(&g->xm_x16, g->x16, g->x16 + g->x_lo, S * T, H);
    ok &= make_xmaps(&g->xm_ctx, g->ctx, g->ctx + g->ctx_lo, S * T, H);
    ok &= make_xmaps(&g->xm_ffn, g->ffn, g->ffn + g->ffn_lo, S * T, F);
    ok &= make_xmaps(&g->xm_cls, g->cls16, g->cls16 + g->cls_lo, S * B, H);
    ok &= make_xmaps(&g->xm_cln, g->cln, g->cln + g->cls_lo, S * B, H);
    ok &= make_xmaps(&g->xm_ctxc, g->ctxc, g->ctxc + g->cls_lo, S * B, H);
    ok &= make_xmaps(&g->xm_ffnc, g->ffnc, g->ffnc + g->cf_lo, S * B, F);
    const uint32_t head_box = (H / c.n_heads == 32) ? 32 : 64;  // head_dim-32 tiles: 64-byte rows
    // over both planes: a lo tile is the hi tile's rows + S * T
    ok &= make_map(&g->m_qkv_attn, g->qkv, 2 * S * T, 3 * H, 128, head_box);
    ok &= make_map(&g->m_qkv_kv64, g->qkv, 2 * S * T, 3 * H, 64, head_box);
    // rows past a request's tokens are read (masked) by the attention tiles: keep them finite
    if (cudaMemset(g->qkv, 0, 2 * S * T * 3 * H * sizeof(half)) != cudaSuccess) ok = false;
    if (!ok) return bail(fail(SP_EINVAL, "tensor-map creation failed (pointer alignment / shape)"));
  } else {
    if (!w.w_in || !w.b_in || !w.w_layers || !w.b_layers || !w.alpha || !w.w_cls || !w.b_cls)
      return bail(fail(SP_EINVAL, "missing dense weight pointer"));
    g->h_lo = (long long)(S * T * H);
    if ((rc = dev_alloc(g, &g->ha, 2 * S * T * H))) return bail(rc);
    if ((rc = dev_alloc(g, &g->hb, 2 * S * T * H))) return bail(rc);
    const auto* wl = static_cast<const half*>(w.w_layers);
    g->m_layers.resize(c.n_layers);
    bool ok = make_map(&g->m_in, w.w_in, S * H, c.d_in, 128);
    for (int l = 0; l < c.n_layers; ++l) ok &= make_map(&g->m_layers[l], wl + (size_t)l * S * H * H, S * H, H, 128);
    if ((w.w_in_lo == nullptr) != (w.w_layers_lo == nullptr))
      return bail(fail(SP_EINVAL, "w_in_lo and w_layers_lo must be given together"));
    g->dense_whilo = w.w_in_lo != nullptr;
    if (g->dense_whilo) {
      const auto* wll = static_cast<const half*>(w.w_layers_lo);
      g->m_layers_lo.resize(c.n_layers);
      ok &= make_map(&g->m_in_lo, w.w_in_lo, S * H, c.d_in, 128);
      for (int l = 0; l < c.n_layers; ++l)
        ok &= make_map(&g->m_layers_lo[l], wll + (size_t)l * S * H * H, S * H, H, 128);
    }
    ok &= make_xmaps(&g->xm_ha, g->ha, g->ha + g->h_lo, S * T, H);
    ok &= make_xmaps(&g->xm_hb, g->hb, g->hb + g->h_lo, S * T, H);
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

// Attention kernel by length: 0 = mma.sync (sp_attn.cu; head_dim 32), 1 = two-pass tcgen05
// (sp_attn_tc.cu), 2 = single-pass tcgen05, two CTAs per SM, 3 = the same with 64-key chunks at
// three CTAs per SM (sp_attn_tc2.cu). Measured in-graph (tools/len_probe.py): tc3 (the shortest
// latency chain) up to 64 tokens (-2 us), tc1 to 128, tc2 from 129; above 384 (4 query tiles per
// head) tc3's one wave at three CTAs per SM beats tc2's two waves (-6..-10 us per request).
// SP_ATTN_TC=0..3 forces one kernel (the forced-kernel parity tests).
// Attention inputs as (hi, lo) pairs. SP_ATTN_LO: 0 = hi only (A/B switch), 1 = V and P of the
// tensor-core attention (Q / K / V of the CLS attention), 2 = Q and K of the tensor-core attention too
constexpr int kAttnLoDefault = 2;
int attn_lo_level() {
  static const int level = [] {
    const char* v = getenv("SP_ATTN_LO");
    return v == nullptr ? kAttnLoDefault : atoi(v);
  }();
  return level;
}
bool attn_lo_enabled() { return attn_lo_level() > 0; }
bool attn_qk_lo() { return attn_lo_level() >= 2; }

// lo: Q/K/V carry (hi, lo) pairs — only the three-CTA kernel takes them (unless a kernel is forced)
int attn_kind(int head_dim, int max_len, bool lo = false) {
  static const int mode = [] {
    const char* v = getenv("SP_ATTN_TC");
    return v == nullptr ? -1 : atoi(v);
  }();
  if (max_len > 512 || (head_dim != 64 && head_dim != 32)) return 0;
  if (head_dim == 32) return mode == 0 ? 0 : 3;  // the three-CTA tcgen05 kernel has a head_dim-32 variant
  if (lo && mode < 0) return 3;
  if (mode >= 0) return mode;
  if (max_len <= 64) return 3;
  return max_len <= 128 ? 1 : (max_len <= 384 ? 2 : 3);
}

void launch_attention_any(int kind, const CUtensorMap& map_qkv, const CUtensorMap& map_kv64, const half* qkv,
                          half* ctx, long long lo_off, const int* cu, int n_seqs, int max_len, int groups, int n_heads,
                          int head_dim, int hidden, long long group_rows, cudaStream_t st, long long lo_rows = 0,
                          bool qk_lo = false) {
  if (kind == 3)
    sp::launch_attention_tc3(map_qkv, map_kv64, ctx, lo_off, cu, n_seqs, max_len, groups, n_heads, hidden, group_rows,
                             st, lo_rows, qk_lo);
  else if (kind == 2)
    sp::launch_attention_tc2(map_qkv, ctx, lo_off, cu, n_seqs, max_len, groups, n_heads, hidden, group_rows, st);
  else if (kind == 1)
    sp::launch_attention_tc(map_qkv, ctx, lo_off, cu, n_seqs, max_len, groups, n_heads, hidden, group_rows, st);
  else
    sp::launch_attention(qkv, ctx, lo_off, cu, n_seqs, max_len, groups, n_heads, head_dim, hidden, group_rows, st);
}

// One grouped projection (one kernel launch). Output fp16 with out_lo_off != 0: (hi, lo) pair.
void run_gemm(sp_group* grp, int kind, const CUtensorMap& wmap, const XMaps& xm, int groups, int n_out, int k_dim,
              int t_rows, int x_group_rows, const float* bias, int bias_gs, int act, void* out, long long out_gs,
              long long out_lo_off, int out_f32, int splits, long long split_stride, cudaStream_t st,
              const int* t_dev = nullptr, int out_ld = 0, int w_gs = 0, int w_r0 = 0,
              const CUtensorMap* wlo = nullptr, int lo_from = 0) {
  sp::GemmParams p{};
  p.t_dev = t_dev;
  p.n_out = n_out;
  p.w_gs = w_gs ? w_gs : n_out;
  p.w_r0 = w_r0;
  p.k_dim = k_dim;
  p.t_rows = t_rows;
  p.x_group_rows = x_group_rows;
  p.m_tiles = n_out / 128;
  p.hilo = xm.hilo ? 1 : 0;
  p.out = out;
  p.out_group_stride = out_gs;
  p.out_lo_off = out_f32 ? 0 : out_lo_off;
  p.lo_from = lo_from;
  p.out_ld = out_ld ? out_ld : n_out;
  p.bias = bias;
  p.bias_group_stride = bias_gs;
  p.act = act;
  p.out_f32 = out_f32;
  sp::GemmMapsW maps;
  maps.w = wmap;
  p.whilo = wlo ? 1 : 0;
  if (wlo) maps.wl = *wlo;
  maps.x64 = xm.x64;
  maps.x16 = xm.x16;
  maps.xl64 = xm.xl64;
  maps.xl16 = xm.xl16;
  // profiling: algorithmic bytes of a projection = its weights + bias (the activations
  // are L2-resident at batch-1 and not part of the request's compulsory HBM traffic)
  const double G = groups, N = n_out, K = k_dim, T = t_rows;
  const double wbytes = G * N * K * 2.0 * (wlo ? 2 : 1) + (bias ? G * N * 4.0 : 0.0);
  // one-split projections from 33 tokens on: the persistent kernel (2.8-4 us faster at 48-64 tokens;
  // at 17-32 tokens the small kernel is ~2 us faster, measured on the final engine)
  if (splits == 1 && t_rows >= 33) {
    p.splits = 1;
    p.kb_per_split = k_dim / 64;
    sp::gemm_configure_persistent(t_rows, out_f32 != 0, groups * p.m_tiles, sp::sm_count(),
                                  sp::gemm_persistent_pair(t_rows, p.m_tiles, groups), &p.bn, &p.n_tiles, &p.stages);
    if (wlo)  // a second weight tile per stage: re-derive the ring depth (same smem budget)
      p.stages = sp::gemm_whilo_stages(sp::gemm_persistent_pair(t_rows, p.m_tiles, groups) ? p.bn / 2 : p.bn, true,
                                       out_f32 != 0);
    // weights re-read by many token tiles stay in L2 (evict_last); streamed up to four times
    // (batch-1, <= 512 tokens) they must not push the activations out (evict_first: -1..-2 us at
    // 384-512 tokens against evict_last from 3 tiles, measured)
    p.w_keep = p.n_tiles > 4 ? 2 : 0;
    if (grp) grp->rec_begin(kind, wbytes, 2.0 * G * N * K * T);
    sp::launch_gemm_persistent(maps, p, groups, st);
    if (grp) grp->rec_end();
    return;
  }
  p.cluster = 1;
  p.w_keep = 0;  // evict_last for re-read weights measured 1-4 us slower at 160-256 tokens
  sp::gemm_configure_tiles(t_rows, &p.bn, &p.n_tiles, &p.stages);
  if (wlo) p.stages = sp::gemm_whilo_stages(p.bn, false, out_f32 != 0);
  p.epi_warps = sp::gemm_epi_warps(p.bn, p.n_tiles);
  p.splits = splits;
  p.kb_per_split = (k_dim / 64) / splits;
  p.out_split_stride = split_stride;
  if (grp) grp->rec_begin(kind, wbytes, 2.0 * G * N * K * T);
  sp::launch_gemm(maps, p, groups, st);
  if (grp) grp->rec_end();
}

// FFN1 (+GELU) and FFN2 of layer l as one persistent kernel (sp_mlp.cu); FFN2's raw projection
// lands in g->part (one split) for the LayerNorm kernel. Returns the FFN2 split count.
int run_mlp(sp_group* g, int l, int k, int n_tokens, const int* t_dev, cudaStream_t st) {
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
  sp::gemm_configure_persistent(n_tokens, false, k * (F / 128), sp::sm_count(), false, &p.bn_a, &p.n_tiles_a, &stages,
                                32);
  sp::gemm_configure_persistent(n_tokens, true, k * (H / 128), sp::sm_count(), false, &p.bn_b, &p.n_tiles_b, &stages,
                                32);
  sp::mlp_smem_bytes(std::max(p.bn_a, p.bn_b), &p.stages);
  p.groups = k;
  p.t_rows = n_tokens;
  p.x_group_rows = T;
  p.t_dev = t_dev;
  p.out_a = g->ffn;
  p.out_a_gs = (long long)T * F;
  p.out_a_lo_off = g->ffn_lo;
  p.out_a_ld = F;
  p.bias_a = w.b_ffn1 + lS * F;
  p.bias_a_gs = F;
  p.out_b = g->part;
  p.out_b_gs = (long long)T * H;
  p.out_b_ld = H;
  p.out_b_ss = (long long)c.n_students * T * H;
  // FFN2 in one split: phase B already fills one round (144 deep units at bn = 192), and more,
  // shorter units under the static reverse-order dealing measured +5..18 us at L = 384..512
  p.splits_b = 1;
  p.done = g->mlp_done;
  sp::MlpMaps m;
  m.w_a = g->m_f1[l];
  m.xa64 = g->xm_x16.x64;
  m.xa16 = g->xm_x16.x16;
  m.xal64 = g->xm_x16.xl64;
  m.xal16 = g->xm_x16.xl16;
  m.w_b = g->m_f2[l];
  m.xb64 = g->xm_ffn.x64;
  m.xb16 = g->xm_ffn.x16;
  m.xbl64 = g->xm_ffn.xl64;
  m.xbl16 = g->xm_ffn.xl16;
  const double G = k, Tt = n_tokens;
  g->rec_begin(SP_LAUNCH_GEMM_FFN1, G * 2.0 * F * H * 2.0 + G * F * 4.0, 2.0 * 2.0 * G * F * H * Tt);
  sp::launch_mlp(m, p, st);
  g->rec_end();
  return p.splits_b;
}

// dyn = true (graph capture): n_tokens / max_len are bucket bounds used for grids and tiles; every
// kernel reads the live token count from cu_seqlens[n_seqs] on the device.
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
  g->rec_reset(st);
  if (k > 0) {
    const double GTH = (double)k * n_tokens * H;
    g->rec_begin(SP_LAUNCH_EMBED_LN, GTH * 8.0, 0.0);
    sp::launch_embed_ln(ids, cu, n_seqs, n_rows_arg, k, static_cast<const half*>(w.word_emb),
                        static_cast<const half*>(w.pos_emb), static_cast<const half*>(w.type_emb),
                        (long long)c.vocab * H, (long long)c.max_pos * H, w.emb_ln_gamma, w.emb_ln_beta, H, c.ln_eps,
                        nullptr, g->x16, xgs, g->x_lo, st);
    g->rec_end();
    ++launches;
    int bn, n_tiles, stages;
    sp::gemm_configure_tiles(n_tokens, &bn, &n_tiles, &stages);
    const long long part_ss = (long long)S * xgs;
    const int s_o = choose_splits(k * (H / 128) * n_tiles, H / 64, kMaxSplits, bn);
    const int s_f = choose_splits(k * (H / 128) * n_tiles, F / 64, kMaxSplits, bn);
    const int akind = attn_kind(H / c.n_heads, max_len, attn_lo_enabled());
    // CLS-row projections of the last layer: n_seqs rows per student
    const long long bgs = (long long)B * H, partc_ss = (long long)S * bgs;
    int bn_c, n_tiles_c;
    sp::gemm_configure_tiles(n_seqs, &bn_c, &n_tiles_c, &stages);
    const int s_oc = choose_splits(k * (H / 128) * n_tiles_c, H / 64, kMaxSplits, bn_c);
    const int s_fc = choose_splits(k * (H / 128) * n_tiles_c, F / 64, kMaxSplits, bn_c);
    const double GBH = (double)k * n_seqs * H;
    // last layer: K/V of every token + the CLS query as a second GEMM only for the largest requests
    // (L12 at 512 tokens: -4.7 us); for B8 it measured 2-4.5 us slower at every length (256-512)
    const bool split_q = c.n_layers > 1 && (long long)n_tokens * H >= 448LL * 1024;
    const long long qkv_lo = attn_lo_enabled() ? g->qkv_lo : 0;
    // one LayerNorm launch (rows of k students)
    auto layer_norm = [&](const float* part, int splits, long long pss, long long pgs, const float* b_, const float* g_,
                          const float* be_, const float* x_in, long long in_gs, const int* in_rows, float* x_out,
                          long long out_gs, half* x16, long long x16_gs, long long lo, int n_rows, double rows,
                          half* cls_copy = nullptr) {
      sp::RowLn a{};
      a.cls16 = cls_copy;  // CLS rows also to cls_copy (the last layer's query operand)
      a.cls_gs = bgs;
      a.cls_lo_off = g->cls_lo;
      a.part = part;
      a.splits = splits;
      a.part_ss = pss;
      a.part_gs = pgs;
      a.bias = b_;
      a.gamma = g_;
      a.beta = be_;
      a.x_in = x_in;
      if (x_in == nullptr) {  // residual = the (hi, lo) stream itself (no separate fp32 copy)
        a.x_in16 = g->x16;
        a.x_in16_lo = g->x_lo;
      }
      a.in_gs = in_gs;
      a.in_rows = in_rows;
      a.x_out = x_out;
      a.out_gs = out_gs;
      a.x16 = x16;
      a.x16_gs = x16_gs;
      a.x_lo_off = lo;
      a.hidden = H;
      a.eps = c.ln_eps;
      a.n_rows = n_rows;
      a.cu = cu;
      a.n_seqs = n_seqs;
      // bytes: partials + residual (4 B: fp32 or the fp16 pair) + (hi, lo) out (+ fp32 out)
      g->rec_begin(SP_LAUNCH_REDUCE_LN, rows * H * (4.0 * splits + 8.0 + (x_out ? 4.0 : 0.0)), 0.0);
      sp::launch_reduce_ln(a, k, st);
      g->rec_end();
      ++launches;
    };
    for (int l = 0; l < c.n_layers; ++l) {
      const size_t lS = (size_t)l * S;
      const bool last = (l == c.n_layers - 1);
      if (split_q && last) {
        // long requests, last layer: K and V of every token (weight rows [H, 3H) of each student's
        // QKV slab), the query of the CLS rows only (rows [0, H) on the CLS copies the previous
        // LayerNorm wrote)
        run_gemm(g, SP_LAUNCH_GEMM_QKV, g->m_qkv[l], g->xm_x16, k, 2 * H, H, n_tokens, T, w.b_qkv + lS * 3 * H + H,
                 3 * H, sp::ACT_NONE, g->qkv + H, (long long)T * 3 * H, qkv_lo, 0, 1, 0, st, t_dev, 3 * H, 3 * H, H);
        run_gemm(g, SP_LAUNCH_GEMM_QKV, g->m_qkv[l], g->xm_cls, k, H, H, n_seqs, B, w.b_qkv + lS * 3 * H, 3 * H,
                 sp::ACT_NONE, g->qc, bgs, qkv_lo ? (long long)S * B * H : 0, 0, 1, 0, st, nullptr, H, 3 * H, 0);
        launches += 2;
      } else {
        // lo terms where they matter (tools/diag_prefix.py, worst prefix cases: V 0.7-3.0e-3 of
        // max|z|, Q and K together <= 4.8e-4): V for the tensor-core attention of the inner layers,
        // Q, K and V for the last layer's fp32 CLS attention (without q / K lo the worst case went
        // from 6.7e-4 to 8.1e-4 at no measurable saving)
        run_gemm(g, SP_LAUNCH_GEMM_QKV, g->m_qkv[l], g->xm_x16, k, 3 * H, H, n_tokens, T, w.b_qkv + lS * 3 * H,
                 3 * H, sp::ACT_NONE, g->qkv, (long long)T * 3 * H, qkv_lo, 0, 1, 0, st, t_dev, 0, 0, 0, nullptr,
                 last || attn_qk_lo() ? 0 : 2 * H);
        ++launches;
      }
      if (last) {
        // Only the CLS row of the last layer reaches the pooler: attention of the CLS query over
        // the sequence's keys, then O, LayerNorm-1, FFN and LayerNorm-2 on the CLS rows alone
        // (n_seqs rows per student; the residual input is gathered at cu_seqlens[b]).
        g->rec_begin(SP_LAUNCH_ATTENTION, GTH * 4.0, 4.0 * k * H * (double)n_tokens);
        sp::launch_attention_cls(g->qkv, (long long)T * 3 * H, split_q ? g->qc : nullptr, bgs, cu, n_seqs, k,
                                 c.n_heads, H / c.n_heads, H, g->ctxc, bgs, g->cls_lo, max_len, st, qkv_lo,
                                 split_q ? (qkv_lo ? (long long)S * B * H : 0) : qkv_lo);
        g->rec_end();
        run_gemm(g, SP_LAUNCH_GEMM_O, g->m_o[l], g->xm_ctxc, k, H, H, n_seqs, B, nullptr, H, sp::ACT_NONE, g->partc,
                 bgs, 0, 1, s_oc, partc_ss, st);
        ++launches;
        layer_norm(g->partc, s_oc, partc_ss, bgs, w.b_o + lS * H, w.ln1_gamma + lS * H, w.ln1_beta + lS * H, nullptr,
                   xgs, cu, g->xc32, bgs, g->cln, bgs, g->cls_lo, n_seqs, GBH);
        run_gemm(g, SP_LAUNCH_GEMM_FFN1, g->m_f1[l], g->xm_cln, k, F, H, n_seqs, B, w.b_ffn1 + lS * F, F,
                 sp::ACT_GELU, g->ffnc, (long long)B * F, g->cf_lo, 0, 1, 0, st);
        run_gemm(g, SP_LAUNCH_GEMM_FFN2, g->m_f2[l], g->xm_ffnc, k, H, F, n_seqs, B, nullptr, H, sp::ACT_NONE,
                 g->partc, bgs, 0, 1, s_fc, partc_ss, st);
        launches += 2;
        layer_norm(g->partc, s_fc, partc_ss, bgs, w.b_ffn2 + lS * H, w.ln2_gamma + lS * H, w.ln2_beta + lS * H,
                   g->xc32, bgs, nullptr, g->xc32, bgs, g->cls16, bgs, g->cls_lo, n_seqs, GBH);
        break;
      }
      g->rec_begin(SP_LAUNCH_ATTENTION, GTH * 10.0, 4.0 * k * H * g->sum_len_sq);
      launch_attention_any(akind, g->m_qkv_attn, g->m_qkv_kv64, g->qkv, g->ctx, g->ctx_lo, cu, n_seqs, max_len, k,
                           c.n_heads, H / c.n_heads, H, T, st, akind == 3 && qkv_lo ? (long long)S * T : 0,
                           attn_qk_lo());
      g->rec_end();
      // O and FFN2 write raw partial sums; the reduce+LN kernel owns bias, residual and LayerNorm
      run_gemm(g, SP_LAUNCH_GEMM_O, g->m_o[l], g->xm_ctx, k, H, H, n_tokens, T, nullptr, H, sp::ACT_NONE, g->part, xgs,
               0, 1, s_o, part_ss, st, t_dev);
      launches += 2;
      layer_norm(g->part, s_o, part_ss, xgs, w.b_o + lS * H, w.ln1_gamma + lS * H, w.ln1_beta + lS * H, nullptr, xgs,
                 nullptr, nullptr, xgs, g->x16, xgs, g->x_lo, n_rows_arg, GTH);
      // FFN1 + FFN2 as one persistent kernel where both would take the single-CTA persistent path
      // (only where FFN2 itself would be a one-split persistent GEMM: measured -2% at L=512, but
      // +3% at L=256 where FFN2's split-K tiles beat the fused kernel's 96-token phase-B tiles)
      // (re-measured on the final engine: it wins only for many students at <= 192 tokens — K32
      // -10 us at 192 — and loses for L12 (K=12) at 144-240 and for K32 at 240 tokens)
      const bool mlp = s_f == 1 && n_tokens >= 129 && n_tokens <= 224 && k > 16 && k <= sp::kMlpMaxStudents &&
                       !sp::gemm_persistent_pair(n_tokens, F / 128, k) &&
                       !sp::gemm_persistent_pair(n_tokens, H / 128, k);
      int s_ln2 = s_f;
      if (mlp) {
        s_ln2 = run_mlp(g, l, k, n_tokens, t_dev, st);
        launches += 1;
      } else {
        run_gemm(g, SP_LAUNCH_GEMM_FFN1, g->m_f1[l], g->xm_x16, k, F, H, n_tokens, T, w.b_ffn1 + lS * F, F,
                 sp::ACT_GELU, g->ffn, (long long)T * F, g->ffn_lo, 0, 1, 0, st, t_dev);
        run_gemm(g, SP_LAUNCH_GEMM_FFN2, g->m_f2[l], g->xm_ffn, k, H, F, n_tokens, T, nullptr, H, sp::ACT_NONE,
                 g->part, xgs, 0, 1, s_f, part_ss, st, t_dev);
        launches += 2;
      }
      layer_norm(g->part, s_ln2, part_ss, xgs, w.b_ffn2 + lS * H, w.ln2_gamma + lS * H, w.ln2_beta + lS * H, nullptr,
                 xgs, nullptr, nullptr, xgs, g->x16, xgs, g->x_lo, n_rows_arg, GTH,
                 split_q && l == c.n_layers - 2 ? g->cls16 : nullptr);
    }
    // pooler on the CLS rows: tanh(W_p h_CLS + b_p). Few rows: split-K partials (more CTAs stream the
    // pooler weights), finished by the head kernel; many rows: one pass with the tanh epilogue.
    const int s_p = n_seqs <= 128 ? choose_splits(k * (H / 128), H / 64, kMaxSplits, bn_c) : 1;
    pool_splits = s_p;
    run_gemm(g, SP_LAUNCH_GEMM_POOL, g->m_pool, g->xm_cls, k, H, H, n_seqs, B, s_p > 1 ? nullptr : w.b_pool, H,
             sp::ACT_TANH, g->final32, (long long)g->rows_cap * H, 0, 1, s_p, (long long)S * g->rows_cap * H, st);
    ++launches;
  }
  g->rec_begin(SP_LAUNCH_HEAD, (double)k * n_seqs * H * 4.0 * (pool_splits > 1 ? pool_splits : 1) +
                                   (double)c.n_classes * H * 4.0 + n_seqs * H * 4.0, 0.0);
  sp::launch_head(g->final32, (long long)g->rows_cap * H, (long long)S * g->rows_cap * H,
                  pool_splits > 1 ? pool_splits : 0, w.b_pool, k, w.alpha, w.w_cls, w.b_cls, c.n_classes, H, n_seqs,
                  add_bias, rep, logits, st, g->eval_finals, g->head_flag, g->head_seq);
  g->rec_end();
  ++launches;
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

// 16-token bucket of a batch-1 request, capped at the longest sequence the group accepts.
int bucket_of(const sp_group* g, int n_tokens) { return std::min(((n_tokens + 15) / 16) * 16, g->tok_cap()); }

// Batch-1 graphs: one instantiated graph per (16-token bucket, k, add_bias) replays the whole
// forward (PDL-chained kernels) with a single launch; kernels read the live length from d_cu.
//   host = true: the request's H2D copy of the pinned [cu | ids] staging is the graph's first node
//                and the head kernel publishes logits + sequence flag to mapped host memory;
//   host = false: the forward reads the group's device staging and writes d_logits.
int get_graph(sp_group* g, int n_tokens, int k, int add_bias, bool host, cudaGraphExec_t* out) {
  const int bucket = bucket_of(g, n_tokens);
  const auto key = std::make_tuple(bucket, k, add_bias);
  auto& cache = host ? g->graphs : g->dgraphs;
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return SP_OK;
  }
  if (g->cap_stream == nullptr) SP_CUDA(cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking));
  SP_CUDA(cudaStreamBeginCapture(g->cap_stream, cudaStreamCaptureModeThreadLocal));
  if (host) {
    cudaMemcpyAsync(g->d_cu, g->h_stage, sizeof(int32_t) * ((size_t)g->cu_pad + bucket), cudaMemcpyHostToDevice,
                    g->cap_stream);
    g->head_flag = g->d_flag;               // the head kernel publishes the request's sequence number
    g->head_seq = g->d_cu + g->cu_pad - 1;  // (staged in the last cu slot) after the mapped logits
  }
  int rc = bert_forward(g, g->d_ids, g->d_cu, 1, bucket, bucket, k, nullptr, host ? g->d_out : g->d_logits, add_bias,
                        g->cap_stream, true);
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
  // upload now so that the bucket's first request does not pay for it
  e = cudaGraphUpload(exec, g->cap_stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->cap_stream);
  if (e != cudaSuccess) return fail(SP_ECUDA, "graph upload: %s", cudaGetErrorString(e));
  g->graph_launches = g->last_launches;
  cache[key] = exec;
  *out = exec;
  return SP_OK;
}

void dense_forward(sp_group* g, const XMaps& xin_maps, int n_rows, int k, float* rep, float* logits, int add_bias,
                   cudaStream_t st) {
  const sp_config& c = g->cfg;
  const sp_weights& w = g->w;
  const int S = c.n_students, H = c.hidden, T = c.max_tokens;
  const long long hgs = (long long)T * H;
  const long long fgs = (long long)g->rows_cap * H;
  int launches = 0;
  g->rec_reset(st);
  if (k > 0) {
    // input_proj: every student reads the same rows (x_group_rows = 0); hidden states ping-pong
    // between ha and hb as (hi, lo) pairs; the last layer writes the fp32 final representation
    half* bufs[2] = {g->ha, g->hb};
    const XMaps* maps[2] = {&g->xm_ha, &g->xm_hb};
    run_gemm(g, SP_LAUNCH_GEMM_DENSE, g->m_in, xin_maps, k, H, c.d_in, n_rows, 0, w.b_in, H, sp::ACT_TANH, bufs[0],
             hgs, g->h_lo, 0, 1, 0, st, nullptr, 0, 0, 0, g->dense_whilo ? &g->m_in_lo : nullptr);
    ++launches;
    int cur = 0;
    for (int l = 0; l < c.n_layers; ++l) {
      const bool last = (l == c.n_layers - 1);
      const size_t lS = (size_t)l * S;
      void* out = last ? static_cast<void*>(g->final32) : static_cast<void*>(bufs[cur ^ 1]);
      run_gemm(g, SP_LAUNCH_GEMM_DENSE, g->m_layers[l], *maps[cur], k, H, H, n_rows, T, w.b_layers + lS * H, H,
               sp::ACT_TANH, out, last ? fgs : hgs, last ? 0 : g->h_lo, last ? 1 : 0, 1, 0, st, nullptr, 0, 0, 0,
               g->dense_whilo ? &g->m_layers_lo[l] : nullptr);
      ++launches;
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

int sp_group_forward_dense(sp_group* g, const void* x, const void* x_lo, int32_t n_rows, int32_t k_active,
                           float* rep_out, float* logits_out, int32_t add_bias, void* stream) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  const sp_config& c = g->cfg;
  if (c.kind != SP_KIND_DENSE) return fail(SP_EINVAL, "sp_group_forward_dense needs a dense-kind group");
  if (k_active < 0 || k_active > c.n_students)
    return fail(SP_EINVAL, "k=%d out of range 0..%d", k_active, c.n_students);
  if (n_rows < 1 || n_rows > c.max_tokens) return fail(SP_EINVAL, "n_rows=%d outside 1..%d", n_rows, c.max_tokens);
  if (!x || !logits_out) return fail(SP_EINVAL, "null buffer");
  cudaSetDevice(g->device);
  XMaps xm;
  if (!make_xmaps(&xm, x, x_lo, (uint64_t)n_rows, (uint64_t)c.d_in))
    return fail(SP_EINVAL, "input tensor map failed (x must be 16-byte aligned fp16 [n_rows][d_in])");
  dense_forward(g, xm, n_rows, k_active, rep_out, logits_out, add_bias, static_cast<cudaStream_t>(stream));
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

int sp_group_forward_dense_eval(sp_group* g, const void* x, const void* x_lo, int32_t n_rows, int32_t k_active,
                                float* finals_out, float* prefix_logits_out, void* stream) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  if (k_active < 1 || k_active > g->cfg.n_students)
    return fail(SP_EINVAL, "k=%d out of range 1..%d", k_active, g->cfg.n_students);
  cudaSetDevice(g->device);
  int rc = eval_begin(g, finals_out, prefix_logits_out);
  if (rc) return rc;
  rc = sp_group_forward_dense(g, x, x_lo, n_rows, k_active, nullptr, g->d_logits, 1, stream);
  eval_end(g);
  return rc;
}

int sp_group_forward_host(sp_group* g, const int32_t* ids, const int32_t* cu, int32_t n_seqs, int32_t n_tokens,
                          int32_t k_active, float* logits_out, int32_t add_bias, void* stream) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  const sp_config& c = g->cfg;
  if (c.kind != SP_KIND_BERT) return fail(SP_EINVAL, "sp_group_forward_host needs a BERT-kind group");
  if (!ids || !cu || !logits_out) return fail(SP_EINVAL, "null buffer");
  if (k_active < 0 || k_active > c.n_students)
    return fail(SP_EINVAL, "k=%d out of range 0..%d", k_active, c.n_students);
  if (n_seqs < 1 || n_seqs > c.max_seqs) return fail(SP_EINVAL, "n_seqs=%d outside 1..%d", n_seqs, c.max_seqs);
  if (cu[0] != 0) return fail(SP_EINVAL, "cu_seqlens[0] must be 0");
  int max_len = 0;
  double sum_sq = 0.0;
  for (int b = 0; b < n_seqs; ++b) {
    const int len = cu[b + 1] - cu[b];
    sum_sq += double(len) * double(len);
    if (len < 1) return fail(SP_EINVAL, "sequence %d is empty or cu_seqlens decreases", b);
    if (len > c.max_pos) return fail(SP_EINVAL, "sequence %d has %d tokens > max_pos %d", b, len, c.max_pos);
    max_len = std::max(max_len, len);
  }
  if (cu[n_seqs] != n_tokens) return fail(SP_EINVAL, "cu_seqlens[-1]=%d != n_tokens=%d", cu[n_seqs], n_tokens);
  if (n_tokens > c.max_tokens) return fail(SP_EINVAL, "n_tokens=%d > capacity %d", n_tokens, c.max_tokens);
  for (int t = 0; t < n_tokens; ++t)
    if (ids[t] < 0 || ids[t] >= c.vocab) return fail(SP_EINVAL, "token id %d at %d outside vocab", ids[t], t);
  g->sum_len_sq = sum_sq;
  cudaSetDevice(g->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool use_graph = graphs_enabled() && n_seqs == 1 && !g->profiling;
  cudaGraphExec_t exec = nullptr;
  if (use_graph) {
    int rc = get_graph(g, n_tokens, k_active, add_bias, true, &exec);
    if (rc) return rc;
  }
  // pinned staging ([cu | ids] block; the caller's buffers may be pageable). Every call returns only
  // after its forward finished, so the previous request no longer reads h_stage.
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

int sp_op_gemm(const void* w, const void* x, const void* x_lo, int32_t groups, int32_t n_out, int32_t k_dim,
               int32_t t_rows, int32_t x_group_rows, int32_t x_rows_total, const float* bias, int32_t act, void* out,
               void* out_lo, int32_t out_f32, int32_t splits, void* stream) {
  if (!w || !x || !out) return fail(SP_EINVAL, "null buffer");
  if (groups < 1 || n_out < 128 || n_out % 128 || k_dim < 64 || k_dim % 64 || t_rows < 1)
    return fail(SP_EINVAL, "bad gemm shape groups=%d n_out=%d k=%d t=%d", groups, n_out, k_dim, t_rows);
  if (splits < 1 || (k_dim / 64) % splits) return fail(SP_EINVAL, "splits=%d must divide k/64", splits);
  if (act < 0 || act > 2) return fail(SP_EINVAL, "unknown activation %d", act);
  const bool f32 = splits > 1 || out_f32;
  if (out_lo && f32) return fail(SP_EINVAL, "out_lo needs an fp16 output (out_f32 = 0, splits = 1)");
  CUtensorMap wm;
  XMaps xm;
  if (!make_map(&wm, w, (uint64_t)groups * n_out, k_dim, 128) || !make_xmaps(&xm, x, x_lo, x_rows_total, k_dim))
    return fail(SP_EINVAL, "tensor-map creation failed");
  const long long ogs = (long long)t_rows * n_out;
  const long long lo_off = out_lo ? (static_cast<half*>(out_lo) - static_cast<half*>(out)) : 0;
  run_gemm(nullptr, 0, wm, xm, groups, n_out, k_dim, t_rows, x_group_rows, bias, n_out, act, out, ogs, lo_off,
           f32 ? 1 : 0, splits, ogs * groups, static_cast<cudaStream_t>(stream));
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

int sp_op_attention(const void* qkv, void* ctx, void* ctx_lo, const int32_t* cu_seqlens, int32_t n_seqs,
                    int32_t max_seq_len, int32_t groups, int32_t n_heads, int32_t head_dim, int32_t group_rows,
                    void* stream) {
  if (!qkv || !ctx || !ctx_lo || !cu_seqlens) return fail(SP_EINVAL, "null buffer");
  if (head_dim != 32 && head_dim != 64) return fail(SP_EINVAL, "head_dim must be 32 or 64");
  if (n_seqs < 1 || groups < 1 || n_heads < 1 || max_seq_len < 1) return fail(SP_EINVAL, "bad attention shape");
  const int hidden = n_heads * head_dim;
  const int kind = attn_kind(head_dim, max_seq_len);
  CUtensorMap m{}, m64{};
  const uint32_t head_box = head_dim == 32 ? 32 : 64;
  if (kind != 0 && (!make_map(&m, qkv, (uint64_t)groups * group_rows, 3 * hidden, 128, head_box) ||
                    !make_map(&m64, qkv, (uint64_t)groups * group_rows, 3 * hidden, 64, head_box)))
    return fail(SP_EINVAL, "attention tensor map failed");
  const long long lo_off = static_cast<half*>(ctx_lo) - static_cast<half*>(ctx);
  launch_attention_any(kind, m, m64, static_cast<const half*>(qkv), static_cast<half*>(ctx), lo_off, cu_seqlens,
                       n_seqs, max_seq_len, groups, n_heads, head_dim, hidden, group_rows,
                       static_cast<cudaStream_t>(stream));
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_group_forward_graph(sp_group* g, const int32_t* ids, const int32_t* cu_seqlens, int32_t n_tokens,
                           int32_t k_active, float* logits_out, int32_t add_bias, void* stream) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  const sp_config& c = g->cfg;
  if (c.kind != SP_KIND_BERT) return fail(SP_EINVAL, "sp_group_forward_graph needs a BERT-kind group");
  if (!ids || !cu_seqlens || !logits_out) return fail(SP_EINVAL, "null buffer");
  if (k_active < 1 || k_active > c.n_students) return fail(SP_EINVAL, "k=%d out of range 1..%d", k_active, c.n_students);
  if (n_tokens < 1 || n_tokens > g->tok_cap())
    return fail(SP_EINVAL, "n_tokens=%d outside 1..%d", n_tokens, g->tok_cap());
  if (g->profiling || !graphs_enabled())
    return sp_group_forward(g, ids, cu_seqlens, 1, n_tokens, n_tokens, k_active, nullptr, logits_out, add_bias, stream);
  cudaSetDevice(g->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaGraphExec_t exec = nullptr;
  int rc = get_graph(g, n_tokens, k_active, add_bias, false, &exec);
  if (rc) return rc;
  // the graph reads the group's staging and writes the group's logits slot; one D2D copy hands the
  // logits to the caller (so graphs are not keyed by — nor re-captured for — the caller's buffer)
  SP_CUDA(cudaMemcpyAsync(g->d_cu, cu_seqlens, 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  SP_CUDA(cudaMemcpyAsync(g->d_ids, ids, sizeof(int32_t) * n_tokens, cudaMemcpyDeviceToDevice, st));
  SP_CUDA(cudaGraphLaunch(exec, st));
  SP_CUDA(cudaMemcpyAsync(logits_out, g->d_logits, sizeof(float) * c.n_classes, cudaMemcpyDeviceToDevice, st));
  g->last_launches = g->graph_launches;
  return SP_OK;
}

int sp_group_prepare_graphs(sp_group* g, int32_t max_tokens, int32_t k_active, int32_t add_bias) {
  if (g == nullptr) return fail(SP_EINVAL, "null group");
  if (g->cfg.kind != SP_KIND_BERT) return fail(SP_EINVAL, "graphs serve BERT-kind groups");
  if (k_active < 0 || k_active > g->cfg.n_students) return fail(SP_EINVAL, "k out of range");
  if (!graphs_enabled()) return SP_OK;
  cudaSetDevice(g->device);
  const int top = std::min<int>(max_tokens, g->tok_cap());
  for (int t = 16; t - 15 <= top; t += 16) {
    cudaGraphExec_t exec;
    int rc = get_graph(g, std::min(t, top), k_active, add_bias, true, &exec);
    if (rc) return rc;
  }
  return SP_OK;
}

}  // extern "C"
