// sp_kernels.cuh — launch wrappers for the student-group kernels (internal to the .so).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <utility>

namespace sp {

// Every kernel of the library runs with the same (maximum) shared-memory carveout, so the SM's
// L1/shared split never changes between consecutive kernels of the chain (SP_CARVEOUT=-1: driver
// default per kernel). Set once per kernel; defined in sp_runtime.cu.
void prefer_max_smem(const void* fn);

// Launch with programmatic stream serialization: the kernel may start while its predecessor in
// the stream finishes; every kernel of this library calls griddepcontrol.wait before touching
// data the predecessor produces (and only prefetches read-only weights before that).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
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
  prefer_max_smem(reinterpret_cast<const void*>(kernel));
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

enum Act : int { ACT_NONE = 0, ACT_TANH = 1, ACT_GELU = 2 };

// One student-batched ("grouped") projection, swap-AB form:
//   Y[g][t][n] = act( sum_k W[g][n][k] * X[g][t][k] + b[g][n] )     g < groups, t < t_rows, n < n_out
// W: fp16 [groups * n_out, k_dim] (row = output feature, K-major — the reference's (out,in) layout,
//    nnkernel.py:73). X: fp16 rows g * x_group_rows + t of a [rows, k_dim] tensor (x_group_rows = 0:
//    every student reads the same input). With splits > 1, raw fp32 partial sums are written to
//    out[split][g][t][n] and bias/act are applied by the consumer (split-K reduce kernel).
struct GemmParams {
  int n_out;        // multiple of 128
  int k_dim;        // multiple of 64
  int t_rows;       // valid rows per student
  int x_group_rows; // X row stride between students
  int bn;           // token tile, multiple of 16, <= 256
  int n_tiles;
  int m_tiles;
  int splits;
  int kb_per_split;
  int stages;
  void* out;
  long long out_group_stride;  // elements
  long long out_split_stride;  // elements
  int out_ld;                  // elements between rows
  const float* bias;           // [groups][n_out] or null
  int bias_group_stride;
  int act;
  int out_f32;
  unsigned long long* trace;  // debug: 8 globaltimer stamps per CTA, or null
  int cluster;                // 1, or 2: CTA pairs along M share the token tile via TMA multicast
  int w_keep;                 // keep weight tiles in L2 (evict_last) when n_tiles > 1
  int groups;                 // students in the launch (persistent path)
  int l2_prefetch;            // pull the rest of the weight slab into L2 before griddepcontrol.wait
  const int* t_dev;           // if set: live token count (device), t_rows is only the tile bound
  int direct_store;           // persistent epilogue: warp-wide stores from registers (no smem staging)
  int epi_warps;              // small-T kernel: 4 or 8 epilogue warps (gemm_epi_warps)
  int g0;                     // first student of the launch (student-split request chains)
  unsigned long long* progress;  // weight streamer pacing (sp_stream.cu): += weight bytes requested, or null
};

// Weight streamer (sp_stream.cu): L2 prefetch of a request's projection weights in consumption
// order on a side branch, paced against GemmParams.progress.
constexpr int kStreamMaxSegs = 24;
struct StreamPlan {
  const void* ptr[kStreamMaxSegs];
  unsigned long long bytes[kStreamMaxSegs];
  int n;
  unsigned long long skip;    // leading bytes the chain loads itself (first projection)
  unsigned long long window;  // max bytes prefetched ahead of the projections' progress
  unsigned long long total;   // progress the request's projections add (sum of bytes)
  unsigned long long chunk;   // bytes per bulk prefetch
  unsigned long long max_wait_ns;
};
void launch_weight_stream(const StreamPlan& plan, unsigned long long* state, int ctas, cudaStream_t stream);

// Debug hook: when set, every GEMM launch records a per-CTA timeline into this device buffer.
void set_gemm_trace(unsigned long long* buf);
int gemm_trace_counts(int* out, int max);

struct GemmMaps {
  CUtensorMap w;    // box {64, 128}
  CUtensorMap x64;  // box {64, 64}
  CUtensorMap x16;  // box {64, 16}
};

void launch_gemm(const GemmMaps& maps, const GemmParams& p, int groups, cudaStream_t stream);

// Projection + bias + residual + LayerNorm (cluster of the n_out/128 feature-tile CTAs of a row).
struct LnParams {
  const float* bias;   // [groups][hidden]
  const float* gamma;  // [groups][hidden]
  const float* beta;
  float eps;
  float* x32;          // residual in / normalised out, [groups][x_gs]
  half* x16;           // normalised out (next GEMM operand)
  long long x_gs;      // elements per student
  half* cls16;         // optional CLS rows [groups][cls_gs]
  long long cls_gs;
  const int* cu;
  int n_seqs;
  int hidden;
};
void launch_gemm_ln(const GemmMaps& maps, const GemmParams& p, const LnParams& ln, int groups, cudaStream_t stream);
size_t gemm_ln_smem_bytes(int bn, int stages);
// Persistent variant for large token counts (splits must be 1).
void launch_gemm_persistent(const GemmMaps& maps, const GemmParams& p, int groups, cudaStream_t stream);
bool gemm_persistent_pair(int t_rows, int m_tiles, int groups);
void gemm_configure_persistent(int t_rows, bool out_f32, int units_per_tile, int n_ctas, bool pair, int* bn,
                               int* n_tiles, int* stages);
int sm_count();
size_t gemm_smem_bytes(int bn, int stages);
void gemm_configure_tiles(int t_rows, bool cluster2, int* bn, int* n_tiles, int* stages);
int gemm_epi_warps(int bn, int n_tiles);

// Unpadded multi-head attention over cu_seqlens-packed sequences.
//   qkv: fp16 [groups][x_group_rows][3H] (Q | K | V, head h at columns h*D within each third)
//   ctx: fp16 [groups][x_group_rows][H]
// (pf_ptr, pf_bytes): weights of the NEXT projection, pulled into L2 while this kernel runs.
void launch_attention(const half* qkv, half* ctx, const int* cu_seqlens, int n_seqs, int max_len, int groups,
                      int n_heads, int head_dim, int hidden, long long group_rows, cudaStream_t stream,
                      const void* pf_ptr = nullptr, unsigned long long pf_bytes = 0);

// Tensor-core attention (head_dim 64, L <= 512). map_qkv: 2-D map over the qkv buffer
// [groups * group_rows, 3H] fp16 with a {64, 128} box and 128-byte swizzle.
void launch_attention_tc(const CUtensorMap& map_qkv, half* ctx, const int* cu_seqlens, int n_seqs, int max_len,
                         int groups, int n_heads, int hidden, long long group_rows, cudaStream_t stream);

// Single-pass tensor-core attention, two CTAs per SM (sp_attn_tc2.cu); same map as above.
void launch_attention_tc2(const CUtensorMap& map_qkv, half* ctx, const int* cu_seqlens, int n_seqs, int max_len,
                          int groups, int n_heads, int hidden, long long group_rows, cudaStream_t stream);

void set_attn_trace(unsigned long long* buf);
// 64-key-chunk variant, three CTAs per SM; map_kv: the qkv buffer with a {64, 64} box.
void launch_attention_tc3(const CUtensorMap& map_q, const CUtensorMap& map_kv, half* ctx, const int* cu_seqlens,
                          int n_seqs, int max_len, int groups, int n_heads, int hidden, long long group_rows,
                          cudaStream_t stream);  // debug: per-CTA timeline of attn_tc2 (16 stamps)

// Embedding gather + LayerNorm: x = LN(E_word[g][id_t] + E_pos[g][pos_t] + E_type[g][0]).
void launch_embed_ln(const int* ids, const int* cu_seqlens, int n_seqs, int n_tokens, int groups,
                     const half* word, const half* pos, const half* type, long long word_gs, long long pos_gs,
                     const float* gamma, const float* beta, int hidden, float eps, float* x32, half* x16,
                     long long x_gs, cudaStream_t stream, const void* pf_ptr = nullptr,
                     unsigned long long pf_bytes = 0);

// Split-K reduce + bias + residual + LayerNorm:
//   x = LN(x + b + sum_s part[s]); optional CLS rows copied to cls16[g][seq].
void launch_reduce_ln(const float* part, int splits, long long part_split_stride, const float* bias,
                      const float* gamma, const float* beta, int hidden, float eps, float* x32, half* x16,
                      long long x_gs, int n_tokens, int groups, const int* cu_seqlens, int n_seqs, half* cls16,
                      long long cls_gs, cudaStream_t stream, const void* pf_ptr = nullptr,
                      unsigned long long pf_bytes = 0);

// Boosting sum + shared classifier (distill.py:169-178, :512):
//   final[m][b] = splits ? tanh(sum_s part[s][m][b] + b_pool[m]) : final_rep[m][b]
//   rep[b] = sum_{m < groups} alpha[m] * final[m][b];  logits[b] = W_c rep[b] (+ b_c)
void launch_head(const float* final_rep, long long final_gs, long long split_stride, int splits,
                 const float* b_pool, int groups, const float* alpha, const float* w_cls, const float* b_cls,
                 int n_classes, int hidden, int n_rows, int add_bias, float* rep, float* logits,
                 cudaStream_t stream, float* finals = nullptr, int* ready_flag = nullptr,
                 const int* seq_src = nullptr);

// Training-side evaluation (distill.py:483-494): logits of every prefix k = 1..groups from the
// per-student finals written by launch_head. out [groups][n_rows][n_classes].
void launch_prefix_logits(const float* finals, int groups, const float* alpha, const float* w_cls,
                          const float* b_cls, int n_classes, int hidden, int n_rows, int add_bias, float* out,
                          cudaStream_t stream);


// ---------------------------------------------------------------------------------------------
// Whole-request persistent kernel (sp_request.cu): every stage of a short request (<= 128 tokens)
// in one launch, one CTA per SM. See the file header for the design.
constexpr int kReqMaxLayers = 4;
constexpr int kReqMaxTokens = 128;
constexpr int kReqMaxPhases = 4 * kReqMaxLayers + 1;
constexpr int kReqMaxTiles = 1024;   // students x feature tiles of one projection
constexpr int kReqMaxStudents = 32;
constexpr int kReqMaxSplit = 4;      // split-K chunks per tile (partials reduced by the consumer)
// dataflow counter bank (ints); two banks alternate between consecutive requests
constexpr int kReqOffDone = 64;                                               // [phase][student]
constexpr int kReqOffRows = kReqOffDone + kReqMaxPhases * kReqMaxStudents;    // [row stage][student]
constexpr int kReqOffAtt = kReqOffRows + (2 * kReqMaxLayers + 1) * kReqMaxStudents;  // [layer][student]
constexpr int kReqOffPoolTotal = kReqOffAtt + kReqMaxLayers * kReqMaxStudents;
constexpr int kReqBankInts = kReqOffPoolTotal + 64;

struct ReqMaps {
  CUtensorMap w[kReqMaxLayers][4];  // per layer: QKV, O, FFN1, FFN2 weights (box {64, 128})
  CUtensorMap w_pool;
  CUtensorMap x16_64, x16_16;  // LN outputs (QKV / FFN1 operand)
  CUtensorMap ctx_64, ctx_16;  // attention output (O operand)
  CUtensorMap ffn_64, ffn_16;  // GELU output (FFN2 operand)
  CUtensorMap cls_64, cls_16;  // CLS rows (pooler operand)
};

struct ReqParams {
  const int* ids;
  const int* cu;
  int n_seqs, k, s_total, hidden, ffn, n_heads, n_layers, t_cap, b_cap, rows_cap, n_classes, add_bias;
  int ring_bytes;
  long long part_ss, pool_ss;  // split strides of the O/FFN2 partials (pre) and pooler partials
  float eps, scale_log2;
  const half *word, *pos, *type;
  long long word_gs, pos_gs;
  const float *emb_g, *emb_b, *b_qkv, *b_o, *ln1_g, *ln1_b, *b_f1, *b_f2, *ln2_g, *ln2_b, *b_pool;
  const float *alpha, *w_cls, *b_cls;
  float* x32;
  half *x16, *qkv, *ctx, *ffn_act, *cls16;
  float *pre, *pool_part, *logits, *rep;
  int* banks;
  int* epoch;
  unsigned long long* trace;  // optional per-CTA timeline (64 stamps per CTA), else null
};

// FFN1 + FFN2 of one layer in one persistent kernel (sp_mlp.cu).
struct MlpMaps {
  CUtensorMap w_a, xa64, xa16;  // FFN1 weights [S*F, H]; LayerNorm output x16
  CUtensorMap w_b, xb64, xb16;  // FFN2 weights [S*H, F]; GELU activations
};
struct MlpParams {
  int n_a, k_a, bn_a, n_tiles_a;  // FFN1: n_out = F, k = H
  int n_b, k_b, bn_b, n_tiles_b;  // FFN2: n_out = H, k = F
  int groups, t_rows, x_group_rows, stages;
  const int* t_dev;
  half* out_a;  // GELU activations [S][x_group_rows][F]
  long long out_a_gs;
  int out_a_ld;
  const float* bias_a;
  int bias_a_gs;
  float* out_b;  // raw FFN2 projection [split][S][x_group_rows][H] (split-K partials, summed by the LayerNorm)
  long long out_b_gs;
  long long out_b_ss;  // split stride (elements)
  int splits_b;        // FFN2 split-K count (phase-B units = students x tiles x splits)
  int out_b_ld;
  int* done;  // [kReqMaxStudents + 1] FFN1 tiles finished per student + exit counter (zero between launches)
};
int mlp_smem_bytes(int bn_max, int* stages);
void launch_mlp(const MlpMaps& m, const MlpParams& p, cudaStream_t stream);

// Dynamic shared memory of the per-request kernel for head_dim d (ring + attention K/V + barriers).
int request_smem_bytes(int head_dim, int* ring_bytes);
// Returns false if (hidden, head_dim) has no instantiation.
bool launch_request(const ReqMaps& m, const ReqParams& p, int grid, cudaStream_t stream);

}  // namespace sp
