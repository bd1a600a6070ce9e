// sp_kernels.cuh — launch wrappers for the student-group kernels (internal to the .so).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <utility>

namespace sp {

// Record the message sp_last_error() returns and pass the status code through (sp_runtime.cu).
int report_error(int code, const char* msg);

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
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Plain launch (full stream order): the first kernel of a request, so that whatever the caller ran
// before it on the stream (a copy, or its own kernel producing the ids) is complete.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_plain(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

enum Act : int { ACT_NONE = 0, ACT_TANH = 1, ACT_GELU = 2 };

// One student-batched ("grouped") projection, swap-AB form:
//   Y[g][t][n] = act( sum_k W[g][n][k] * X[g][t][k] + b[g][n] )     g < groups, t < t_rows, n < n_out
// W: fp16 [groups * n_out, k_dim] (row = output feature, K-major — the reference's (out,in) layout,
//    nnkernel.py:73). X: rows g * x_group_rows + t of a [rows, k_dim] tensor (x_group_rows = 0:
//    every student reads the same input), as an fp16 (hi, lo) pair when hilo = 1 (two MMAs per
//    k-slice into one accumulator, sp_device.cuh split_half2). With splits > 1, raw fp32 partial
//    sums are written to out[split][g][t][n] and bias/act are applied by the consumer (split-K
//    reduce kernel). fp16 outputs with out_lo_off != 0 are written as (hi, lo) pairs, lo at
//    out + out_lo_off (the next GEMM's operand).
struct GemmParams {
  int n_out;        // multiple of 128
  int w_gs;         // weight rows per student in the map (>= n_out; the QKV slab is 3H rows)
  int w_r0;         // first weight row of the launch within a student's slab (K|V of QKV: H)
  int k_dim;        // multiple of 64
  int t_rows;       // valid rows per student
  int x_group_rows; // X row stride between students
  int bn;           // token tile, multiple of 16, <= 256
  int n_tiles;
  int m_tiles;
  int splits;
  int kb_per_split;
  int stages;
  int hilo;         // X operand is an (hi, lo) pair (maps xl64 / xl16)
  int whilo;        // W operand is an (hi, lo) pair too (map wl): weights of a float64 source (dense kind)
  void* out;
  long long out_group_stride;  // elements
  long long out_split_stride;  // elements
  long long out_lo_off;        // fp16 output: lo term at out + out_lo_off (0: hi only)
  int lo_from;                 // lo term only for output features >= lo_from (the V third of a QKV tile)
  int out_ld;                  // elements between rows
  const float* bias;           // [groups][n_out] or null
  int bias_group_stride;
  int act;
  int out_f32;
  unsigned long long* trace;  // debug: 8 globaltimer stamps per CTA, or null
  int cluster;                // persistent path: 1, or 2 = CTA pairs (cta_group::2)
  int w_keep;                 // weight L2 policy: 0 evict_first, 1 normal, 2 evict_last
  int groups;                 // students in the launch (persistent path)
  const int* t_dev;           // if set: live token count (device), t_rows is only the tile bound
  int epi_warps;              // small-T kernel: 4 or 8 epilogue warps (gemm_epi_warps)
};

// Debug hook: when set, every GEMM launch records a per-CTA timeline into this device buffer.
void set_gemm_trace(unsigned long long* buf);
int gemm_trace_counts(int* out, int max);
// debug: trace slots (8 per CTA) for a non-GEMM launch, kind 1 = LayerNorm, 2 = attention;
// recorded as -(kind * 100000 + ctas); null when tracing is off
unsigned long long* trace_alloc_aux(int ctas, int kind);

struct GemmMaps {
  CUtensorMap w;      // box {64, 128}
  CUtensorMap x64;    // box {64, 64}   hi term
  CUtensorMap x16;    // box {64, 16}
  CUtensorMap xl64;   // box {64, 64}   lo term (hilo)
  CUtensorMap xl16;   // box {64, 16}
};
// + the weights' lo term (dense kind, whilo): only the WHILO kernel instantiations take this one,
// so the BERT kernels' parameters and loops carry nothing for it
struct GemmMapsW : GemmMaps {
  CUtensorMap wl;     // box {64, 128}
};

void launch_gemm(const GemmMapsW& maps, const GemmParams& p, int groups, cudaStream_t stream);
// Persistent variant for large token counts (splits must be 1).
void launch_gemm_persistent(const GemmMapsW& maps, const GemmParams& p, int groups, cudaStream_t stream);
bool gemm_persistent_pair(int t_rows, int m_tiles, int groups);
// gran: token-tile granularity override (0: 16, or 32 for pairs; the fused MLP kernel needs 32)
void gemm_configure_persistent(int t_rows, bool out_f32, int units_per_tile, int n_ctas, bool pair, int* bn,
                               int* n_tiles, int* stages, int gran = 0);
int sm_count();
size_t gemm_smem_bytes(int bn, int stages, int whilo = 0);
// ring depth when every stage also holds the weights' lo tile (x_rows = token rows staged per CTA)
int gemm_whilo_stages(int x_rows, bool persistent, bool out_f32);
void gemm_configure_tiles(int t_rows, int* bn, int* n_tiles, int* stages);
int gemm_epi_warps(int bn, int n_tiles);

// Unpadded multi-head attention over cu_seqlens-packed sequences.
//   qkv: fp16 [groups][x_group_rows][3H] (Q | K | V, head h at columns h*D within each third)
//   ctx: fp16 [groups][x_group_rows][H] hi term, lo term at ctx + lo_off (the O projection's operand)
void launch_attention(const half* qkv, half* ctx, long long lo_off, const int* cu_seqlens, int n_seqs, int max_len,
                      int groups, int n_heads, int head_dim, int hidden, long long group_rows, cudaStream_t stream);

// Tensor-core attention (head_dim 64, L <= 512). map_qkv: 2-D map over the qkv buffer
// [groups * group_rows, 3H] fp16 with a {64, 128} box and 128-byte swizzle.
void launch_attention_tc(const CUtensorMap& map_qkv, half* ctx, long long lo_off, const int* cu_seqlens, int n_seqs,
                         int max_len, int groups, int n_heads, int hidden, long long group_rows, cudaStream_t stream);

// Single-pass tensor-core attention, two CTAs per SM (sp_attn_tc2.cu); same map as above.
void launch_attention_tc2(const CUtensorMap& map_qkv, half* ctx, long long lo_off, const int* cu_seqlens, int n_seqs,
                          int max_len, int groups, int n_heads, int hidden, long long group_rows, cudaStream_t stream);

void set_attn_trace(unsigned long long* buf);  // debug: per-CTA timeline of attn_tc2 (16 stamps)
// 64-key-chunk variant, three CTAs per SM; map_kv: the qkv buffer with a {64, 64} box.
void launch_attention_tc3(const CUtensorMap& map_q, const CUtensorMap& map_kv, half* ctx, long long lo_off,
                          const int* cu_seqlens, int n_seqs, int max_len, int groups, int n_heads, int hidden,
                          long long group_rows, cudaStream_t stream, long long lo_rows = 0, bool qk_lo = false);

// Embedding gather + LayerNorm: x = LN(E_word[g][id_t] + E_pos[g][pos_t] + E_type[g][0]); writes
// x32 and the (hi, lo) operand pair x16 / x16 + x_lo_off.
void launch_embed_ln(const int* ids, const int* cu_seqlens, int n_seqs, int n_tokens, int groups,
                     const half* word, const half* pos, const half* type, long long word_gs, long long pos_gs,
                     const float* gamma, const float* beta, int hidden, float eps, float* x32, half* x16,
                     long long x_gs, long long x_lo_off, cudaStream_t stream);

// Split-K reduce + bias + residual + LayerNorm over rows t < n_rows of `groups` students:
//   x_out[t] = LN(x_in[in_rows ? in_rows[t] : t] + b + sum_s part[s][t])  (fp32)
//   x16[t] / x16[t] + x_lo_off = the (hi, lo) fp16 operand pair of the next projection
//   cls16[seq] (+ cls_lo_off) = the same pair for the sequences' CLS rows, when cls16 is set.
// Group strides (elements) per buffer; n_rows < 0: live count = cu[n_seqs] (graph replay).
struct RowLn {
  const float* part;
  int splits;
  long long part_ss, part_gs;
  const float *bias, *gamma, *beta;  // [groups][hidden], already at the layer
  const float* x_in;   // fp32 residual, or null: the residual is the (hi, lo) pair x_in16 (+ x_in16_lo)
  const half* x_in16;
  long long x_in16_lo;
  long long in_gs;
  const int* in_rows;  // residual row of output row t (the CLS rows: cu_seqlens), or null
  float* x_out;        // fp32 output rows, or null (the (hi, lo) output is the residual stream)
  long long out_gs;
  half* x16;
  long long x16_gs, x_lo_off;
  half* cls16;
  long long cls_gs, cls_lo_off;
  int hidden;
  float eps;
  int n_rows;
  const int* cu;
  int n_seqs;
  unsigned long long* trace;  // debug: set by launch_reduce_ln when the GEMM trace is on
};
void launch_reduce_ln(const RowLn& a, int groups, cudaStream_t stream);

// Attention of the CLS query only (the last layer: only the CLS row reaches the pooler): per
// (student, sequence, head) softmax(q_CLS K^T / sqrt(d)) V over the sequence's keys, fp32. Keys and
// values from qkv [g][T][3H]; the query from q[g][seq] (row stride hidden, group stride q_gs), or,
// when q is null, from the CLS row of qkv. The context row is written as an (hi, lo) pair to
// ctx[g][seq] (row stride hidden, group stride ctx_gs).
// qkv_lo / q_lo: element offsets of the (hi, lo) lo planes of qkv / q (0: hi only).
void launch_attention_cls(const half* qkv, long long qkv_gs, const half* q, long long q_gs, const int* cu_seqlens,
                          int n_seqs, int groups, int n_heads, int head_dim, int hidden, half* ctx, long long ctx_gs,
                          long long lo_off, int max_len, cudaStream_t stream, long long qkv_lo = 0,
                          long long q_lo = 0);

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


constexpr int kMlpMaxStudents = 64;  // per-student FFN1 counters of the fused MLP kernel

// FFN1 + FFN2 of one layer in one persistent kernel (sp_mlp.cu).
struct MlpMaps {
  CUtensorMap w_a, xa64, xa16, xal64, xal16;  // FFN1 weights [S*F, H]; LayerNorm output x16 (hi, lo)
  CUtensorMap w_b, xb64, xb16, xbl64, xbl16;  // FFN2 weights [S*H, F]; GELU activations (hi, lo)
};
struct MlpParams {
  int n_a, k_a, bn_a, n_tiles_a;  // FFN1: n_out = F, k = H
  int n_b, k_b, bn_b, n_tiles_b;  // FFN2: n_out = H, k = F
  int groups, t_rows, x_group_rows, stages;
  const int* t_dev;
  half* out_a;  // GELU activations [S][x_group_rows][F], lo term at out_a + out_a_lo_off
  long long out_a_gs;
  long long out_a_lo_off;
  int out_a_ld;
  const float* bias_a;
  int bias_a_gs;
  float* out_b;  // raw FFN2 projection [split][S][x_group_rows][H] (split-K partials, summed by the LayerNorm)
  long long out_b_gs;
  long long out_b_ss;  // split stride (elements)
  int splits_b;        // FFN2 split-K count (phase-B units = students x tiles x splits)
  int out_b_ld;
  int* done;  // [kMlpMaxStudents + 1] FFN1 tiles finished per student + exit counter (zero between launches)
};
int mlp_smem_bytes(int bn_max, int* stages);
void launch_mlp(const MlpMaps& m, const MlpParams& p, cudaStream_t stream);

}  // namespace sp
