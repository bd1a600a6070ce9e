/* studentpar_b200.h — C ABI of the B200 student-group inference engine.
 *
 * The reference (arXiv 2408.12526 artifact, /root/reference/pkg/src/studentpar) is pure Python; its
 * hot path sits behind a Python object API, not an FFI. Each entry point below replaces one piece of
 * that API; the Python host (paper_2408_12526_b200/group.py) binds them with ctypes exactly as a
 * reference maintainer would (INTEGRATION.md shows the binding).
 *
 *   sp_group_create        <- EnsembleState(students, multipliers, classifier)   distill.py:147-154
 *                             (students from StudentModel.build nnkernel.py:270-274 or
 *                              load_ensemble distill.py:610-612); weights are packed ONCE (snapshot)
 *   sp_group_forward       <- EnsembleState.rep(x, k) + classifier.forward(rep)  distill.py:169-178, :512
 *                             (BERT-kind students: token ids + cu_seqlens, device buffers)
 *   sp_group_forward_dense <- the same for the reference's dense StudentModel      nnkernel.py:289-301
 *   sp_group_forward_graph <- the same for one sequence on device buffers, as a CUDA-graph replay
 *   sp_group_forward_host  <- the same call with HOST buffers (ids in, logits out), the serving seam
 *                             Simulation._dispatch -> service_time                 servesim.py:486, :287-307
 *   sp_group_forward_eval  <- the forward half of accumulate_prefix_gradients (every student's
 *   (+ _dense_eval)           final representation, logits of every prefix k) distill.py:483-494
 *   sp_last_error          <- the ValueError / RuntimeError message the reference would raise
 *
 * Conventions: plain pointers and sizes only. "device" pointers are CUDA device addresses on the
 * group's device; `stream` is a cudaStream_t (NULL = legacy default stream). Every call is
 * re-entrant per stream for distinct groups (the reference forward is not: nnkernel.py:74).
 * Return value: SP_OK or an SP_E* code; sp_last_error() then describes the failure.
 *
 * Precision: weights fp16 (exact: the host rounds them once, weights.py); every activation a
 * projection reads is carried as an fp16 (hi, lo) pair and every accumulation is fp32, so the
 * logits match the float64 reference on the same rounded weights within 1e-3 of max|logit|.
 */
#ifndef STUDENTPAR_B200_H
#define STUDENTPAR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 3

enum sp_status {
  SP_OK = 0,
  SP_EINVAL = 1, /* argument error: the reference raises ValueError (distill.py:172-173, nnkernel.py:71-72) */
  SP_ECUDA = 2,  /* CUDA launch/runtime failure: RuntimeError */
  SP_ENOMEM = 3  /* device allocation failed */
};

enum sp_kind {
  SP_KIND_DENSE = 0, /* reference StudentModel: tanh(input_proj) -> n_layers x tanh(H x H) (nnkernel.py:256-301) */
  SP_KIND_BERT = 1   /* paper's BERT-style student: embeddings+LN -> n_layers post-LN encoder -> tanh pooler */
};

typedef struct sp_config {
  int32_t kind;         /* enum sp_kind */
  int32_t n_students;   /* students resident on this device (the local shard of the group) */
  int32_t hidden;       /* H, multiple of 128 (dense kind: rep_dim zero-padded to 128) */
  int32_t n_layers;     /* BERT: encoder layers; dense: H x H tanh layers after input_proj (>= 2) */
  int32_t n_heads;      /* BERT: attention heads, head_dim = hidden / n_heads in {32, 64} */
  int32_t ffn;          /* BERT: intermediate width F, multiple of 128 */
  int32_t d_in;         /* dense: input width, multiple of 64 (zero-padded) */
  int32_t vocab;        /* BERT: word-embedding rows */
  int32_t max_pos;      /* BERT: position-embedding rows = longest sequence */
  int32_t n_classes;    /* classifier outputs C */
  int32_t max_tokens;   /* capacity: packed tokens (BERT) or rows (dense) per call */
  int32_t max_seqs;     /* capacity: sequences per call (BERT) */
  float ln_eps;         /* LayerNorm epsilon (BERT) */
} sp_config;

/* Device pointers. Every per-student tensor is stacked over the local students on its leading
 * axis (S = n_students); per-layer tensors are additionally stacked over layers: [n_layers][S]...
 * Matrices are row-major (out, in) — the reference's DenseLayer.weight layout (nnkernel.py:73).
 * fp16 = IEEE half, f32 = float. */
typedef struct sp_weights {
  /* BERT kind */
  const void* word_emb;       /* fp16 [S][vocab][H] */
  const void* pos_emb;        /* fp16 [S][max_pos][H] */
  const void* type_emb;       /* fp16 [S][H]   (token type 0) */
  const float* emb_ln_gamma;  /* f32 [S][H] */
  const float* emb_ln_beta;   /* f32 [S][H] */
  const void* w_qkv;          /* fp16 [n_layers][S][3H][H]  rows: Q | K | V */
  const float* b_qkv;         /* f32  [n_layers][S][3H] */
  const void* w_o;            /* fp16 [n_layers][S][H][H] */
  const float* b_o;           /* f32  [n_layers][S][H] */
  const float* ln1_gamma;     /* f32  [n_layers][S][H] */
  const float* ln1_beta;
  const void* w_ffn1;         /* fp16 [n_layers][S][F][H] */
  const float* b_ffn1;        /* f32  [n_layers][S][F] */
  const void* w_ffn2;         /* fp16 [n_layers][S][H][F] */
  const float* b_ffn2;        /* f32  [n_layers][S][H] */
  const float* ln2_gamma;     /* f32  [n_layers][S][H] */
  const float* ln2_beta;
  const void* w_pool;         /* fp16 [S][H][H]  pooler: tanh(W h_CLS + b) */
  const float* b_pool;        /* f32  [S][H] */
  /* dense kind */
  const void* w_in;           /* fp16 [S][H][d_in]   input_proj (tanh) */
  const float* b_in;          /* f32  [S][H] */
  const void* w_layers;       /* fp16 [n_layers][S][H][H] (tanh) */
  const float* b_layers;      /* f32  [n_layers][S][H] */
  /* group head (both kinds) */
  const float* alpha;         /* f32 [S]     boosting multipliers of the local students */
  const float* w_cls;         /* f32 [C][H]  shared classifier (identity activation, distill.py:535) */
  const float* b_cls;         /* f32 [C] */
  /* dense kind, optional (ABI v3): the fp16 lo terms W - fp16(W) of weights whose source is wider
   * than fp16 (the reference trains in float64). With them every dense projection runs as
   * (W_hi + W_lo)(x_hi + x_lo) minus the lo x lo term — ~22-bit operands on the tensor cores.
   * NULL = the fp16 weights are exact. Same shapes as w_in / w_layers. */
  const void* w_in_lo;
  const void* w_layers_lo;
} sp_weights;

typedef struct sp_group sp_group;

int sp_abi_version(void);
const char* sp_last_error(void);

/* Allocate workspace on `device`, build TMA descriptors over the packed weights. The weight
 * buffers are borrowed (not copied) and must outlive the group. */
int sp_group_create(const sp_config* cfg, const sp_weights* weights, int device, sp_group** out);
int sp_group_destroy(sp_group* group);

/* BERT kind. ids: int32 [n_tokens] device; cu_seqlens: int32 [n_seqs + 1] device (cu[0] = 0,
 * strictly increasing, cu[n_seqs] = n_tokens); max_seq_len = max_b (cu[b+1] - cu[b]).
 * k_active: number of leading local students that take part (0 .. n_students; the host maps the
 * reference's global prefix k, distill.py:171-173, to the local count).
 * rep_out: f32 [n_seqs][H] or NULL — sum_{m<k} alpha_m * pooled_m (EnsembleState.rep).
 * logits_out: f32 [n_seqs][C] — W_c rep (+ b_c iff add_bias; a multi-GPU shard passes 0 and the
 * root adds the bias once after the reduce). */
int sp_group_forward(sp_group* group, const int32_t* ids, const int32_t* cu_seqlens, int32_t n_seqs,
                     int32_t n_tokens, int32_t max_seq_len, int32_t k_active, float* rep_out, float* logits_out,
                     int32_t add_bias, void* stream);

/* Dense kind: x fp16 [n_rows][d_in] device (one row per sample, shared by every student); x_lo
 * (optional, may be NULL) the fp16 residual x - x_hi of a wider input, read as a second operand term. */
int sp_group_forward_dense(sp_group* group, const void* x, const void* x_lo, int32_t n_rows, int32_t k_active,
                           float* rep_out, float* logits_out, int32_t add_bias, void* stream);

/* Training-side evaluation (offline distillation / pruning, not the serving path):
 *   finals_out        fp32 [k_active][n_seqs][hidden]     student m's final representation S_m(x)
 *                     (the `finals` list of accumulate_prefix_gradients, distill.py:483-486)
 *   prefix_logits_out fp32 [k_active][n_seqs][n_classes]  classifier(sum_{m<=j} alpha_m S_m(x)) + b_c
 *                     for every prefix j = 1..k_active (distill.py:489-492), accumulated left to right
 * Either output may be NULL (not both). Device buffers; k_active >= 1. Not re-entrant per group. */
int sp_group_forward_eval(sp_group* group, const int32_t* ids, const int32_t* cu_seqlens, int32_t n_seqs,
                          int32_t n_tokens, int32_t max_seq_len, int32_t k_active, float* finals_out,
                          float* prefix_logits_out, void* stream);
int sp_group_forward_dense_eval(sp_group* group, const void* x, const void* x_lo, int32_t n_rows, int32_t k_active,
                                float* finals_out, float* prefix_logits_out, void* stream);

/* BERT kind end to end with HOST buffers: validates ids/cu_seqlens like the reference validates its
 * inputs, copies them to the device, runs the group and returns once the logits are in
 * `logits_out`. One sequence: the bucket's CUDA graph is replayed and the logits arrive through
 * mapped pinned memory plus a sequence flag the call polls (no stream synchronize; a failed launch
 * is detected with cudaStreamQuery); several sequences: eager launches, D2H copy, stream sync. */
int sp_group_forward_host(sp_group* group, const int32_t* ids, const int32_t* cu_seqlens, int32_t n_seqs,
                          int32_t n_tokens, int32_t k_active, float* logits_out, int32_t add_bias, void* stream);

/* Batch-1 request on DEVICE buffers replayed as the bucket's CUDA graph (one sequence:
 * ids int32 [n_tokens], cu_seqlens int32 [2] = {0, n_tokens}; logits f32 [C] device). The inputs
 * are copied device-to-device into the group's staging, one graph launch runs the forward into the
 * group's logits slot and one device-to-device copy hands them to logits_out; asynchronous on
 * `stream`. The first call per (16-token bucket, k, add_bias) captures the graph. Same result as
 * sp_group_forward (graph replay is bit-identical to eager). */
int sp_group_forward_graph(sp_group* group, const int32_t* ids, const int32_t* cu_seqlens, int32_t n_tokens,
                           int32_t k_active, float* logits_out, int32_t add_bias, void* stream);

/* Capture (ahead of serving) the CUDA graphs that sp_group_forward_host replays for
 * single-sequence requests: one per 16-token bucket up to max_tokens, for this k_active/add_bias.
 * Optional — buckets are otherwise captured on first use. SP_GRAPHS=0 disables graphs. */
int sp_group_prepare_graphs(sp_group* group, int32_t max_tokens, int32_t k_active, int32_t add_bias);

/* Number of kernels the last forward call on this group launched. */
int sp_group_last_launches(const sp_group* group);

/* Per-launch profiling: when enabled, every kernel of a forward is bracketed by CUDA events on
 * the call's stream (adds a few microseconds of host work per launch; off by default). */
enum sp_launch_kind {
  SP_LAUNCH_EMBED_LN = 1,
  SP_LAUNCH_GEMM_QKV = 2,
  SP_LAUNCH_ATTENTION = 3,
  SP_LAUNCH_GEMM_O = 4,
  SP_LAUNCH_REDUCE_LN = 5,
  SP_LAUNCH_GEMM_FFN1 = 6,
  SP_LAUNCH_GEMM_FFN2 = 7,
  SP_LAUNCH_GEMM_POOL = 8,
  SP_LAUNCH_HEAD = 9,
  SP_LAUNCH_GEMM_DENSE = 10
};

typedef struct sp_launch_record {
  int32_t kind;   /* enum sp_launch_kind */
  float ms;       /* device duration (CUDA events) */
  double bytes;   /* algorithmic HBM bytes: projections = weights + bias; row kernels and
                     attention = their activation reads + writes */
  double flops;   /* algorithmic flops (projections 2 N K T; the tensor pipe runs twice that: one MMA per
                     operand term) */
} sp_launch_record;

int sp_group_set_profiling(sp_group* group, int enable);
/* Waits for the last forward's events; fills up to max_records entries; returns the number of
 * launches recorded (or a negative sp_status). */
int sp_group_profile_read(sp_group* group, sp_launch_record* out, int max_records);

/* Device-side logit reduce of a sharded group (replaces the NCCL reduce of partial logits):
 * a mailbox on the ROOT rank's GPU (sp_reduce_mailbox_bytes, zero-initialised device memory,
 * mapped into the other ranks' processes with the IPC calls below); every rank publishes its
 * partial logits f32 [n_rows][C] for request `seq` (1, 2, ...: the same on every rank, strictly
 * increasing) into its slot and raises its flag; the root's combine waits for all `world` flags of
 * `seq`, sums the slots in rank order (+ bias once, if non-NULL) into `out` (device or host-mapped
 * memory) and, if `out_flag` is set (host-mapped int), then writes seq there. Asynchronous on
 * `stream`; at most 4 requests in flight per mailbox (a publisher waits for the root to consume
 * request seq - 4). */
long long sp_reduce_mailbox_bytes(int32_t world, int32_t max_rows, int32_t n_classes);
/* Allocate (zeroed, its own cudaMalloc so IPC maps it whole) / free a mailbox on `device`. */
int sp_mailbox_create(int32_t world, int32_t max_rows, int32_t n_classes, int32_t device, void** mailbox_out);
int sp_mailbox_destroy(void* mailbox);
int sp_reduce_publish(void* mailbox, const float* partial, int32_t rank, int32_t world, int32_t n_rows,
                      int32_t max_rows, int32_t n_classes, int64_t seq, void* stream);
int sp_reduce_combine(void* mailbox, int32_t world, int32_t n_rows, int32_t max_rows, int32_t n_classes, int64_t seq,
                      const float* bias, float* out, int32_t* out_flag, void* stream);
/* CUDA IPC of a device allocation (64-byte handle), to map the root's mailbox in peer processes. */
int sp_ipc_get_handle(const void* dev_ptr, void* handle_out);
int sp_ipc_open_handle(const void* handle, void** dev_ptr_out);
int sp_ipc_close_handle(void* dev_ptr);

/* Op-level entry points (single kernels, used by the per-kernel parity tests).
 * GEMM: x / x_lo fp16 [x_rows_total][k_dim] operand terms (x_lo may be NULL); fp16 output with
 * out_lo != NULL is written as an (hi, lo) pair. Attention: ctx / ctx_lo the (hi, lo) context. */
int sp_op_gemm(const void* w, const void* x, const void* x_lo, int32_t groups, int32_t n_out, int32_t k_dim,
               int32_t t_rows, int32_t x_group_rows, int32_t x_rows_total, const float* bias, int32_t act, void* out,
               void* out_lo, int32_t out_f32, int32_t splits, void* stream);
int sp_op_attention(const void* qkv, void* ctx, void* ctx_lo, const int32_t* cu_seqlens, int32_t n_seqs,
                    int32_t max_seq_len, int32_t groups, int32_t n_heads, int32_t head_dim, int32_t group_rows,
                    void* stream);

/* Debug: when non-NULL, every subsequent GEMM launch writes 8 %globaltimer stamps per CTA
 * (entry, prologue done, first TMA, last TMA, first MMA, last commit, epilogue start, exit) into
 * this device buffer, indexed by CTA. */
int sp_debug_set_gemm_trace(void* device_buf);
/* Debug: per-CTA timeline (16 %globaltimer stamps) of the single-pass attention kernel, or NULL. */
int sp_debug_set_attn_trace(void* device_buf);
/* Debug: CTA count of every GEMM launch traced since the last sp_debug_set_gemm_trace. */
int sp_debug_gemm_trace_launches(int32_t* ctas_per_launch, int32_t max_launches);

#ifdef __cplusplus
}
#endif

#endif /* STUDENTPAR_B200_H */
