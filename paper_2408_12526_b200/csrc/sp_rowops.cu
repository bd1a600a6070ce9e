// sp_rowops.cu — row-wise HBM-bound kernels: embedding gather + LN, split-K reduce + residual + LN,
// and the boosting-sum + classifier head. One warp per row; statistics in fp32 via warp shuffles.
// Every load of a row is issued before the first use (no dependent load chains), and every kernel
// is PDL-launched: griddepcontrol.wait first, then it lets the next projection start prefetching.
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"
#include "sp_device.cuh"

namespace sp {

static constexpr int kMaxSplitsRow = 4;
// CTAs up to which the row kernels preload gamma / beta (more registers: ~3 CTAs per SM fit)
static constexpr long long kPreLnCtas = 3 * 148;

template <int NC>
__global__ void __launch_bounds__(128)
    embed_ln_kernel(const int* __restrict__ ids, const int* __restrict__ cu, int n_seqs, int n_tokens,
                    const half* __restrict__ word, const half* __restrict__ pos, const half* __restrict__ type,
                    long long word_gs, long long pos_gs, const float* __restrict__ gamma,
                    const float* __restrict__ beta, int hidden, float eps, float* x32, half* x16, long long x_gs,
                    long long x_lo_off) {
  // The first kernel of a request is launched WITHOUT programmatic serialization (launch_embed_ln),
  // so whatever the caller ran before it on the stream — a copy or its own kernel producing ids /
  // cu_seqlens — has completed; only the next projection is released early.
  pdl_launch_dependents();
  const int t = blockIdx.x * 4 + warp_id();
  if (n_tokens < 0) n_tokens = __ldg(cu + n_seqs);  // graph replay: live count = cu_seqlens[n_seqs]
  if (t >= n_tokens) return;
  const int g = blockIdx.y;
  const int lane = lane_id();
  const int id = __ldg(ids + t);
  const int b = seq_of(cu, n_seqs, t);
  const int p = t - __ldg(cu + b);
  const half* wr = word + g * word_gs + (long long)id * hidden;
  const half* pr = pos + g * pos_gs + (long long)p * hidden;
  const half* tr = type + (long long)g * hidden;
  uint2 wa[NC], pa[NC], ta[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int f = c * 128 + lane * 4;
    wa[c] = __ldg(reinterpret_cast<const uint2*>(wr + f));
    pa[c] = __ldg(reinterpret_cast<const uint2*>(pr + f));
    ta[c] = __ldg(reinterpret_cast<const uint2*>(tr + f));
  }
  float v[NC][4];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float a[4], bb[4], cc[4];
    h4_to_f4(wa[c], a);
    h4_to_f4(pa[c], bb);
    h4_to_f4(ta[c], cc);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[c][j] = a[j] + bb[j] + cc[j];
  }
  const long long row = (long long)g * x_gs + (long long)t * hidden;
  layer_norm_store<NC>(v, gamma + (long long)g * hidden, beta + (long long)g * hidden, eps, hidden,
                       x32 ? x32 + row : nullptr, x16 + row, x_lo_off, nullptr, 0);
}

// SPLITS: number of split-K partials, a template parameter so only the live ones hold registers
// (4 x NC float4 partials capped occupancy at 4 blocks/SM when the persistent path writes one).
// Row t: x_out[t] = LN(x_in[in_rows ? in_rows[t] : t] + b + sum_s part[s][t]); the (hi, lo) operand
// to x16; the CLS rows of the sequences also to cls16 (when set).
// RES16: the residual is the (hi, lo) fp16 stream (x_in16), else the fp32 rows x_in.
template <int NC, int SPLITS, bool RES16, bool PRE>
__global__ void __launch_bounds__(128) reduce_ln_kernel(const RowLn a) {
  // request inputs (cu_seqlens) and weights (bias) are read before the dependency wait
  pdl_launch_dependents();
  unsigned long long* tr = a.trace ? a.trace + 8ull * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  const int g = blockIdx.y;
  const int hidden = a.hidden;
  __shared__ float4 s_gb[PRE ? 2 * NC * 32 : 1];  // this student's gamma | beta
  if constexpr (PRE) {  // weights: staged before the dependency wait (every thread, before any exit)
    const float4* gm4 = reinterpret_cast<const float4*>(a.gamma + (long long)g * hidden);
    const float4* bt4 = reinterpret_cast<const float4*>(a.beta + (long long)g * hidden);
    for (int i = threadIdx.x; i < NC * 32; i += blockDim.x) {
      s_gb[i] = __ldg(gm4 + i);
      s_gb[NC * 32 + i] = __ldg(bt4 + i);
    }
    __syncthreads();
  }
  const int t = blockIdx.x * 4 + warp_id();
  const int n_rows = a.n_rows < 0 ? __ldg(a.cu + a.n_seqs) : a.n_rows;
  if (t >= n_rows) return;
  const int lane = lane_id();
  float4 r[NC], bs[NC], pv[SPLITS][NC];
#pragma unroll
  for (int c = 0; c < NC; ++c)
    bs[c] = __ldg(reinterpret_cast<const float4*>(a.bias + (long long)g * hidden + c * 128 + lane * 4));
  half* cls_row = nullptr;
  if (a.cls16 != nullptr) {
    const int b = seq_of(a.cu, a.n_seqs, t);
    if (__ldg(a.cu + b) == t) cls_row = a.cls16 + (long long)g * a.cls_gs + (long long)b * hidden;
  }
  const int t_in = a.in_rows ? __ldg(a.in_rows + t) : t;
  const long long in_row = (long long)g * a.in_gs + (long long)t_in * hidden;
  const float* part = a.part + (long long)g * a.part_gs + (long long)t * hidden;
  pdl_wait();
  if (tr && threadIdx.x == 0) tr[3] = globaltimer();
  // then every load of the row at once: residual and up to kMaxSplitsRow partial sums
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int f = c * 128 + lane * 4;
    if constexpr (RES16) {  // residual = the (hi, lo) stream itself (~22 significant bits)
      float h[4], l[4];
      h4_to_f4(*reinterpret_cast<const uint2*>(a.x_in16 + in_row + f), h);
      h4_to_f4(*reinterpret_cast<const uint2*>(a.x_in16 + a.x_in16_lo + in_row + f), l);
      r[c] = make_float4(h[0] + l[0], h[1] + l[1], h[2] + l[2], h[3] + l[3]);
    } else {
      r[c] = *reinterpret_cast<const float4*>(a.x_in + in_row + f);
    }
#pragma unroll
    for (int s = 0; s < SPLITS; ++s) pv[s][c] = *reinterpret_cast<const float4*>(part + s * a.part_ss + f);
  }
  float v[NC][4];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    v[c][0] = r[c].x + bs[c].x;
    v[c][1] = r[c].y + bs[c].y;
    v[c][2] = r[c].z + bs[c].z;
    v[c][3] = r[c].w + bs[c].w;
#pragma unroll
    for (int s = 0; s < SPLITS; ++s) {  // fixed order: deterministic
      v[c][0] += pv[s][c].x;
      v[c][1] += pv[s][c].y;
      v[c][2] += pv[s][c].z;
      v[c][3] += pv[s][c].w;
    }
  }
  layer_norm_store<NC, PRE>(v, a.gamma + (long long)g * hidden, a.beta + (long long)g * hidden, a.eps, hidden,
                       a.x_out ? a.x_out + (long long)g * a.out_gs + (long long)t * hidden : nullptr,
                       a.x16 + (long long)g * a.x16_gs + (long long)t * hidden, a.x_lo_off, cls_row, a.cls_lo_off,
                       s_gb);
  if (tr && threadIdx.x == 0) tr[7] = globaltimer();
}

// One CTA per output row b, one thread per feature j (blockDim = hidden <= 1024).
// Final representation of student m: either given (`splits == 0`: final_rep already activated), or
// the pooler's split-K partial sums, finished here: tanh(sum_s part[s][m][b][j] + b_pool[m][j]).
// rep[b][j] = sum_{m < groups} alpha_m * final_m[b][j] accumulated in student order
// (distill.py:174-177); logits[b][c] = sum_j W_c[c][j] rep[b][j] (+ b_c once).
// All student/split loads of a thread are issued together (8 students x up to 4 splits).
__global__ void __launch_bounds__(1024)
    head_kernel(const float* __restrict__ final_rep, long long final_gs, long long split_stride, int splits,
                const float* __restrict__ b_pool, int groups, const float* __restrict__ alpha,
                const float* __restrict__ w_cls, const float* __restrict__ b_cls, int n_classes, int hidden,
                int add_bias, float* __restrict__ rep, float* __restrict__ logits, float* __restrict__ finals,
                int* ready_flag, const int* __restrict__ seq_src) {
  // weights (the first classifier rows) are read before the dependency wait;
  // the dependents are released first so these loads never delay them
  pdl_launch_dependents();
  __shared__ float red[32][4];
  const int b = blockIdx.x;
  const int j = threadIdx.x;
  const int nsp = splits > 0 ? splits : 1;
  float wc0[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) wc0[c] = (j < hidden && c < n_classes) ? __ldg(w_cls + (long long)c * hidden + j) : 0.f;
  pdl_wait();
  float r = 0.f;
  if (j < hidden) {
    for (int m0 = 0; m0 < groups; m0 += 8) {
      float vals[8][kMaxSplitsRow], bp[8], al[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool ok = m0 + i < groups;
        const long long base = (long long)(m0 + i) * final_gs + (long long)b * hidden + j;
#pragma unroll
        for (int s = 0; s < kMaxSplitsRow; ++s) vals[i][s] = (ok && s < nsp) ? final_rep[base + s * split_stride] : 0.f;
        bp[i] = (ok && splits > 0) ? __ldg(b_pool + (long long)(m0 + i) * hidden + j) : 0.f;
        al[i] = ok ? __ldg(alpha + m0 + i) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (m0 + i < groups) {
          float v;
          if (splits > 0) {
            v = vals[i][0];
#pragma unroll
            for (int s = 1; s < kMaxSplitsRow; ++s)
              if (s < splits) v += vals[i][s];
            v = tanhf(v + bp[i]);
          } else {
            v = vals[i][0];
          }
          if (finals) finals[((long long)(m0 + i) * gridDim.x + b) * hidden + j] = v;
          r += al[i] * v;
        }
      }
    }
    if (rep) rep[(long long)b * hidden + j] = r;
  }
  const int warps = (blockDim.x + 31) >> 5;
  for (int c0 = 0; c0 < n_classes; c0 += 4) {
    float acc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      acc[c] = (j < hidden && c0 + c < n_classes)
                   ? (c0 == 0 ? wc0[c] : __ldg(w_cls + (long long)(c0 + c) * hidden + j)) * r
                   : 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = warp_sum(acc[c]);
    if (lane_id() == 0)
#pragma unroll
      for (int c = 0; c < 4; ++c) red[warp_id()][c] = acc[c];
    __syncthreads();
    if (threadIdx.x < 4 && c0 + threadIdx.x < n_classes) {
      const int c = threadIdx.x;
      float z = 0.f;
      for (int w = 0; w < warps; ++w) z += red[w][c];
      if (add_bias) z += b_cls[c0 + c];
      logits[(long long)b * n_classes + c0 + c] = z;
      if (ready_flag) __threadfence_system();  // logits (mapped host memory) before the flag
    }
    __syncthreads();
  }
  // batch-1 host path: publish the request's sequence number to the host-mapped flag it polls
  if (ready_flag != nullptr && threadIdx.x == 0) {
    __threadfence_system();
    *reinterpret_cast<volatile int*>(ready_flag) = __ldg(seq_src);
  }
}

bool rowops_supported_hidden(int hidden) {
  const int nc = hidden / 128;
  return hidden % 128 == 0 && (nc == 1 || nc == 2 || nc == 4 || nc == 6 || nc == 8);
}

template <int NC>
static void embed_ln_t(dim3 grid, cudaStream_t st, const int* ids, const int* cu, int n_seqs, int n_tokens,
                       const half* word, const half* pos, const half* type, long long word_gs, long long pos_gs,
                       const float* gamma, const float* beta, int hidden, float eps, float* x32, half* x16,
                       long long x_gs, long long x_lo_off) {
  launch_plain(embed_ln_kernel<NC>, grid, dim3(128), 0, st, ids, cu, n_seqs, n_tokens, word, pos, type, word_gs,
               pos_gs, gamma, beta, hidden, eps, x32, x16, x_gs, x_lo_off);
}

void launch_embed_ln(const int* ids, const int* cu_seqlens, int n_seqs, int n_tokens, int groups, const half* word,
                     const half* pos, const half* type, long long word_gs, long long pos_gs, const float* gamma,
                     const float* beta, int hidden, float eps, float* x32, half* x16, long long x_gs,
                     long long x_lo_off, cudaStream_t stream) {
  if (n_tokens == 0 || groups <= 0) return;
  // n_tokens < 0: grid sized for -n_tokens rows, live count read from cu_seqlens (graph replay)
  dim3 grid(((n_tokens < 0 ? -n_tokens : n_tokens) + 3) / 4, groups);
  if (n_tokens < 0) n_tokens = -1;
#define SP_EMBED(NC_)                                                                                      \
  embed_ln_t<NC_>(grid, stream, ids, cu_seqlens, n_seqs, n_tokens, word, pos, type, word_gs, pos_gs, gamma, \
                  beta, hidden, eps, x32, x16, x_gs, x_lo_off)
  switch (hidden / 128) {
    case 1: SP_EMBED(1); break;
    case 2: SP_EMBED(2); break;
    case 4: SP_EMBED(4); break;
    case 6: SP_EMBED(6); break;
    case 8: SP_EMBED(8); break;
    default: break;
  }
#undef SP_EMBED
}

void launch_reduce_ln(const RowLn& a_in, int groups, cudaStream_t stream) {
  if (a_in.n_rows == 0 || groups <= 0) return;
  // n_rows < 0: grid sized for -n_rows rows, live count read from cu_seqlens (graph replay)
  dim3 grid(((a_in.n_rows < 0 ? -a_in.n_rows : a_in.n_rows) + 3) / 4, groups);
  RowLn a = a_in;
  a.trace = trace_alloc_aux(static_cast<int>(grid.x * grid.y), 1);
  // short launches (<= one wave at the PRE kernels' register count) load gamma / beta up front
  const bool pre = (long long)grid.x * grid.y <= kPreLnCtas;
#define SP_REDUCE_S(NC_, S_)                                                                       \
  do {                                                                                             \
    if (a.x_in16) {                                                                                \
      if (pre) launch_pdl(reduce_ln_kernel<NC_, S_, true, true>, grid, dim3(128), 0, stream, a);   \
      else launch_pdl(reduce_ln_kernel<NC_, S_, true, false>, grid, dim3(128), 0, stream, a);      \
    } else {                                                                                       \
      if (pre) launch_pdl(reduce_ln_kernel<NC_, S_, false, true>, grid, dim3(128), 0, stream, a);  \
      else launch_pdl(reduce_ln_kernel<NC_, S_, false, false>, grid, dim3(128), 0, stream, a);     \
    }                                                                                              \
  } while (0)
#define SP_REDUCE(NC_)                     \
  do {                                     \
    if (a.splits <= 1) SP_REDUCE_S(NC_, 1);  \
    else if (a.splits == 2) SP_REDUCE_S(NC_, 2); \
    else if (a.splits == 3) SP_REDUCE_S(NC_, 3); \
    else SP_REDUCE_S(NC_, 4);              \
  } while (0)
  switch (a.hidden / 128) {
    case 1: SP_REDUCE(1); break;
    case 2: SP_REDUCE(2); break;
    case 4: SP_REDUCE(4); break;
    case 6: SP_REDUCE(6); break;
    case 8: SP_REDUCE(8); break;
    default: break;
  }
#undef SP_REDUCE
#undef SP_REDUCE_S
}

void launch_head(const float* final_rep, long long final_gs, long long split_stride, int splits,
                 const float* b_pool, int groups, const float* alpha, const float* w_cls, const float* b_cls,
                 int n_classes, int hidden, int n_rows, int add_bias, float* rep, float* logits,
                 cudaStream_t stream, float* finals, int* ready_flag, const int* seq_src) {
  if (n_rows <= 0) return;
  const int threads = ((hidden + 31) / 32) * 32;
  launch_pdl(head_kernel, dim3(n_rows), dim3(threads), 0, stream, final_rep, final_gs, split_stride, splits, b_pool,
             groups, alpha, w_cls, b_cls, n_classes, hidden, add_bias, rep, logits, finals, ready_flag, seq_src);
}

// Logits of every prefix k = 1..groups from the students' final representations — the forward half
// of accumulate_prefix_gradients (distill.py:483-494): rep_k = rep_{k-1} + alpha[k-1] * finals[k-1]
// accumulated left to right (:490, as EnsembleState.rep :177), z_k = W_c rep_k (+ b_c).
// One CTA per row; finals [groups][n_rows][hidden], out [groups][n_rows][n_classes].
__global__ void __launch_bounds__(1024)
    prefix_logits_kernel(const float* __restrict__ finals, int groups, const float* __restrict__ alpha,
                         const float* __restrict__ w_cls, const float* __restrict__ b_cls, int n_classes,
                         int hidden, int add_bias, float* __restrict__ out) {
  pdl_enter();
  __shared__ float red[32][4];
  const int b = blockIdx.x;
  const int j = threadIdx.x;
  const int n_rows = gridDim.x;
  const int warps = (blockDim.x + 31) >> 5;
  float r = 0.f;
  for (int m = 0; m < groups; ++m) {
    if (j < hidden) r += __ldg(alpha + m) * finals[((long long)m * n_rows + b) * hidden + j];
    for (int c0 = 0; c0 < n_classes; c0 += 4) {
      float acc[4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        acc[c] = (j < hidden && c0 + c < n_classes) ? __ldg(w_cls + (long long)(c0 + c) * hidden + j) * r : 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c] = warp_sum(acc[c]);
      if (lane_id() == 0)
#pragma unroll
        for (int c = 0; c < 4; ++c) red[warp_id()][c] = acc[c];
      __syncthreads();
      if (threadIdx.x < 4 && c0 + threadIdx.x < n_classes) {
        const int c = threadIdx.x;
        float z = 0.f;
        for (int w = 0; w < warps; ++w) z += red[w][c];
        if (add_bias) z += b_cls[c0 + c];
        out[((long long)m * n_rows + b) * n_classes + c0 + c] = z;
      }
      __syncthreads();
    }
  }
}

void launch_prefix_logits(const float* finals, int groups, const float* alpha, const float* w_cls,
                          const float* b_cls, int n_classes, int hidden, int n_rows, int add_bias, float* out,
                          cudaStream_t stream) {
  if (n_rows <= 0 || groups <= 0) return;
  const int threads = ((hidden + 31) / 32) * 32;
  launch_pdl(prefix_logits_kernel, dim3(n_rows), dim3(threads), 0, stream, finals, groups, alpha, w_cls, b_cls,
             n_classes, hidden, add_bias, out);
}

}  // namespace sp
