// sp_rowops.cu — row-wise HBM-bound kernels: embedding gather + LN, split-K reduce + residual + LN,
// and the boosting-sum + classifier head. One warp per row; statistics in fp32 via warp shuffles.
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"

namespace sp {

// Largest b with cu[b] <= t (cu is nondecreasing, cu[0] = 0).
__device__ __forceinline__ int seq_of(const int* cu, int n_seqs, int t) {
  int lo = 0, hi = n_seqs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(cu + mid) <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Each lane owns NC chunks of 4 consecutive features: feature = c*128 + lane*4 + j.
template <int NC>
__device__ __forceinline__ void layer_norm_store(float (&v)[NC][4], const float* gamma, const float* beta, float eps,
                                                 int hidden, float* x32, half* x16, half* cls16) {
  const int lane = lane_id();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += v[c][0] + v[c][1] + v[c][2] + v[c][3];
  const float mean = warp_sum(s) / hidden;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float d = v[c][j] - mean;
      q += d * d;
    }
  const float rstd = rsqrtf(warp_sum(q) / hidden + eps);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int f = c * 128 + lane * 4;
    const float4 gm = *reinterpret_cast<const float4*>(gamma + f);
    const float4 bt = *reinterpret_cast<const float4*>(beta + f);
    float4 y;
    y.x = (v[c][0] - mean) * rstd * gm.x + bt.x;
    y.y = (v[c][1] - mean) * rstd * gm.y + bt.y;
    y.z = (v[c][2] - mean) * rstd * gm.z + bt.z;
    y.w = (v[c][3] - mean) * rstd * gm.w + bt.w;
    *reinterpret_cast<float4*>(x32 + f) = y;
    __half2 h01 = __floats2half2_rn(y.x, y.y), h23 = __floats2half2_rn(y.z, y.w);
    uint2 packed = make_uint2(*reinterpret_cast<uint32_t*>(&h01), *reinterpret_cast<uint32_t*>(&h23));
    *reinterpret_cast<uint2*>(x16 + f) = packed;
    if (cls16) *reinterpret_cast<uint2*>(cls16 + f) = packed;
  }
}

__device__ __forceinline__ void load_h4(const half* p, float (&o)[4]) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  o[0] = a.x;
  o[1] = a.y;
  o[2] = b.x;
  o[3] = b.y;
}

template <int NC>
__global__ void __launch_bounds__(128)
    embed_ln_kernel(const int* __restrict__ ids, const int* __restrict__ cu, int n_seqs, int n_tokens,
                    const half* __restrict__ word, const half* __restrict__ pos, const half* __restrict__ type,
                    long long word_gs, long long pos_gs, const float* __restrict__ gamma,
                    const float* __restrict__ beta, int hidden, float eps, float* x32, half* x16, long long x_gs) {
  const int t = blockIdx.x * 4 + warp_id();
  if (t >= n_tokens) return;
  const int g = blockIdx.y;
  const int lane = lane_id();
  const int b = seq_of(cu, n_seqs, t);
  const int p = t - __ldg(cu + b);
  const int id = __ldg(ids + t);
  const half* wr = word + g * word_gs + (long long)id * hidden;
  const half* pr = pos + g * pos_gs + (long long)p * hidden;
  const half* tr = type + (long long)g * hidden;
  float v[NC][4];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int f = c * 128 + lane * 4;
    float a[4], bb[4], cc[4];
    load_h4(wr + f, a);
    load_h4(pr + f, bb);
    load_h4(tr + f, cc);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[c][j] = a[j] + bb[j] + cc[j];
  }
  const long long row = (long long)g * x_gs + (long long)t * hidden;
  layer_norm_store<NC>(v, gamma + (long long)g * hidden, beta + (long long)g * hidden, eps, hidden, x32 + row,
                       x16 + row, nullptr);
}

template <int NC>
__global__ void __launch_bounds__(128)
    reduce_ln_kernel(const float* __restrict__ part, int splits, long long part_split_stride,
                     const float* __restrict__ bias, const float* __restrict__ gamma, const float* __restrict__ beta,
                     int hidden, float eps, float* x32, half* x16, long long x_gs, int n_tokens,
                     const int* __restrict__ cu, int n_seqs, half* cls16, long long cls_gs) {
  const int t = blockIdx.x * 4 + warp_id();
  if (t >= n_tokens) return;
  const int g = blockIdx.y;
  const int lane = lane_id();
  const long long row = (long long)g * x_gs + (long long)t * hidden;
  float v[NC][4];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int f = c * 128 + lane * 4;
    const float4 r = *reinterpret_cast<const float4*>(x32 + row + f);
    const float4 bs = *reinterpret_cast<const float4*>(bias + (long long)g * hidden + f);
    v[c][0] = r.x + bs.x;
    v[c][1] = r.y + bs.y;
    v[c][2] = r.z + bs.z;
    v[c][3] = r.w + bs.w;
    for (int s = 0; s < splits; ++s) {  // fixed order: deterministic
      const float4 pv = *reinterpret_cast<const float4*>(part + s * part_split_stride + row + f);
      v[c][0] += pv.x;
      v[c][1] += pv.y;
      v[c][2] += pv.z;
      v[c][3] += pv.w;
    }
  }
  half* cls_row = nullptr;
  if (cls16 != nullptr) {
    const int b = seq_of(cu, n_seqs, t);
    if (__ldg(cu + b) == t) cls_row = cls16 + (long long)g * cls_gs + (long long)b * hidden;
  }
  layer_norm_store<NC>(v, gamma + (long long)g * hidden, beta + (long long)g * hidden, eps, hidden, x32 + row,
                       x16 + row, cls_row);
}

// One CTA per output row b. rep is accumulated over students in index order (distill.py:174-177).
__global__ void __launch_bounds__(256)
    head_kernel(const float* __restrict__ final_rep, long long final_gs, int groups, const float* __restrict__ alpha,
                const float* __restrict__ w_cls, const float* __restrict__ b_cls, int n_classes, int hidden,
                int add_bias, float* __restrict__ rep, float* __restrict__ logits) {
  extern __shared__ float srep[];
  __shared__ float red[8];
  const int b = blockIdx.x;
  for (int j = threadIdx.x; j < hidden; j += blockDim.x) {
    float r = 0.f;
    for (int m = 0; m < groups; ++m) r += alpha[m] * final_rep[m * final_gs + (long long)b * hidden + j];
    srep[j] = r;
    if (rep) rep[(long long)b * hidden + j] = r;
  }
  __syncthreads();
  for (int c = 0; c < n_classes; ++c) {
    float acc = 0.f;
    for (int j = threadIdx.x; j < hidden; j += blockDim.x) acc += w_cls[(long long)c * hidden + j] * srep[j];
    acc = warp_sum(acc);
    if (lane_id() == 0) red[warp_id()] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      float z = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) z += red[w];
      if (add_bias) z += b_cls[c];
      logits[(long long)b * n_classes + c] = z;
    }
    __syncthreads();
  }
}

bool rowops_supported_hidden(int hidden) {
  const int nc = hidden / 128;
  return hidden % 128 == 0 && (nc == 1 || nc == 2 || nc == 4 || nc == 6 || nc == 8);
}

void launch_embed_ln(const int* ids, const int* cu_seqlens, int n_seqs, int n_tokens, int groups, const half* word,
                     const half* pos, const half* type, long long word_gs, long long pos_gs, const float* gamma,
                     const float* beta, int hidden, float eps, float* x32, half* x16, long long x_gs,
                     cudaStream_t stream) {
  if (n_tokens <= 0 || groups <= 0) return;
  dim3 grid((n_tokens + 3) / 4, groups);
  switch (hidden / 128) {
    case 1: embed_ln_kernel<1><<<grid, 128, 0, stream>>>(ids, cu_seqlens, n_seqs, n_tokens, word, pos, type, word_gs, pos_gs, gamma, beta, hidden, eps, x32, x16, x_gs); break;
    case 2: embed_ln_kernel<2><<<grid, 128, 0, stream>>>(ids, cu_seqlens, n_seqs, n_tokens, word, pos, type, word_gs, pos_gs, gamma, beta, hidden, eps, x32, x16, x_gs); break;
    case 4: embed_ln_kernel<4><<<grid, 128, 0, stream>>>(ids, cu_seqlens, n_seqs, n_tokens, word, pos, type, word_gs, pos_gs, gamma, beta, hidden, eps, x32, x16, x_gs); break;
    case 6: embed_ln_kernel<6><<<grid, 128, 0, stream>>>(ids, cu_seqlens, n_seqs, n_tokens, word, pos, type, word_gs, pos_gs, gamma, beta, hidden, eps, x32, x16, x_gs); break;
    case 8: embed_ln_kernel<8><<<grid, 128, 0, stream>>>(ids, cu_seqlens, n_seqs, n_tokens, word, pos, type, word_gs, pos_gs, gamma, beta, hidden, eps, x32, x16, x_gs); break;
    default: break;
  }
}

void launch_reduce_ln(const float* part, int splits, long long part_split_stride, const float* bias,
                      const float* gamma, const float* beta, int hidden, float eps, float* x32, half* x16,
                      long long x_gs, int n_tokens, int groups, const int* cu_seqlens, int n_seqs, half* cls16,
                      long long cls_gs, cudaStream_t stream) {
  if (n_tokens <= 0 || groups <= 0) return;
  dim3 grid((n_tokens + 3) / 4, groups);
  switch (hidden / 128) {
    case 1: reduce_ln_kernel<1><<<grid, 128, 0, stream>>>(part, splits, part_split_stride, bias, gamma, beta, hidden, eps, x32, x16, x_gs, n_tokens, cu_seqlens, n_seqs, cls16, cls_gs); break;
    case 2: reduce_ln_kernel<2><<<grid, 128, 0, stream>>>(part, splits, part_split_stride, bias, gamma, beta, hidden, eps, x32, x16, x_gs, n_tokens, cu_seqlens, n_seqs, cls16, cls_gs); break;
    case 4: reduce_ln_kernel<4><<<grid, 128, 0, stream>>>(part, splits, part_split_stride, bias, gamma, beta, hidden, eps, x32, x16, x_gs, n_tokens, cu_seqlens, n_seqs, cls16, cls_gs); break;
    case 6: reduce_ln_kernel<6><<<grid, 128, 0, stream>>>(part, splits, part_split_stride, bias, gamma, beta, hidden, eps, x32, x16, x_gs, n_tokens, cu_seqlens, n_seqs, cls16, cls_gs); break;
    case 8: reduce_ln_kernel<8><<<grid, 128, 0, stream>>>(part, splits, part_split_stride, bias, gamma, beta, hidden, eps, x32, x16, x_gs, n_tokens, cu_seqlens, n_seqs, cls16, cls_gs); break;
    default: break;
  }
}

void launch_head(const float* final_rep, long long final_gs, int groups, const float* alpha, const float* w_cls,
                 const float* b_cls, int n_classes, int hidden, int n_rows, int add_bias, float* rep, float* logits,
                 cudaStream_t stream) {
  if (n_rows <= 0) return;
  head_kernel<<<n_rows, 256, hidden * sizeof(float), stream>>>(final_rep, final_gs, groups, alpha, w_cls, b_cls,
                                                               n_classes, hidden, add_bias, rep, logits);
}

}  // namespace sp
