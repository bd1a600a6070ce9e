// sp_attn_cls.cu — attention of the CLS query only, for the last encoder layer.
//
// Only the CLS row of the last layer reaches the pooler (tanh(W_p h_CLS + b_p)), so
// the last layer needs K and V of every token but the query, the context, the O projection, the
// LayerNorms and the FFN of the CLS row alone; the engine computes exactly that (the result is the
// same function: the other rows are dead). Per (student, sequence, head) one CTA of 4 warps:
//   1. scores s_j = q . k_j / sqrt(d) in fp32, one thread per key (16-byte loads of the key row),
//      kept in shared memory;
//   2. softmax in fp32 (block max / sum);
//   3. context c = sum_j p_j v_j: each warp a quarter of the keys, each lane 2 (d = 64) or 1 (d = 32)
//      of the dims (one coalesced 128 / 64-byte row per key), four independent keys in flight; the
//      warps' partial sums combined through shared memory, written as an (hi, lo) fp16 pair.
// Unlike the tensor-core kernels, P stays fp32 (no fp16 rounding of the probabilities).
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"
#include "sp_device.cuh"

namespace sp {

namespace {
constexpr int kClsThreads = 128;
}

// Keys and values of the (student, sequence, head) staged in shared memory with one burst of
// 16-byte cp.async copies right after the dependency wait (one global round trip instead of one per
// phase); up to kClsSmemRows keys (longer sequences stream K / V from global memory).
constexpr int kClsSmemRows = 512;

// LO: K and V are (hi, lo) fp16 pairs (lo planes at qkv + qkv_lo; q too when q_lo != 0): the products
// are taken on hi + lo in fp32 (~22-bit operands, as the projections' inputs) — the attention
// inputs' fp16 rounding dominated the adaptive-prefix cases whose logits cancel (tools/diag_prefix.py).
template <int D, bool SMEM, bool LO>
__global__ void __launch_bounds__(kClsThreads)
    attn_cls_kernel(const half* __restrict__ qkv, long long qkv_gs, const half* __restrict__ qs, long long q_gs,
                    const int* __restrict__ cu, int n_heads, int hidden, half* __restrict__ ctx, long long ctx_gs,
                    long long lo_off, float scale, long long qkv_lo, long long q_lo) {
  // keys staged in shared memory; LO: K (hi, lo) first, then V (hi, lo) into the same region once
  // the scores are done (two planes of kClsSmemRows either way)
  constexpr int kRows = kClsSmemRows;
  extern __shared__ __align__(16) uint8_t cls_smem[];
  __shared__ float red[4][D];
  __shared__ float stat[8];
  __shared__ __align__(16) half qsm[2][D];
  __shared__ __align__(16) float qf[D];
  pdl_launch_dependents();
  const int gh = blockIdx.x;
  const int g = gh / n_heads, h = gh % n_heads;
  const int b = blockIdx.y;
  const int c0 = __ldg(cu + b), c1 = __ldg(cu + b + 1);  // request input: before the dependency wait
  const int L = c1 - c0;
  const int tid = threadIdx.x, warp = warp_id(), lane = lane_id();
  const long long row3 = 3LL * hidden;
  const half* base = qkv + (long long)g * qkv_gs + (long long)c0 * row3 + h * D;
  const half* qrow = qs ? qs + (long long)g * q_gs + (long long)b * hidden + h * D : base;
  constexpr int CH = D / 8;  // 16-byte chunks per row
  constexpr size_t kPlane = SMEM ? (size_t)kRows * D : 0;
  half* Ks = reinterpret_cast<half*>(cls_smem);                    // [L][D]
  half* P2 = Ks + kPlane;                                          // second plane: V, or (LO) K lo
  float* sc = reinterpret_cast<float*>(P2 + kPlane);               // [L] scores
  // LO layout: <= kRows / 2 keys: K hi | K lo | V hi | V lo in the two planes' halves; longer: V hi /
  // V lo overwrite K hi / K lo after the scores
  const int lo_half = LO && L <= kRows / 2 ? kRows / 2 : 0;
  half* Kls = LO ? (lo_half ? Ks + (size_t)lo_half * D : P2) : P2;
  half* Vs = LO ? (lo_half ? P2 : Ks) : P2;
  half* Vls = LO ? (lo_half ? P2 + (size_t)lo_half * D : P2) : P2;
  const long long qlo = q_lo;
  // LO: K and V both staged up front when they fit (four planes for <= kRows / 2 keys), else K
  // first and V into the same region once the scores are done
  const bool kv_together = !LO || L <= kRows / 2;
  pdl_wait();
  if (tid < CH) cp_async16(qsm[0] + tid * 8, qrow + tid * 8, 16);
  if (LO && qlo && tid >= 32 && tid < 32 + CH) cp_async16(qsm[1] + (tid - 32) * 8, qrow + qlo + (tid - 32) * 8, 16);
  if constexpr (SMEM) {
    for (int i = tid; i < L * CH; i += kClsThreads) {
      const int r = i / CH, c = i - r * CH;
      const half* kr = base + (long long)r * row3 + hidden + c * 8;
      cp_async16(Ks + r * D + c * 8, kr, 16);
      if constexpr (LO) cp_async16(Kls + r * D + c * 8, kr + qkv_lo, 16);
      if (kv_together) cp_async16(Vs + r * D + c * 8, kr + hidden, 16);
      if (LO && kv_together) cp_async16(Vls + r * D + c * 8, kr + hidden + qkv_lo, 16);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  // q of the CLS row (fp32, scaled) in shared memory: lanes read it at their key's chunk
  if (tid < D) qf[tid] = (__half2float(qsm[0][tid]) + (LO && qlo ? __half2float(qsm[1][tid]) : 0.f)) * scale;
  __syncthreads();
  // 1. scores, one thread per key (chunks read in a rotated order: no shared-memory bank conflicts)
  float mx = -INFINITY;
  for (int j = tid; j < L; j += kClsThreads) {
    float s = 0.f;
#pragma unroll
    for (int cc = 0; cc < CH; ++cc) {
      const int c = (cc + j) & (CH - 1);
      const uint4 u = SMEM ? *reinterpret_cast<const uint4*>(Ks + j * D + c * 8)
                           : *reinterpret_cast<const uint4*>(base + (long long)j * row3 + hidden + c * 8);
      const __half2* hp = reinterpret_cast<const __half2*>(&u);
      const float4 qa = *reinterpret_cast<const float4*>(qf + c * 8);
      const float4 qb = *reinterpret_cast<const float4*>(qf + c * 8 + 4);
      float2 f0 = __half22float2(hp[0]), f1 = __half22float2(hp[1]);
      float2 f2 = __half22float2(hp[2]), f3 = __half22float2(hp[3]);
      if constexpr (LO) {  // k = hi + lo
        const uint4 ul = SMEM ? *reinterpret_cast<const uint4*>(Kls + j * D + c * 8)
                              : *reinterpret_cast<const uint4*>(base + (long long)j * row3 + hidden + qkv_lo + c * 8);
        const __half2* lp = reinterpret_cast<const __half2*>(&ul);
        const float2 g0 = __half22float2(lp[0]), g1 = __half22float2(lp[1]);
        const float2 g2 = __half22float2(lp[2]), g3 = __half22float2(lp[3]);
        f0.x += g0.x; f0.y += g0.y; f1.x += g1.x; f1.y += g1.y;
        f2.x += g2.x; f2.y += g2.y; f3.x += g3.x; f3.y += g3.y;
      }
      s = fmaf(qa.x, f0.x, s);
      s = fmaf(qa.y, f0.y, s);
      s = fmaf(qa.z, f1.x, s);
      s = fmaf(qa.w, f1.y, s);
      s = fmaf(qb.x, f2.x, s);
      s = fmaf(qb.y, f2.y, s);
      s = fmaf(qb.z, f3.x, s);
      s = fmaf(qb.w, f3.y, s);
    }
    sc[j] = s;
    mx = fmaxf(mx, s);
  }
  // 2. softmax statistics
  mx = warp_max(mx);
  if (lane == 0) stat[warp] = mx;
  __syncthreads();  // (also: every thread is done reading K)
  if (LO && SMEM && !kv_together) {  // V (hi, lo) into the K region while the softmax runs
    for (int i = tid; i < L * CH; i += kClsThreads) {
      const int r = i / CH, c = i - r * CH;
      const half* vr = base + (long long)r * row3 + 2 * hidden + c * 8;
      cp_async16(Vs + r * D + c * 8, vr, 16);
      cp_async16(Vls + r * D + c * 8, vr + qkv_lo, 16);
    }
    cp_async_commit();
  }
  mx = fmaxf(fmaxf(stat[0], stat[1]), fmaxf(stat[2], stat[3]));
  float sum = 0.f;
  for (int j = tid; j < L; j += kClsThreads) {
    const float p = __expf(sc[j] - mx);
    sc[j] = p;
    sum += p;
  }
  sum = warp_sum(sum);
  if (LO && SMEM && !kv_together) cp_async_wait<0>();
  __syncthreads();  // stat[] reads above are done; sc[] complete (LO: V staged)
  if (lane == 0) stat[4 + warp] = sum;
  __syncthreads();
  const float inv = 1.f / ((stat[4] + stat[5]) + (stat[6] + stat[7]));
  // 3. context: warp w takes keys w, w+4, ...; lane owns DPL consecutive dims
  constexpr int DPL = D / 32;
  float acc[4][DPL];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int d = 0; d < DPL; ++d) acc[u][d] = 0.f;
  auto vrow = [&](int jj) -> const half* {
    return SMEM ? Vs + jj * D + lane * DPL : base + (long long)jj * row3 + 2 * hidden + lane * DPL;
  };
  auto vrow_lo = [&](int jj) -> const half* {  // LO: the lo term of the same element
    return SMEM ? Vls + jj * D + lane * DPL : base + (long long)jj * row3 + 2 * hidden + qkv_lo + lane * DPL;
  };
  int j = warp;
  for (; j + 12 < L; j += 16) {  // four independent keys per iteration
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int jj = j + 4 * u;
      const float p = sc[jj];
      if constexpr (DPL == 2) {
        float2 f = __half22float2(*reinterpret_cast<const __half2*>(vrow(jj)));
        if constexpr (LO) {
          const float2 fl = __half22float2(*reinterpret_cast<const __half2*>(vrow_lo(jj)));
          f.x += fl.x;
          f.y += fl.y;
        }
        acc[u][0] = fmaf(p, f.x, acc[u][0]);
        acc[u][1] = fmaf(p, f.y, acc[u][1]);
      } else {
        acc[u][0] = fmaf(p, __half2float(*vrow(jj)) + (LO ? __half2float(*vrow_lo(jj)) : 0.f), acc[u][0]);
      }
    }
  }
  for (; j < L; j += 4) {
    const float p = sc[j];
    if constexpr (DPL == 2) {
      float2 f = __half22float2(*reinterpret_cast<const __half2*>(vrow(j)));
      if constexpr (LO) {
        const float2 fl = __half22float2(*reinterpret_cast<const __half2*>(vrow_lo(j)));
        f.x += fl.x;
        f.y += fl.y;
      }
      acc[0][0] = fmaf(p, f.x, acc[0][0]);
      acc[0][1] = fmaf(p, f.y, acc[0][1]);
    } else {
      acc[0][0] = fmaf(p, __half2float(*vrow(j)) + (LO ? __half2float(*vrow_lo(j)) : 0.f), acc[0][0]);
    }
  }
#pragma unroll
  for (int d = 0; d < DPL; ++d) red[warp][lane * DPL + d] = (acc[0][d] + acc[1][d]) + (acc[2][d] + acc[3][d]);
  __syncthreads();
  if (tid < D / 2) {
    const int d = 2 * tid;
    const float o0 = ((red[0][d] + red[1][d]) + (red[2][d] + red[3][d])) * inv;
    const float o1 = ((red[0][d + 1] + red[1][d + 1]) + (red[2][d + 1] + red[3][d + 1])) * inv;
    uint32_t hi, lo;
    split_half2(o0, o1, hi, lo);
    half* out = ctx + (long long)g * ctx_gs + (long long)b * hidden + h * D + d;
    *reinterpret_cast<uint32_t*>(out) = hi;
    *reinterpret_cast<uint32_t*>(out + lo_off) = lo;
  }
}

template <int D, bool SMEM, bool LO>
static void launch_cls_t(dim3 grid, size_t smem, cudaStream_t stream, const half* qkv, long long qkv_gs, const half* q,
                         long long q_gs, const int* cu, int n_heads, int hidden, half* ctx, long long ctx_gs,
                         long long lo_off, float scale, long long qkv_lo, long long q_lo) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_cls_kernel<D, SMEM, LO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(2 * (size_t)kClsSmemRows * 64 * 2 + 4 * 8192));
    attr = true;
  }
  launch_pdl(attn_cls_kernel<D, SMEM, LO>, grid, dim3(kClsThreads), smem, stream, qkv, qkv_gs, q, q_gs, cu, n_heads,
             hidden, ctx, ctx_gs, lo_off, scale, qkv_lo, q_lo);
}

template <int D>
static void launch_cls_d(dim3 grid, int max_len, cudaStream_t stream, const half* qkv, long long qkv_gs, const half* q,
                         long long q_gs, const int* cu, int n_heads, int hidden, half* ctx, long long ctx_gs,
                         long long lo_off, float scale, long long qkv_lo, long long q_lo) {
  const bool lo = qkv_lo != 0;
  const int rows = kClsSmemRows;
  const bool in_smem = max_len <= rows;
  const size_t smem = in_smem ? 2 * (size_t)rows * D * 2 + sizeof(float) * rows : sizeof(float) * (size_t)max_len;
  if (lo) {
    if (in_smem) launch_cls_t<D, true, true>(grid, smem, stream, qkv, qkv_gs, q, q_gs, cu, n_heads, hidden, ctx,
                                             ctx_gs, lo_off, scale, qkv_lo, q_lo);
    else launch_cls_t<D, false, true>(grid, smem, stream, qkv, qkv_gs, q, q_gs, cu, n_heads, hidden, ctx, ctx_gs,
                                      lo_off, scale, qkv_lo, q_lo);
  } else {
    if (in_smem) launch_cls_t<D, true, false>(grid, smem, stream, qkv, qkv_gs, q, q_gs, cu, n_heads, hidden, ctx,
                                              ctx_gs, lo_off, scale, 0, 0);
    else launch_cls_t<D, false, false>(grid, smem, stream, qkv, qkv_gs, q, q_gs, cu, n_heads, hidden, ctx, ctx_gs,
                                       lo_off, scale, 0, 0);
  }
}

void launch_attention_cls(const half* qkv, long long qkv_gs, const half* q, long long q_gs, const int* cu_seqlens,
                          int n_seqs, int groups, int n_heads, int head_dim, int hidden, half* ctx, long long ctx_gs,
                          long long lo_off, int max_len, cudaStream_t stream, long long qkv_lo, long long q_lo) {
  if (n_seqs <= 0 || groups <= 0) return;
  const float scale = 1.0f / sqrtf(static_cast<float>(head_dim));
  dim3 grid(groups * n_heads, n_seqs);
  if (head_dim == 64)
    launch_cls_d<64>(grid, max_len, stream, qkv, qkv_gs, q, q_gs, cu_seqlens, n_heads, hidden, ctx, ctx_gs, lo_off,
                     scale, qkv_lo, q_lo);
  else
    launch_cls_d<32>(grid, max_len, stream, qkv, qkv_gs, q, q_gs, cu_seqlens, n_heads, hidden, ctx, ctx_gs, lo_off,
                     scale, qkv_lo, q_lo);
}

}  // namespace sp
