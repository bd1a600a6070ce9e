// sp_device.cuh — device helpers shared by the attention, row-op and per-request kernels:
// mma.sync / ldmatrix / cp.async wrappers and the warp-per-row LayerNorm store.
#pragma once
#include <cuda_fp16.h>
#include "sp_ptx.cuh"

namespace sp {

// PDL entry of the row / attention kernels: wait for the producer, then release the next kernel.
// (Releasing before the wait, so the next projection's CTAs prefetch earlier, measured no faster;
// DESIGN.md section 7.)
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_launch_dependents();
}
// Kernels that read request inputs / weights before the wait: release the next kernel first (so
// those loads never delay its launch), issue the independent loads, then pdl_wait().

__device__ __forceinline__ void mma_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// 2^x on the SFU (MUFU.EX2), flush-to-zero: exp2f without the denormal fix-up instructions.
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Every activation a GEMM reads is stored as an fp16 pair (hi, lo) with hi = fp16(x) and
// lo = fp16(x - hi): the GEMM issues one MMA per term into the same fp32 accumulator, so the operand
// carries ~22 significant bits instead of 11 (fp16 rounding of the LayerNorm / attention / GELU
// outputs alone moved the logits by up to 1.2e-3 relative; profiles/r1_precision_anatomy.txt).
__device__ __forceinline__ void split_half2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

// 16-byte async copy global -> shared; src_bytes = 0 zero-fills (rows past the sequence end).
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}


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
// Writes the (hi, lo) fp16 pair (lo at x16 + x_lo_off) — both the next GEMM's operand and the
// residual stream (hi + lo carries ~22 significant bits) — plus fp32 rows to x32 when set (the
// last layer's CLS rows), and the same pair for the CLS row (cls16, cls16 + cls_lo_off) when set.
// PRE: gamma / beta were staged in shared memory by the caller (before its dependency wait: weights,
// off the critical path; gb_pre[c * 32 + lane] / gb_pre[NC * 32 + c * 32 + lane]) — short launches,
// where the global round trip after the mean reduction costs ~1 us. Otherwise they are loaded after
// the mean (the row's inputs are dead by then, so they add no registers).
template <int NC, bool PRE = false>
__device__ __forceinline__ void layer_norm_store(float (&v)[NC][4], const float* gamma, const float* beta, float eps,
                                                 int hidden, float* x32, half* x16, long long x_lo_off, half* cls16,
                                                 long long cls_lo_off, const float4* gb_pre = nullptr) {
  const int lane = lane_id();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += (v[c][0] + v[c][1]) + (v[c][2] + v[c][3]);
  const float mean = warp_sum(s) / hidden;
  float4 gm[NC], bt[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    if constexpr (PRE) {
      gm[c] = gb_pre[c * 32 + lane];
      bt[c] = gb_pre[NC * 32 + c * 32 + lane];
    } else {
      gm[c] = __ldg(reinterpret_cast<const float4*>(gamma + c * 128 + lane * 4));
      bt[c] = __ldg(reinterpret_cast<const float4*>(beta + c * 128 + lane * 4));
    }
  }
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
    float4 y;
    y.x = (v[c][0] - mean) * rstd * gm[c].x + bt[c].x;
    y.y = (v[c][1] - mean) * rstd * gm[c].y + bt[c].y;
    y.z = (v[c][2] - mean) * rstd * gm[c].z + bt[c].z;
    y.w = (v[c][3] - mean) * rstd * gm[c].w + bt[c].w;
    if (x32) *reinterpret_cast<float4*>(x32 + f) = y;
    uint2 hi, lo;
    split_half2(y.x, y.y, hi.x, lo.x);
    split_half2(y.z, y.w, hi.y, lo.y);
    *reinterpret_cast<uint2*>(x16 + f) = hi;
    *reinterpret_cast<uint2*>(x16 + x_lo_off + f) = lo;
    if (cls16) {
      *reinterpret_cast<uint2*>(cls16 + f) = hi;
      *reinterpret_cast<uint2*>(cls16 + cls_lo_off + f) = lo;
    }
  }
}

__device__ __forceinline__ void h4_to_f4(const uint2 u, float (&o)[4]) {
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  o[0] = a.x;
  o[1] = a.y;
  o[2] = b.x;
  o[3] = b.y;
}

}  // namespace sp
