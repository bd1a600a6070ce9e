// sp_attn.cu — unpadded variable-length multi-head attention for the student group.
//
// Sequences are packed back to back (cu_seqlens), no padding tokens and no mask beyond each
// sequence's own length: every (student, sequence, head, 64-query block) is one CTA; its four
// warps each own 16 query rows and stream 64-key blocks through shared memory with an online
// (flash-style) softmax in fp32. QK^T and PV run on mma.sync m16n8k16 (fp16 in, fp32 accumulate).
//
// There is no reference counterpart (SPEC.md:129 puts attention out of the artifact's scope); the
// semantics are standard BERT self-attention softmax(Q K^T / sqrt(d)) V, restated in
// oracle/bert.py:attention and pinned there by closed-form known-answer tests.
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"

namespace sp {

__device__ __forceinline__ void mma_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

template <int D>
__global__ void __launch_bounds__(128)
    attn_kernel(const half* __restrict__ qkv, half* __restrict__ ctx, const int* __restrict__ cu, int n_heads,
                int hidden, long long group_rows, float scale_log2) {
  constexpr int BQ = 64, BK = 64, LD = D + 8;  // +8 halfs: conflict-free fragment loads
  __shared__ __align__(16) half sQ[BQ * LD];
  __shared__ __align__(16) half sK[BK * LD];
  __shared__ __align__(16) half sV[BK * LD];

  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.y;
  const int s0 = cu[b];
  const int L = cu[b + 1] - s0;
  const int q0 = blockIdx.x * BQ;
  if (q0 >= L) return;
  const int g = blockIdx.z / n_heads;
  const int h = blockIdx.z % n_heads;
  const long long row_stride = 3LL * hidden;
  const half* base = qkv + ((long long)g * group_rows + s0) * row_stride;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int gr = lane >> 2, tq = lane & 3;
  constexpr int VPR = D / 8;  // 16-byte vectors per row

  // Q tile
  for (int i = tid; i < BQ * VPR; i += 128) {
    const int r = i / VPR, c = (i % VPR) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (q0 + r < L) v = *reinterpret_cast<const uint4*>(base + (long long)(q0 + r) * row_stride + h * D + c);
    *reinterpret_cast<uint4*>(&sQ[r * LD + c]) = v;
  }
  __syncthreads();
  uint32_t qa[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    const int r = warp * 16 + gr, c = kk * 16 + 2 * tq;
    qa[kk][0] = *reinterpret_cast<const uint32_t*>(&sQ[r * LD + c]);
    qa[kk][1] = *reinterpret_cast<const uint32_t*>(&sQ[(r + 8) * LD + c]);
    qa[kk][2] = *reinterpret_cast<const uint32_t*>(&sQ[r * LD + c + 8]);
    qa[kk][3] = *reinterpret_cast<const uint32_t*>(&sQ[(r + 8) * LD + c + 8]);
  }

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY};
  float l_run[2] = {0.f, 0.f};

  for (int k0 = 0; k0 < L; k0 += BK) {
    __syncthreads();
    for (int i = tid; i < BK * VPR; i += 128) {
      const int r = i / VPR, c = (i % VPR) * 8;
      uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
      if (k0 + r < L) {
        const half* rowp = base + (long long)(k0 + r) * row_stride + h * D + c;
        kv = *reinterpret_cast<const uint4*>(rowp + hidden);
        vv = *reinterpret_cast<const uint4*>(rowp + 2 * hidden);
      }
      *reinterpret_cast<uint4*>(&sK[r * LD + c]) = kv;
      *reinterpret_cast<uint4*>(&sV[r * LD + c]) = vv;
    }
    __syncthreads();

    float s[BK / 8][4];
#pragma unroll
    for (int nt = 0; nt < BK / 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int kr = nt * 8 + gr, c = kk * 16 + 2 * tq;
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&sK[kr * LD + c]);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(&sK[kr * LD + c + 8]);
        mma_16816(s[nt], qa[kk], b0, b1);
      }
    }
    // scale (log2 domain) + key mask, row max
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < BK / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + nt * 8 + 2 * tq + (e & 1);
        float x = s[nt][e] * scale_log2;
        if (key >= L) x = -INFINITY;
        s[nt][e] = x;
        mx[e >> 1] = fmaxf(mx[e >> 1], x);
      }
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float m_new = fmaxf(m_run[r], mx[r]);
      corr[r] = exp2f(m_run[r] - m_new);
      m_run[r] = m_new;
      l_run[r] *= corr[r];
    }
#pragma unroll
    for (int nt = 0; nt < BK / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float pv = exp2f(s[nt][e] - m_run[e >> 1]);
        s[nt][e] = pv;
        l_run[e >> 1] += pv;
      }
    }
#pragma unroll
    for (int dt = 0; dt < D / 8; ++dt) {
      o[dt][0] *= corr[0];
      o[dt][1] *= corr[0];
      o[dt][2] *= corr[1];
      o[dt][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int kc = 0; kc < BK / 16; ++kc) {
      uint32_t pa[4];
      pa[0] = pack_half2(s[2 * kc][0], s[2 * kc][1]);
      pa[1] = pack_half2(s[2 * kc][2], s[2 * kc][3]);
      pa[2] = pack_half2(s[2 * kc + 1][0], s[2 * kc + 1][1]);
      pa[3] = pack_half2(s[2 * kc + 1][2], s[2 * kc + 1][3]);
#pragma unroll
      for (int dt = 0; dt < D / 8; dt += 2) {
        const int mi = lane >> 3;  // which 8x8 matrix this lane addresses
        const int vr = kc * 16 + (mi & 1) * 8 + (lane & 7);
        const int vc = (dt + (mi >> 1)) * 8;
        uint32_t vb[4];
        ldmatrix_x4_trans(vb, &sV[vr * LD + vc]);
        mma_16816(o[dt], pa, vb[0], vb[1]);
        mma_16816(o[dt + 1], pa, vb[2], vb[3]);
      }
    }
  }

#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 1);
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 2);
  }
  const float inv0 = 1.f / l_run[0], inv1 = 1.f / l_run[1];
  const int r0 = q0 + warp * 16 + gr;
  half* out = ctx + ((long long)g * group_rows + s0) * hidden + h * D;
#pragma unroll
  for (int dt = 0; dt < D / 8; ++dt) {
    const int c = dt * 8 + 2 * tq;
    if (r0 < L)
      *reinterpret_cast<__half2*>(out + (long long)r0 * hidden + c) = __floats2half2_rn(o[dt][0] * inv0, o[dt][1] * inv0);
    if (r0 + 8 < L)
      *reinterpret_cast<__half2*>(out + (long long)(r0 + 8) * hidden + c) =
          __floats2half2_rn(o[dt][2] * inv1, o[dt][3] * inv1);
  }
}

void launch_attention(const half* qkv, half* ctx, const int* cu_seqlens, int n_seqs, int max_len, int groups,
                      int n_heads, int head_dim, int hidden, long long group_rows, cudaStream_t stream) {
  if (n_seqs <= 0 || max_len <= 0 || groups <= 0) return;
  dim3 grid((max_len + 63) / 64, n_seqs, groups * n_heads);
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(head_dim));
  if (head_dim == 64)
    launch_pdl(attn_kernel<64>, grid, dim3(128), 0, stream, qkv, ctx, cu_seqlens, n_heads, hidden, group_rows,
               scale_log2);
  else
    launch_pdl(attn_kernel<32>, grid, dim3(128), 0, stream, qkv, ctx, cu_seqlens, n_heads, hidden, group_rows,
               scale_log2);
}

}  // namespace sp
