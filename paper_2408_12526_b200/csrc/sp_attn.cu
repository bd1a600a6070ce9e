// sp_attn.cu — unpadded variable-length multi-head attention for the student group.
//
// Sequences are packed back to back (cu_seqlens), no padding tokens and no mask beyond each
// sequence's own length. One CTA per (student, sequence, head, BQ-query block) with NW warps of 16
// query rows each (BQ = 16 * NW); 64-key K/V blocks stream through a double-buffered cp.async
// pipeline (next block in flight while the current one is consumed), fragments come from
// ldmatrix, QK^T and PV run on mma.sync m16n8k16 (fp16 in, fp32 accumulate), and the online
// softmax is kept in fp32 in the exp2 domain.
//
// There is no reference counterpart (SPEC.md:129 puts attention out of the artifact's scope); the
// semantics are standard BERT self-attention softmax(Q K^T / sqrt(d)) V, restated in
// oracle/bert.py:attention and pinned there by closed-form known-answer tests.
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"
#include "sp_device.cuh"

namespace sp {

// NBUF: K/V blocks in the cp.async ring (NBUF-1 in flight ahead of the one being consumed).
template <int D, int NW, int MINB, int NBUF>
__global__ void __launch_bounds__(32 * NW, MINB)
    attn_kernel(const half* __restrict__ qkv, half* __restrict__ ctx, const int* __restrict__ cu, int n_heads,
                int hidden, long long group_rows, float scale_log2, long long lo_off) {
  constexpr int BQ = 16 * NW, BK = 64, LD = D + 8;  // +8 halfs: conflict-free ldmatrix rows
  constexpr int NT = 32 * NW;
  constexpr int VPR = D / 8;  // 16-byte vectors per row
  extern __shared__ __align__(16) uint8_t attn_smem[];
  half* sQ = reinterpret_cast<half*>(attn_smem);
  half* sK = sQ + BQ * LD;         // [NBUF][BK][LD]
  half* sV = sK + NBUF * BK * LD;  // [NBUF][BK][LD]

  const int b = blockIdx.y;
  pdl_launch_dependents();
  const int c0 = __ldg(cu + b);  // request input: issued before the dependency wait
  const int c1 = __ldg(cu + b + 1);
  pdl_wait();
  const int s0 = c0;
  const int L = c1 - c0;
  const int q0 = blockIdx.x * BQ;
  if (q0 >= L) return;
  const int g = blockIdx.z / n_heads;
  const int h = blockIdx.z % n_heads;
  const long long row_stride = 3LL * hidden;
  const half* base = qkv + ((long long)g * group_rows + s0) * row_stride + h * D;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int gr = lane >> 2, tq = lane & 3;

  auto load_kv = [&](int buf, int k0) {
    half* dk = sK + buf * BK * LD;
    half* dv = sV + buf * BK * LD;
    for (int i = tid; i < BK * VPR; i += NT) {
      const int r = i / VPR, c = (i % VPR) * 8;
      const bool ok = k0 + r < L;
      const half* rowp = base + (long long)(ok ? k0 + r : 0) * row_stride + c;
      cp_async16(dk + r * LD + c, rowp + hidden, ok ? 16u : 0u);
      cp_async16(dv + r * LD + c, rowp + 2 * hidden, ok ? 16u : 0u);
    }
  };

  // Q tile + the first NBUF-1 K/V blocks (one commit group each, empty groups past the end)
  for (int i = tid; i < BQ * VPR; i += NT) {
    const int r = i / VPR, c = (i % VPR) * 8;
    const bool ok = q0 + r < L;
    cp_async16(sQ + r * LD + c, base + (long long)(ok ? q0 + r : 0) * row_stride + c, ok ? 16u : 0u);
  }
  const int n_blk = (L + BK - 1) / BK;
#pragma unroll
  for (int i = 0; i < NBUF - 1; ++i) {
    if (i < n_blk) load_kv(i, i * BK);
    cp_async_commit();
  }

  uint32_t qa[D / 16][4];
  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY};
  float l_run[2] = {0.f, 0.f};
  const int n_blocks = (L + BK - 1) / BK;

  for (int kb = 0; kb < n_blocks; ++kb) {
    const int buf = kb % NBUF;
    // refill the buffer freed by block kb-1 with block kb+NBUF-1, then wait for block kb
    if (kb + NBUF - 1 < n_blocks) load_kv((kb + NBUF - 1) % NBUF, (kb + NBUF - 1) * BK);
    cp_async_commit();
    cp_async_wait<NBUF - 1>();  // all but the NBUF-1 newest groups have landed: block kb is in
    __syncthreads();
    if (kb == 0) {
      // Q fragments (A operand, row-major 16 x 16 per k-step) via ldmatrix
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int r = warp * 16 + (lane & 15);
        const int c = kk * 16 + (lane >> 4) * 8;
        ldmatrix_x4(qa[kk], sQ + r * LD + c);
      }
    }
    const half* cK = sK + buf * BK * LD;
    const half* cV = sV + buf * BK * LD;
    const int k0 = kb * BK;

    // S = Q K^T for 64 keys: 8 n-tiles of 8 keys
    float s[BK / 8][4];
#pragma unroll
    for (int nt = 0; nt < BK / 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; kk += 2) {
        // matrices: (keys nt*8.., d kk*16+0..7), (.., +8..15), (.., (kk+1)*16+0..7), (.., +8..15)
        uint32_t kf[4];
        const int r = nt * 8 + (lane & 7);
        const int c = kk * 16 + (lane >> 3) * 8;
        ldmatrix_x4(kf, cK + r * LD + c);
        mma_16816(s[nt], qa[kk], kf[0], kf[1]);
        if (kk + 1 < D / 16) mma_16816(s[nt], qa[kk + 1], kf[2], kf[3]);
      }
    }
    // row max of the raw scores (key mask only in the block that crosses the sequence end), then
    // p = 2^(s * scale_log2 - m) as one FFMA + MUFU.EX2 per score; m kept in the scaled domain
    if (k0 + BK > L) {
#pragma unroll
      for (int nt = 0; nt < BK / 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (k0 + nt * 8 + 2 * tq + (e & 1) >= L) s[nt][e] = -INFINITY;
    }
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < BK / 8; ++nt) {
      mx[0] = fmaxf(mx[0], fmaxf(s[nt][0], s[nt][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[nt][2], s[nt][3]));
    }
    float corr[2], neg_m[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float m_new = fmaxf(m_run[r], mx[r] * scale_log2);
      corr[r] = fast_exp2(m_run[r] - m_new);
      m_run[r] = m_new;
      neg_m[r] = -m_new;
      l_run[r] *= corr[r];
    }
#pragma unroll
    for (int nt = 0; nt < BK / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float pv = fast_exp2(fmaf(s[nt][e], scale_log2, neg_m[e >> 1]));
        s[nt][e] = pv;
        l_run[e >> 1] += pv;
      }
    }
    if (__any_sync(0xffffffffu, corr[0] != 1.f || corr[1] != 1.f)) {  // running max moved: rescale O
#pragma unroll
      for (int dt = 0; dt < D / 8; ++dt) {
        o[dt][0] *= corr[0];
        o[dt][1] *= corr[0];
        o[dt][2] *= corr[1];
        o[dt][3] *= corr[1];
      }
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
        const int mi = lane >> 3;
        const int vr = kc * 16 + (mi & 1) * 8 + (lane & 7);
        const int vc = (dt + (mi >> 1)) * 8;
        uint32_t vb[4];
        ldmatrix_x4_trans(vb, cV + vr * LD + vc);
        mma_16816(o[dt], pa, vb[0], vb[1]);
        mma_16816(o[dt + 1], pa, vb[2], vb[3]);
      }
    }
    __syncthreads();  // everyone is done with this buffer before it is refilled
  }

#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 1);
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 2);
  }
  const float inv0 = 1.f / l_run[0], inv1 = 1.f / l_run[1];
  const int r0 = q0 + warp * 16 + gr;
  half* out = ctx + ((long long)g * group_rows + s0) * hidden + h * D;
  // context as an fp16 (hi, lo) pair: the O projection reads both terms (lo at out + lo_off)
#pragma unroll
  for (int dt = 0; dt < D / 8; ++dt) {
    const int c = dt * 8 + 2 * tq;
    uint32_t hi, lo;
    if (r0 < L) {
      split_half2(o[dt][0] * inv0, o[dt][1] * inv0, hi, lo);
      *reinterpret_cast<uint32_t*>(out + (long long)r0 * hidden + c) = hi;
      *reinterpret_cast<uint32_t*>(out + lo_off + (long long)r0 * hidden + c) = lo;
    }
    if (r0 + 8 < L) {
      split_half2(o[dt][2] * inv1, o[dt][3] * inv1, hi, lo);
      *reinterpret_cast<uint32_t*>(out + (long long)(r0 + 8) * hidden + c) = hi;
      *reinterpret_cast<uint32_t*>(out + lo_off + (long long)(r0 + 8) * hidden + c) = lo;
    }
  }
}

template <int D, int NW, int MINB, int NBUF>
static void launch_attn_t(const half* qkv, half* ctx, long long lo_off, const int* cu, int n_seqs, int max_len,
                          int groups, int n_heads, int hidden, long long group_rows, float scale_log2,
                          cudaStream_t stream) {
  constexpr int BQ = 16 * NW, LD = D + 8;
  const size_t smem = (size_t)(BQ + 2 * NBUF * 64) * LD * sizeof(half);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_kernel<D, NW, MINB, NBUF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  dim3 grid((max_len + BQ - 1) / BQ, n_seqs, groups * n_heads);
  launch_pdl(attn_kernel<D, NW, MINB, NBUF>, grid, dim3(32 * NW), smem, stream, qkv, ctx, cu, n_heads, hidden, group_rows,
             scale_log2, lo_off);
}

void launch_attention(const half* qkv, half* ctx, long long lo_off, const int* cu_seqlens, int n_seqs, int max_len,
                      int groups, int n_heads, int head_dim, int hidden, long long group_rows, cudaStream_t stream) {
  if (n_seqs <= 0 || max_len <= 0 || groups <= 0) return;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(head_dim));
  // query-tile height by length (measured sweep, tools/attn_bench.py); 385..448: 64-query tiles at
  // 4 CTAs/SM balance the waves that 128-query tiles quantize (4 tiles per head), 26 vs 29 us.
  // Resident CTAs per SM: 4 for 4 warps, else 2; a 2-deep K/V ring (4 measured no faster: the
  // kernel is compute-bound per CTA).
  const int nw = max_len <= 128 ? 4 : (max_len <= 288 ? 6 : (max_len <= 384 ? 8 : 4));
#define SP_ATTN(D_, NW_, B_) \
  launch_attn_t<D_, NW_, B_, 2>(qkv, ctx, lo_off, cu_seqlens, n_seqs, max_len, groups, n_heads, hidden, group_rows, \
                                scale_log2, stream)
  if (head_dim == 64) {
    if (nw == 8) SP_ATTN(64, 8, 2);
    else if (nw == 6) SP_ATTN(64, 6, 2);
    else SP_ATTN(64, 4, 4);
  } else {
    if (nw == 8) SP_ATTN(32, 8, 2);
    else if (nw == 6) SP_ATTN(32, 6, 2);
    else SP_ATTN(32, 4, 4);
  }
#undef SP_ATTN
}

}  // namespace sp
