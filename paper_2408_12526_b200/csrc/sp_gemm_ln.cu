// sp_gemm_ln.cu — projection + bias + residual + LayerNorm in one kernel (O and FFN2 of a layer).
//
// The H output features of a token row are spread over H/128 feature tiles, so LayerNorm needs
// a reduction across CTAs: the CTAs of one (student, token tile) — one per feature tile — form a
// thread-block cluster (H/128 <= 8 CTAs) and exchange per-token partial sums through distributed
// shared memory. Per CTA:
//   main loop  as sp_gemm.cu (TMA ring, tcgen05.mma into TMEM, weights prefetched before the
//              griddepcontrol.wait), full K (no split-K partials in HBM)
//   phase 1    v = acc + bias + residual  -> smem row buffer, per-token sum over 128 features
//   phase 2    cluster exchange: mean; per-token centered sum of squares (two-pass LayerNorm)
//   phase 3    cluster exchange: rstd; y = (v - mean) * rstd * gamma + beta -> x32, x16 (+ CLS rows)
// This replaces the split-K partial write + reduce_ln kernel pair (one HBM round trip of fp32
// partials and one kernel boundary per LayerNorm). Reference ops: DenseLayer.forward (identity)
// (nnkernel.py:66-76) followed by the post-LN residual of the BERT student (oracle/bert.py).
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"

namespace sp {

static constexpr int kLnBlockM = 128;
static constexpr int kLnBlockK = 64;
static constexpr int kLnATile = kLnBlockM * kLnBlockK * 2;
static constexpr int kLnThreads = 320;  // producer, MMA, 8 epilogue warps
static constexpr int kLnVStride = 129;  // fp32 row stride of the value buffer (conflict-free)

__device__ __forceinline__ int ln_seq_of(const int* cu, int n_seqs, int t) {
  int lo = 0, hi = n_seqs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(cu + mid) <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kLnThreads, 2)
    gemm_ln_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x64,
                   const __grid_constant__ CUtensorMap map_x16, const GemmParams p, const LnParams ln) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = kLnATile + p.bn * 128;
  float* stats = reinterpret_cast<float*>(smem + p.stages * stage_bytes);  // 4 x 128 floats
  float* cta_sum = stats;
  float* cta_sq = stats + 128;
  float* mean_s = stats + 256;
  uint64_t* full = reinterpret_cast<uint64_t*>(stats + 512);
  uint64_t* empty = full + p.stages;
  uint64_t* tmem_full = empty + p.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  float* vbuf = reinterpret_cast<float*>(smem);  // reuses the ring after the main loop: bn x 129 fp32

  const int m_tiles = p.m_tiles;
  const int mt = blockIdx.x % m_tiles;  // == cluster rank (cluster dims = m_tiles)
  const int nt = blockIdx.x / m_tiles;
  const int g = blockIdx.y;
  const int m0 = mt * kLnBlockM;
  const int n0 = nt * p.bn;
  const int nkb = p.k_dim / kLnBlockK;
  const int warp = warp_id();
  const int lane = lane_id();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x64);
    tma_prefetch_desc(&map_x16);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 128);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      const int wrow = g * p.n_out + m0;
      const int xrow = g * p.x_group_rows + n0;
      auto load_x = [&](int s, int kb) {
        uint8_t* sb = smem + s * stage_bytes + kLnATile;
        int r = 0;
        for (; r + 64 <= p.bn; r += 64) tma_load_2d(&map_x64, &full[s], sb + r * 128, kb * kLnBlockK, xrow + r, pol_x);
        for (; r < p.bn; r += 16) tma_load_2d(&map_x16, &full[s], sb + r * 128, kb * kLnBlockK, xrow + r, pol_x);
      };
      const int n_pre = min(p.stages, nkb);
      for (int i = 0; i < n_pre; ++i) {  // weights: independent of the previous kernel
        mbar_arrive_expect_tx(&full[i], stage_bytes);
        tma_load_2d(&map_w, &full[i], smem + i * stage_bytes, i * kLnBlockK, wrow, pol_w);
      }
      pdl_wait();
      for (int i = 0; i < n_pre; ++i) load_x(i, i);
      int s = n_pre % p.stages;
      uint32_t ph = (n_pre == p.stages) ? 1u : 0u;
      for (int kb = n_pre; kb < nkb; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        tma_load_2d(&map_w, &full[s], smem + s * stage_bytes, kb * kLnBlockK, wrow, pol_w);
        load_x(s, kb);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t idesc = umma_idesc_f16(kLnBlockM, p.bn);
      int s = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * stage_bytes);
        const uint64_t adesc = umma_sdesc_sw128(sa);
        const uint64_t bdesc = umma_sdesc_sw128(sa + kLnATile);
#pragma unroll
        for (int k = 0; k < kLnBlockK / 16; ++k)
          umma_f16_ss(tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
        umma_commit(&empty[s]);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
      umma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    // phase 1: v = acc + bias + residual -> vbuf[token][feature]; per-token partial sums
    const int e = warp - 2;
    const int q = warp & 3;
    const int half_cols = p.bn >> 1;
    const int c_begin = (e >> 2) * half_cols;
    const int f = q * 32 + lane;  // feature within the tile
    const float bias = __ldg(ln.bias + (long long)g * ln.hidden + m0 + f);
    const float* resid = ln.x32 + (long long)g * ln.x_gs + m0 + f;
    const int t_rows = p.t_dev ? __ldg(p.t_dev) : p.t_rows;
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16);
    for (int c = c_begin; c < c_begin + half_cols; c += 32) {
      const int n = min(32, c_begin + half_cols - c);
      uint32_t r[32];
      if (n == 32) {
        tmem_ld32_nowait(taddr + c, r);
      } else {
        for (int i = 0; i < n; i += 8) tmem_ld8_nowait(taddr + c + i, r + i);
      }
      float res[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int t = n0 + c + j;
        res[j] = (j < n && t < t_rows) ? resid[(long long)t * ln.hidden] : 0.f;
      }
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < n) vbuf[(c + j) * kLnVStride + f] = __uint_as_float(r[j]) + bias + res[j];
    }
    named_barrier_sync(1, 256);
    for (int col = e; col < p.bn; col += 8) {
      const float* row = vbuf + col * kLnVStride;
      float s = (row[lane] + row[lane + 32]) + (row[lane + 64] + row[lane + 96]);
      s = warp_sum(s);
      if (lane == 0) cta_sum[col] = s;
    }
  }
  __syncthreads();
  cluster_sync();  // every CTA of the row published its partial sums

  const bool epi = warp >= 2;
  const int e = warp - 2;
  if (epi) {
    const float inv_h = 1.0f / static_cast<float>(ln.hidden);
    for (int col = e; col < p.bn; col += 8) {
      float part = 0.f;
      if (lane < m_tiles) part = ld_shared_cluster_f32(mapa_shared(smem_u32(cta_sum + col), lane));
      const float mean = warp_sum(part) * inv_h;  // identical order in every CTA: same value
      const float* row = vbuf + col * kLnVStride;
      float qsum = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float d = row[lane + 32 * i] - mean;
        qsum += d * d;
      }
      qsum = warp_sum(qsum);
      if (lane == 0) {
        cta_sq[col] = qsum;
        mean_s[col] = mean;
      }
    }
  }
  __syncthreads();
  cluster_sync();  // centered sums of squares published

  if (epi) {
    const int t_rows = p.t_dev ? __ldg(p.t_dev) : p.t_rows;
    const float inv_h = 1.0f / static_cast<float>(ln.hidden);
    float gm[4], bt[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      gm[i] = __ldg(ln.gamma + (long long)g * ln.hidden + m0 + lane + 32 * i);
      bt[i] = __ldg(ln.beta + (long long)g * ln.hidden + m0 + lane + 32 * i);
    }
    for (int col = e; col < p.bn; col += 8) {
      float part = 0.f;
      if (lane < m_tiles) part = ld_shared_cluster_f32(mapa_shared(smem_u32(cta_sq + col), lane));
      const float var = warp_sum(part) * inv_h;
      const float rstd = rsqrtf(var + ln.eps);
      const float mean = mean_s[col];
      const int t = n0 + col;
      if (t < t_rows) {
        const float* row = vbuf + col * kLnVStride;
        float* o32 = ln.x32 + (long long)g * ln.x_gs + (long long)t * ln.hidden + m0;
        half* o16 = ln.x16 + (long long)g * ln.x_gs + (long long)t * ln.hidden + m0;
        half* ocls = nullptr;
        if (ln.cls16 != nullptr) {
          const int b = ln_seq_of(ln.cu, ln.n_seqs, t);
          if (__ldg(ln.cu + b) == t) ocls = ln.cls16 + (long long)g * ln.cls_gs + (long long)b * ln.hidden + m0;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int fi = lane + 32 * i;
          const float y = (row[fi] - mean) * rstd * gm[i] + bt[i];
          o32[fi] = y;
          const half hy = __float2half_rn(y);
          o16[fi] = hy;
          if (ocls) ocls[fi] = hy;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peers finished reading this CTA's statistics
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

size_t gemm_ln_smem_bytes(int bn, int stages) {
  return static_cast<size_t>(stages) * (kLnATile + bn * 128) + 512 * sizeof(float) + 1024 + 256;
}

void launch_gemm_ln(const GemmMaps& maps, const GemmParams& p, const LnParams& ln, int groups, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_ln_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.m_tiles * p.n_tiles, groups);
  cfg.blockDim = dim3(kLnThreads);
  cfg.dynamicSmemBytes = gemm_ln_smem_bytes(p.bn, p.stages);
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = p.m_tiles;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  prefer_max_smem(reinterpret_cast<const void*>(gemm_ln_kernel));
  cudaLaunchKernelEx(&cfg, gemm_ln_kernel, maps.w, maps.x64, maps.x16, p, ln);
}

}  // namespace sp
