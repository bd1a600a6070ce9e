// sp_gemm.cu — student-batched projection GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Swap-AB: the weight slab is the UMMA "A" operand (M = 128 output features per CTA) and the
// request's tokens are the "B" operand (N = token tile, 16..256). At batch-1 the token count is
// small, so this puts the large dimension (weights, streamed once from HBM) on M and keeps every
// SM busy streaming a distinct weight slab; the student index is the grid's y axis (group axis).
//
// Warp roles (192 threads, one tile per CTA):
//   warp 0      TMA producer (one elected lane): W tile {64 x 128} + X tile {64 x bn} per stage
//   warp 1      TMEM allocator + MMA issuer (one elected lane): 4 x UMMA 128 x bn x 16 per stage
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers, bias + activation, store (quadrant = warp % 4)
//
// Reference op: DenseLayer.forward, z = x @ W.T + b then act (nnkernel.py:66-76).
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"

namespace sp {

static constexpr int kBlockM = 128;
static constexpr int kBlockK = 64;                      // one 128-byte swizzle row of fp16
static constexpr int kATileBytes = kBlockM * kBlockK * 2;  // 16 KiB
static constexpr int kTmemCols = 256;
static constexpr int kThreads = 192;

__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x64,
                const __grid_constant__ CUtensorMap map_x16, const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = kATileBytes + p.bn * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* tmem_full = empty + p.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  int bid = blockIdx.x;
  const int split = bid % p.splits;
  bid /= p.splits;
  const int nt = bid % p.n_tiles;
  const int mt = bid / p.n_tiles;
  const int g = blockIdx.y;
  const int m0 = mt * kBlockM;
  const int n0 = nt * p.bn;
  const int nkb = p.k_dim / kBlockK;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(kb0 + p.kb_per_split, nkb);

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
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights: streamed once per request
      const uint64_t pol_x = policy_evict_last();   // activations: re-read by every M tile
      const int wrow = g * p.n_out + m0;
      const int xrow = g * p.x_group_rows + n0;
      int s = 0;
      uint32_t ph = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * stage_bytes;
        uint8_t* sb = sa + kATileBytes;
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        const int kc = kb * kBlockK;
        tma_load_2d(&map_w, &full[s], sa, kc, wrow, pol_w);
        int r = 0;
        for (; r + 64 <= p.bn; r += 64) tma_load_2d(&map_x64, &full[s], sb + r * 128, kc, xrow + r, pol_x);
        for (; r < p.bn; r += 16) tma_load_2d(&map_x16, &full[s], sb + r * 128, kc, xrow + r, pol_x);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t idesc = umma_idesc_f16(kBlockM, p.bn);
      int s = 0;
      uint32_t ph = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * stage_bytes);
        const uint64_t adesc = umma_sdesc_sw128(sa);
        const uint64_t bdesc = umma_sdesc_sw128(sa + kATileBytes);
#pragma unroll
        for (int k = 0; k < kBlockK / 16; ++k) {
          // +32 bytes per K=16 slice inside the 128-byte swizzle row (address field is in 16-byte units)
          umma_f16_ss(tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
        }
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
    // Epilogue: warp w owns TMEM lanes 32*(w%4) .. +31, i.e. output features m0 + 32*(w%4) + lane.
    const int q = warp & 3;
    const int feat = m0 + q * 32 + lane;
    const bool partial = p.splits > 1;
    float bias = 0.f;
    if (!partial && p.bias != nullptr) bias = p.bias[(long long)g * p.bias_group_stride + feat];
    const bool has_k = kb1 > kb0;
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const long long obase = (long long)g * p.out_group_stride + (long long)split * p.out_split_stride + feat;
    for (int c = 0; c < p.bn; c += 16) {
      float v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int t = n0 + c + j;
        if (t < p.t_rows) {
          float y = has_k ? v[j] : 0.f;
          if (!partial) {
            y += bias;
            if (p.act == ACT_TANH) y = tanhf(y);
            else if (p.act == ACT_GELU) y = gelu_erf(y);
          }
          const long long o = obase + (long long)t * p.out_ld;
          if (p.out_f32) reinterpret_cast<float*>(p.out)[o] = y;
          else reinterpret_cast<half*>(p.out)[o] = __float2half_rn(y);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

size_t gemm_smem_bytes(int bn, int stages) {
  return static_cast<size_t>(stages) * (kATileBytes + bn * 128) + 1024 /*align*/ + 256 /*barriers*/;
}

void gemm_configure_tiles(int t_rows, int* bn, int* n_tiles, int* stages) {
  int tiles = (t_rows + 255) / 256;
  if (tiles < 1) tiles = 1;
  int per = (t_rows + tiles - 1) / tiles;
  int b = ((per + 15) / 16) * 16;
  if (b < 16) b = 16;
  *bn = b;
  *n_tiles = tiles;
  // <= ~100 KiB for small token tiles (two CTAs per SM), ~200 KiB otherwise.
  const int budget = (b <= 64) ? 100 * 1024 : 200 * 1024;
  int st = budget / (kATileBytes + b * 128);
  if (st > 8) st = 8;
  if (st < 2) st = 2;
  *stages = st;
}

void launch_gemm(const GemmMaps& maps, const GemmParams& p, int groups, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  dim3 grid(p.m_tiles * p.n_tiles * p.splits, groups);
  gemm_kernel<<<grid, kThreads, gemm_smem_bytes(p.bn, p.stages), stream>>>(maps.w, maps.x64, maps.x16, p);
}

}  // namespace sp
