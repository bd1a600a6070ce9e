// sp_mlp.cu — FFN1 (bias + erf-GELU) and FFN2 of one layer in ONE persistent kernel.
//
// Why: between the two projections the kernel boundary costs the FFN1 epilogue tail (the last
// tile's GELU drain, 3-5 us at L >= 256, nothing else runs) plus the FFN2 pipeline refill, and
// FFN1's last round leaves most SMs idle (e.g. 192 FFN1 tiles over 148 CTAs). Here every CTA
// first runs its FFN1 tiles (phase A) and then FFN2 tiles (phase B):
//   * warp 0 streams the weight k-blocks of both phases through the TMA ring; weights do not
//     depend on activations, so FFN2's weights fill the ring while FFN1 finishes;
//   * warp 18 loads the token-side k-blocks: phase A after griddepcontrol.wait (the LayerNorm
//     output), phase B once the student's FFN1 tiles are published (a per-student counter,
//     release/acquire + async-proxy fence), not at the grid boundary;
//   * phase-B tiles are dealt to CTAs in reverse order, so the CTAs with a single FFN1 tile take
//     the students whose FFN1 finished in the first round and run FFN2 while the rest of FFN1 runs.
// MMA / TMEM / epilogue are as in gemm_persistent_kernel (swap-AB 128 x bn tiles, two TMEM
// accumulators, 16 epilogue warps). The counters are reset by the last CTA to leave; the next
// launch cannot overlap this one (the LayerNorm kernel between two MLP launches triggers its
// dependents only after its own griddepcontrol.wait).
#include <algorithm>

#include "sp_kernels.cuh"
#include "sp_ptx.cuh"
#include "sp_device.cuh"

namespace sp {

namespace {

constexpr int kMBlockM = 128, kMBlockK = 64;
constexpr int kMATileBytes = kMBlockM * kMBlockK * 2;
constexpr int kMEpiWarps = 16;
constexpr int kMWarps = 2 + kMEpiWarps + 1;  // W producer, MMA, 16 epilogue, X producer
constexpr int kMThreads = 32 * kMWarps;
constexpr int kMXWarp = kMWarps - 1;
constexpr int kMTmemCols = 512;
constexpr int kMStageRowBytes = 32 * 2;  // epilogue staging row: 32 fp16 (phase A), 16 fp32 (B, two halves)

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct MlpPhase {
  int n_out, nkb, bn, n_tiles, m_tiles, splits, units;  // nkb: k-blocks per unit (one split's share)
};

__device__ __forceinline__ MlpPhase mlp_phase(const MlpParams& p, int ph) {
  MlpPhase f;
  f.n_out = ph == 0 ? p.n_a : p.n_b;
  f.splits = ph == 0 ? 1 : p.splits_b;
  f.nkb = (ph == 0 ? p.k_a : p.k_b) / kMBlockK / f.splits;
  f.bn = ph == 0 ? p.bn_a : p.bn_b;
  f.n_tiles = ph == 0 ? p.n_tiles_a : p.n_tiles_b;
  f.m_tiles = f.n_out / kMBlockM;
  f.units = p.groups * f.m_tiles * f.n_tiles * f.splits;
  return f;
}

// Unit -> (student, feature tile, token tile, split), feature tile fastest, split slowest.
__device__ __forceinline__ void mlp_decode(const MlpPhase& f, int u, int& g, int& mt, int& nt, int& sp) {
  const int per_split = f.units / f.splits;
  sp = u / per_split;
  u -= sp * per_split;
  const int per = f.m_tiles * f.n_tiles;
  g = u / per;
  const int r = u - g * per;
  nt = r / f.m_tiles;
  mt = r - nt * f.m_tiles;
}

// The CTA's k-th unit of phase ph (-1 when done): phase A in CTA order, phase B reversed.
__device__ __forceinline__ int mlp_unit(const MlpPhase& f, int ph, int k) {
  const int G = gridDim.x;
  const int first = ph == 0 ? (int)blockIdx.x : G - 1 - (int)blockIdx.x;
  const int u = first + k * G;
  return u < f.units ? u : -1;
}

__global__ void __launch_bounds__(kMThreads, 1)
    mlp_persistent_kernel(const __grid_constant__ MlpMaps m, const MlpParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // weight tile + the (hi, lo) token terms of the wider phase's tile
  const int stage_bytes = kMATileBytes + 2 * std::max(p.bn_a, p.bn_b) * 128;
  uint8_t* staging = smem + p.stages * stage_bytes;  // 16 warps x 16 rows x 128 B
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + kMEpiWarps * 16 * kMStageRowBytes);
  uint64_t* empty = full + p.stages;
  uint64_t* acc_full = empty + p.stages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 2);  // weight producer + activation producer
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kMEpiWarps);
    }
    fence_barrier_init();
    tma_prefetch_desc(&m.w_a);
    tma_prefetch_desc(&m.w_b);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, kMTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------------ weight producer
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();  // batch-1: each weight tile is read once or twice
      int s = 0;
      uint32_t ph = 0;
      for (int phase = 0; phase < 2; ++phase) {
        const MlpPhase f = mlp_phase(p, phase);
        const CUtensorMap* map = phase == 0 ? &m.w_a : &m.w_b;
        for (int k = 0;; ++k) {
          const int u = mlp_unit(f, phase, k);
          if (u < 0) break;
          int g, mt, nt, sp;
          mlp_decode(f, u, g, mt, nt, sp);
          const int wrow = g * f.n_out + mt * kMBlockM;
          const int kb0 = sp * f.nkb;
          for (int kb = kb0; kb < kb0 + f.nkb; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], kMATileBytes);
            tma_load_2d(map, &full[s], smem + s * stage_bytes, kb * kMBlockK, wrow, pol);
            if (++s == p.stages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == kMXWarp) {
    // ------------------------------------------------------------------ activation producer
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();  // re-read by every feature tile of the student
      int s = 0;
      uint32_t ph = 0;
      pdl_wait();  // phase A reads the LayerNorm output of the previous kernel
      for (int phase = 0; phase < 2; ++phase) {
        const MlpPhase f = mlp_phase(p, phase);
        const CUtensorMap* m64[2] = {phase == 0 ? &m.xa64 : &m.xb64, phase == 0 ? &m.xal64 : &m.xbl64};
        const CUtensorMap* m16[2] = {phase == 0 ? &m.xa16 : &m.xb16, phase == 0 ? &m.xal16 : &m.xbl16};
        const uint32_t x_bytes = (uint32_t)f.bn * 128u;  // per term
        const int a_tiles_per_student = (p.n_a / kMBlockM) * p.n_tiles_a;
        int dep_g = -1;
        for (int k = 0;; ++k) {
          const int u = mlp_unit(f, phase, k);
          if (u < 0) break;
          int g, mt, nt, sp;
          mlp_decode(f, u, g, mt, nt, sp);
          if (phase == 1 && g != dep_g) {  // every FFN1 tile of this student published
            const long long t0 = clock64();
            while (ld_acquire_gpu(p.done + g) < a_tiles_per_student) {
              __nanosleep(64);
              if (clock64() - t0 > 8000000000LL) __trap();
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
            dep_g = g;
          }
          const int xrow = g * p.x_group_rows + nt * f.bn;
          const int kb0 = sp * f.nkb;
          for (int kb = kb0; kb < kb0 + f.nkb; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], 2 * x_bytes);
            uint8_t* sb = smem + s * stage_bytes + kMATileBytes;
            for (int term = 0; term < 2; ++term, sb += x_bytes) {
              int r = 0;
              for (; r + 64 <= f.bn; r += 64)
                tma_load_2d(m64[term], &full[s], sb + r * 128, kb * kMBlockK, xrow + r, pol);
              for (; r < f.bn; r += 16) tma_load_2d(m16[term], &full[s], sb + r * 128, kb * kMBlockK, xrow + r, pol);
            }
            if (++s == p.stages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      int j = 0;
      for (int phase = 0; phase < 2; ++phase) {
        const MlpPhase f = mlp_phase(p, phase);
        const uint32_t idesc = umma_idesc_f16(kMBlockM, f.bn);
        for (int k = 0;; ++k, ++j) {
          if (mlp_unit(f, phase, k) < 0) break;
          const int b = j & 1;
          mbar_wait(&acc_empty[b], ((j >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t acc = tmem + static_cast<uint32_t>(b * 256);
          for (int kb = 0; kb < f.nkb; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + s * stage_bytes);
            const uint64_t adesc = umma_sdesc_sw128(sa);
            const uint64_t bdesc = umma_sdesc_sw128(sa + kMATileBytes);
            const uint64_t ldesc = umma_sdesc_sw128(sa + kMATileBytes + f.bn * 128);  // lo term
#pragma unroll
            for (int kk = 0; kk < kMBlockK / 16; ++kk) {
              umma_f16_ss(acc, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
              umma_f16_ss(acc, adesc + 2 * kk, ldesc + 2 * kk, idesc, 1u);
            }
            umma_commit(&empty[s]);
            if (++s == p.stages) {
              s = 0;
              ph ^= 1;
            }
          }
          umma_commit(&acc_full[b]);
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ epilogue warps
    const int e = warp - 2;
    const int q = warp & 3;
    const int t_rows = p.t_dev ? __ldg(p.t_dev) : p.t_rows;
    uint8_t* stage_base = staging + e * 16 * kMStageRowBytes;
    int j = 0;
    for (int phase = 0; phase < 2; ++phase) {
      const MlpPhase f = mlp_phase(p, phase);
      const int part_cols = f.bn >> 2;  // bn is a multiple of 32
      const int c_begin = (e >> 2) * part_cols;
      for (int k = 0;; ++k, ++j) {
        const int u = mlp_unit(f, phase, k);
        if (u < 0) break;
        int g, mt, nt, sp;
        mlp_decode(f, u, g, mt, nt, sp);
        const int b = j & 1;
        const int m0 = mt * kMBlockM, n0 = nt * f.bn;
        const int feat = m0 + q * 32 + lane;
        const float bias = phase == 0 ? __ldg(p.bias_a + (long long)g * p.bias_a_gs + feat) : 0.f;
        mbar_wait(&acc_full[b], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * 256);
        for (int c = c_begin; c < c_begin + part_cols; c += 16) {
          const int n = min(16, c_begin + part_cols - c);  // 8 or 16
          uint32_t r[16];
          tmem_ld8_nowait(taddr + c, r);
          if (n == 16) tmem_ld8_nowait(taddr + c + 8, r + 8);
          tmem_wait_ld();
          if (c + 16 >= c_begin + part_cols) {  // last TMEM read of this tile: release the accumulator
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);
          }
          if (phase == 0) {  // bias + erf-GELU -> fp16 (hi, lo) ffn activations
            constexpr int kRow = 64, kLanes = kRow / 16, kRowsPass = 32 / kLanes;
            half* st = reinterpret_cast<half*>(stage_base);
            float y[16];
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) y[jj] = gelu_erf(__uint_as_float(r[jj]) + bias);
            for (int term = 0; term < 2; ++term) {
              if (term) __syncwarp();
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) {
                const half h = __float2half_rn(y[jj]);
                st[jj * 32 + lane] = term ? __float2half_rn(y[jj] - __half2float(h)) : h;
              }
              __syncwarp();
              half* out = p.out_a + (term ? p.out_a_lo_off : 0) + (long long)g * p.out_a_gs + m0 + q * 32;
              const int sub = lane % kLanes;
              for (int j0 = 0; j0 < n; j0 += kRowsPass) {
                const int jr = j0 + lane / kLanes;
                const int t = n0 + c + jr;
                if (jr < n && t < t_rows) {
                  const uint4 v = *reinterpret_cast<const uint4*>(stage_base + jr * kRow + sub * 16);
                  *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(out + (long long)t * p.out_a_ld) + sub * 16) = v;
                }
              }
            }
          } else {  // raw fp32 projection (bias + residual + LayerNorm in the next kernel), 8 columns at a time
            constexpr int kRow = 128, kLanes = kRow / 16, kRowsPass = 32 / kLanes;
            float* st = reinterpret_cast<float*>(stage_base);
            float* out = p.out_b + (long long)sp * p.out_b_ss + (long long)g * p.out_b_gs + m0 + q * 32;
            const int sub = lane % kLanes;
            for (int h8 = 0; h8 < n; h8 += 8) {
              if (h8) __syncwarp();
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) st[jj * 32 + lane] = __uint_as_float(r[h8 + jj]);
              __syncwarp();
              for (int j0 = 0; j0 < 8; j0 += kRowsPass) {
                const int jr = j0 + lane / kLanes;
                const int t = n0 + c + h8 + jr;
                if (t < t_rows) {
                  const uint4 v = *reinterpret_cast<const uint4*>(stage_base + jr * kRow + sub * 16);
                  *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(out + (long long)t * p.out_b_ld) + sub * 16) = v;
                }
              }
            }
          }
          __syncwarp();
        }
        if (phase == 0) {  // publish this FFN1 tile for the student's FFN2 tiles
          asm volatile("fence.proxy.async.global;" ::: "memory");  // read next through TMA
          named_barrier_sync(1, 32 * kMEpiWarps);
          if (e == 0 && lane == 0) {
            __threadfence();
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.done + g) : "memory");
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kMTmemCols);
  }
  if (threadIdx.x == 0) {  // the last CTA out resets the counters for the next launch
    __threadfence();
    const int old = atomicAdd(p.done + kMlpMaxStudents, 1);
    if (old == (int)gridDim.x - 1) {
      for (int i = 0; i < p.groups; ++i) p.done[i] = 0;
      p.done[kMlpMaxStudents] = 0;
      __threadfence();
    }
  }
}

}  // namespace

int mlp_smem_bytes(int bn_max, int* stages) {
  const int staging = kMEpiWarps * 16 * kMStageRowBytes;
  const int stage = kMATileBytes + 2 * bn_max * 128;
  int st = (224 * 1024 - staging - 2048) / stage;
  if (st > 8) st = 8;
  if (stages) *stages = st;
  return 1024 + st * stage + staging + 512;
}

void launch_mlp(const MlpMaps& m, const MlpParams& p, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(mlp_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const int smem = mlp_smem_bytes(std::max(p.bn_a, p.bn_b), nullptr);
  const int units_a = p.groups * (p.n_a / kMBlockM) * p.n_tiles_a;
  const int units_b = p.groups * (p.n_b / kMBlockM) * p.n_tiles_b;
  const int n_sm = sm_count();
  int grid = std::max(units_a, units_b);
  if (grid > n_sm) grid = n_sm;
  launch_pdl(mlp_persistent_kernel, dim3(grid), dim3(kMThreads), smem, stream, m, p);
}

}  // namespace sp
