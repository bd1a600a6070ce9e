// sp_gemm.cu — student-batched projection GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Swap-AB: the weight slab is the UMMA "A" operand (M = 128 output features per CTA) and the
// request's tokens are the "B" operand (N = token tile, 16..128). At batch-1 the token count is
// small, so the large dimension (weights, streamed once from HBM) sits on M and every SM streams
// a distinct weight slab; the student index is the grid's y axis (the group axis).
//
// Warp roles (320 threads, one output tile per CTA, <= ~100 KiB smem so two CTAs share an SM):
//   warp 0       TMA producer (one elected lane): W tile {64 x 128} + X tile {64 x bn} per stage
//   warp 1       TMEM allocator + MMA issuer (one elected lane): 4 x UMMA 128 x bn x 16 per stage
//   warps 2..9   epilogue: tcgen05.ld TMEM -> registers (x32), bias + activation, per-warp smem
//                transpose, 16-byte coalesced stores. Warp w reads TMEM lane quadrant w % 4 and
//                one half of the token columns.
//
// Programmatic dependent launch: weights never depend on the previous kernel, so the producer
// issues the weight loads of the first pipeline stages BEFORE griddepcontrol.wait and only the
// activation loads after it — the weight stream of this projection overlaps the tail of the
// previous kernel (attention / LayerNorm / another projection).
//
// Reference op: DenseLayer.forward, z = x @ W.T + b then act (nnkernel.py:66-76).
#include <cstdlib>
#include <type_traits>
#include <vector>

#include <algorithm>

#include "sp_kernels.cuh"
#include "sp_ptx.cuh"

namespace sp {

static constexpr int kBlockM = 128;
static constexpr int kBlockK = 64;                         // one 128-byte swizzle row of fp16
static constexpr int kATileBytes = kBlockM * kBlockK * 2;  // 16 KiB
// TMEM columns of the small-T kernel: the next power of two >= bn (>= 32), so that CTAs of the next
// projection, launched early (PDL), can allocate theirs while this one still runs (512 per SM)
__device__ __forceinline__ uint32_t tmem_cols_for(int bn) {
  uint32_t c = 32;
  while (c < static_cast<uint32_t>(bn)) c <<= 1;
  return c;
}
static constexpr int kEpiWarps = 8;
static constexpr int kThreads = 64 + 32 * kEpiWarps;
static constexpr int kMaxBn = 256;

template <int ACT>
__device__ __forceinline__ float apply_act(float y) {
  if constexpr (ACT == ACT_TANH) return tanhf(y);
  else if constexpr (ACT == ACT_GELU) return gelu_erf(y);
  else return y;
}

// Epilogue store of one warp's 32-feature x n-token block: stage rows in the warp's smem slice,
// then 16-byte row stores (rows past t_rows are skipped).
template <typename OutT, int NR>
__device__ __forceinline__ void warp_store_rows(const float (&y)[NR], int n, OutT* stage, OutT* out, int t0,
                                                int t_rows, int out_ld, bool lo_term) {
  constexpr int kRowBytes = 32 * static_cast<int>(sizeof(OutT));
  constexpr int kLanesPerRow = kRowBytes / 16;
  constexpr int kRowsPerPass = 32 / kLanesPerRow;
  const int lane = lane_id();
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if constexpr (std::is_same<OutT, float>::value) {
      stage[j * 32 + lane] = y[j];
    } else {
      const half h = __float2half_rn(y[j]);
      stage[j * 32 + lane] = lo_term ? __float2half_rn(y[j] - __half2float(h)) : h;
    }
  }
  __syncwarp();
  const int sub = lane % kLanesPerRow;
  for (int j0 = 0; j0 < n; j0 += kRowsPerPass) {
    const int j = j0 + lane / kLanesPerRow;
    const int t = t0 + j;
    if (j < n && t < t_rows) {
      const uint4 v = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(stage) + j * kRowBytes + sub * 16);
      *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(out + (long long)t * out_ld) + sub * 16) = v;
    }
  }
  __syncwarp();
}

template <bool WHILO>
using MapsOf = typename std::conditional<WHILO, GemmMapsW, GemmMaps>::type;

template <int ACT, bool OUT_F32, bool HILO, bool WHILO>
__global__ void __launch_bounds__(kThreads, 2)
    gemm_kernel(const __grid_constant__ MapsOf<WHILO> maps, const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int x_bytes = p.bn * 128;                            // one term of the token tile
  constexpr int a_bytes = kATileBytes * (WHILO ? 2 : 1);     // weight tile (+ its lo term)
  const int stage_bytes = a_bytes + x_bytes * (HILO ? 2 : 1);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* tmem_full = empty + p.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  int bid = blockIdx.x;
  const int mt = bid % p.m_tiles;
  bid /= p.m_tiles;
  const int nt = bid % p.n_tiles;
  const int split = bid / p.n_tiles;
  const int g = blockIdx.y;
  const int m0 = mt * kBlockM;
  const int n0 = nt * p.bn;
  const int nkb = p.k_dim / kBlockK;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(kb0 + p.kb_per_split, nkb);

  const int warp = warp_id();
  const int lane = lane_id();
  unsigned long long* tr = p.trace ? p.trace + 8ull * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  // weights: streamed once per request -> evict_first, unless several token tiles re-read them
  const uint64_t pol_w = (p.n_tiles > 1 && p.w_keep) ? policy_evict_last() : policy_evict_first();
  const int n_pre = min(p.stages, kb1 - kb0);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
    tma_prefetch_desc(&maps.w);
    // first weight stages right away: independent of the TMEM allocation, the CTA barrier and the
    // previous kernel (weights never depend on it)
    for (int i = 0; i < n_pre; ++i) {
      mbar_arrive_expect_tx(&full[i], stage_bytes);
      tma_load_2d(&maps.w, &full[i], smem + i * stage_bytes, (kb0 + i) * kBlockK, g * p.w_gs + p.w_r0 + m0, pol_w);
      if constexpr (WHILO)
        tma_load_2d(&maps.wl, &full[i], smem + i * stage_bytes + kATileBytes, (kb0 + i) * kBlockK,
                    g * p.w_gs + p.w_r0 + m0, pol_w);
    }
    tma_prefetch_desc(&maps.x64);
    tma_prefetch_desc(&maps.x16);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, tmem_cols_for(p.bn));
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();
  if (tr && threadIdx.x == 0) tr[1] = globaltimer();

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_x = policy_evict_last();   // activations: re-read by every M tile
      const int wrow = g * p.w_gs + p.w_r0 + m0;
      const int xrow = g * p.x_group_rows + n0;
      auto load_x = [&](int s, int kb) {
        uint8_t* sb = smem + s * stage_bytes + a_bytes;
        const int kc = kb * kBlockK;
        for (int term = 0; term < (HILO ? 2 : 1); ++term, sb += x_bytes) {
          const CUtensorMap* m64 = term ? &maps.xl64 : &maps.x64;
          const CUtensorMap* m16 = term ? &maps.xl16 : &maps.x16;
          int r = 0;
          for (; r + 64 <= p.bn; r += 64) tma_load_2d(m64, &full[s], sb + r * 128, kc, xrow + r, pol_x);
          for (; r < p.bn; r += 16) tma_load_2d(m16, &full[s], sb + r * 128, kc, xrow + r, pol_x);
        }
      };
      if (tr) tr[2] = globaltimer();
      // activations are produced by the previous kernel
      pdl_wait();
      if (tr) tr[3] = globaltimer();  // dependency released
      for (int i = 0; i < n_pre; ++i) load_x(i, kb0 + i);
      int s = n_pre % p.stages;
      uint32_t ph = (n_pre == p.stages) ? 1u : 0u;
      for (int kb = kb0 + n_pre; kb < kb1; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        tma_load_2d(&maps.w, &full[s], smem + s * stage_bytes, kb * kBlockK, wrow, pol_w);
        if constexpr (WHILO)
          tma_load_2d(&maps.wl, &full[s], smem + s * stage_bytes + kATileBytes, kb * kBlockK, wrow, pol_w);
        load_x(s, kb);
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
        if (tr && kb == kb0) tr[4] = globaltimer();
        const uint32_t sa = smem_u32(smem + s * stage_bytes);
        const uint64_t adesc = umma_sdesc_sw128(sa);
        const uint64_t aldesc = umma_sdesc_sw128(sa + kATileBytes);  // weight lo term (whilo)
        const uint64_t bdesc = umma_sdesc_sw128(sa + a_bytes);
        const uint64_t ldesc = umma_sdesc_sw128(sa + a_bytes + x_bytes);
#pragma unroll
        for (int k = 0; k < kBlockK / 16; ++k) {
          // +32 bytes per K=16 slice inside the 128-byte swizzle row (address field in 16-byte units)
          umma_f16_ss(tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          if constexpr (HILO) umma_f16_ss(tmem, adesc + 2 * k, ldesc + 2 * k, idesc, 1u);
          if constexpr (WHILO) umma_f16_ss(tmem, aldesc + 2 * k, bdesc + 2 * k, idesc, 1u);
        }
        umma_commit(&empty[s]);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
      umma_commit(tmem_full);
      if (tr) tr[5] = globaltimer();
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue
    const int e = warp - 2;  // 0..epi_warps-1
    const int q = warp & 3;  // TMEM lane quadrant (hardware: warp w accesses lanes 32*(w%4)..)
    const int half_cols = p.epi_warps == 8 ? (p.bn >> 1) : p.bn;  // 4 warps: every column
    const int c_begin = (e >> 2) * half_cols;
    const int feat = m0 + q * 32 + lane;
    const bool partial = p.splits > 1;
    float bias = 0.f;
    if (!partial && p.bias != nullptr) bias = __ldg(p.bias + (long long)g * p.bias_group_stride + feat);
    const bool has_k = kb1 > kb0;
    using OutT = typename std::conditional<OUT_F32, float, half>::type;
    OutT* stage = reinterpret_cast<OutT*>(smem + e * 32 * 32 * sizeof(OutT));  // warp-private, ring is free now
    OutT* out = reinterpret_cast<OutT*>(p.out) + (long long)g * p.out_group_stride +
                (long long)split * p.out_split_stride + m0 + q * 32;

    const int t_rows = p.t_dev ? __ldg(p.t_dev) : p.t_rows;  // graph replay: live count from cu_seqlens
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    if (tr && warp == 2 && lane == 0) tr[6] = globaltimer();
    const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const long long lo_off = (OUT_F32 || m0 < p.lo_from) ? 0 : p.out_lo_off;
    // one chunk of NR accumulator columns (NR = 8 / 16 / 32 >= n: a 16-token tile computes its
    // activation for 16 columns, not 32; the columns of a chunk are independent chains)
    auto chunk = [&](auto nr, int c, int n) {
      constexpr int NR = decltype(nr)::value;
      uint32_t r[NR];
      if constexpr (NR == 32) {
        if (n == 32) tmem_ld32_nowait(taddr + c, r);
        else
          for (int i = 0; i < n; i += 8) tmem_ld8_nowait(taddr + c + i, r + i);
      } else {
#pragma unroll
        for (int i = 0; i < NR; i += 8) tmem_ld8_nowait(taddr + c + i, r + i);
      }
      tmem_wait_ld();
      float y[NR];
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        y[j] = has_k ? __uint_as_float(r[j]) : 0.f;
        if (!partial) y[j] = apply_act<ACT>(y[j] + bias);
      }
      warp_store_rows<OutT, NR>(y, n, stage, out, n0 + c, t_rows, p.out_ld, false);
      if (lo_off) warp_store_rows<OutT, NR>(y, n, stage, out + lo_off, n0 + c, t_rows, p.out_ld, true);
    };
    for (int c = c_begin; c < c_begin + half_cols; c += 32) {
      // columns of this chunk that hold live tokens (CLS-row GEMMs: n_seqs of a 16-wide tile;
      // graph replay: the live length inside the bucket), rounded up to the TMEM load width 8
      const int live = t_rows - (n0 + c);
      if (live <= 0) break;                      // warp-uniform
      const int n = min(min(32, c_begin + half_cols - c), (live + 7) & ~7);
      if (n > 16) chunk(std::integral_constant<int, 32>{}, c, n);
      else if (n > 8) chunk(std::integral_constant<int, 16>{}, c, n);
      else chunk(std::integral_constant<int, 8>{}, c, n);
    }
    if (tr && warp == 2 && lane == 0) tr[7] = globaltimer();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols_for(p.bn));
  }
}

// Debug trace: launches append their per-CTA stamps one after another (slot 0 of the buffer
// holds the number of CTAs recorded so far, host-side mirror in g_trace_used).
static unsigned long long* trace_ptr_advance(int ctas, int aux_kind = 0);

// ============================================================================ persistent variant
// For large token counts (T > 128: long batch-1 requests, batched load) one CTA per SM loops over
// output tiles (128 features x bn tokens, bn <= 256) with a continuous TMA ring and two TMEM
// accumulators: the MMAs of tile i+1 run while the 8 epilogue warps drain tile i, so neither the
// pipeline fill nor the epilogue is paid per tile, and there are no partial waves. Tiles are
// ordered m-tile fastest, so concurrently running CTAs share one token tile (L2 hits).
static constexpr int kPersistTmemCols = 512;  // 2 accumulators x 256 columns
static constexpr int kPEpiWarps = 16;          // 4 warps per TMEM lane quadrant, a quarter of the columns each
static constexpr int kPThreads = 64 + 32 * kPEpiWarps;

template <int ACT, bool OUT_F32, bool PAIR, bool HILO, bool WHILO>
__global__ void __launch_bounds__(kPThreads, 1)
    gemm_persistent_kernel(const __grid_constant__ MapsOf<WHILO> maps, const GemmParams p) {
  using OutT = typename std::conditional<OUT_F32, float, half>::type;
  constexpr int kRowBytes = 32 * static_cast<int>(sizeof(OutT));
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // pair mode (cluster of 2, cta_group::2): the pair computes a 256-feature x bn-token tile with one
  // MMA stream issued by the leader; each CTA stages its own 128 weight rows and HALF of the token
  // tile, so per-CTA operand traffic per flop drops by a third (bn = 256) and the leader's TMEM-
  // resident accumulator rows 0-127 / the peer's rows 128-255 are drained by each CTA's epilogue.
  // (a kernel containing cta_group::2 instructions only launches in clusters: PAIR is a template
  // parameter so the single-CTA instantiation has none)
  constexpr bool pair = PAIR;
  const uint32_t crank = pair ? cluster_ctarank() : 0u;
  const bool leader = crank == 0;
  const int x_rows = pair ? (p.bn >> 1) : p.bn;  // token rows staged by this CTA (per term)
  const int x_bytes = x_rows * 128;
  constexpr int a_bytes = kATileBytes * (WHILO ? 2 : 1);  // weight tile (+ its lo term)
  const int stage_bytes = a_bytes + x_bytes * (HILO ? 2 : 1);
  uint8_t* staging = smem + p.stages * stage_bytes;  // 16 warps x 16 rows x kRowBytes
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + kPEpiWarps * 16 * kRowBytes);
  uint64_t* empty = full + p.stages;
  uint64_t* acc_full = empty + p.stages;  // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  unsigned long long* tr = p.trace ? p.trace + 8ull * blockIdx.x : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  const int m_per = pair ? (p.m_tiles >> 1) : p.m_tiles;
  const int units_per_group = m_per * p.n_tiles;
  const int units = units_per_group * p.groups;
  const int u_first = pair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int u_stride = pair ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int nkb = p.k_dim / kBlockK;
  // the leader's barrier collects both CTAs' bytes; the pair's epilogues both release its accumulator
  const uint32_t full_bytes = pair ? 2u * (uint32_t)stage_bytes : (uint32_t)stage_bytes;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], pair ? 2 * kPEpiWarps : kPEpiWarps);
    }
    fence_barrier_init();
    tma_prefetch_desc(&maps.w);
    if constexpr (!PAIR) {  // first unit's weight stages right away (before TMEM allocation / CTA barrier)
      if (u_first < units) {
        const int g = u_first / units_per_group;
        const int mt = (u_first % units_per_group) % m_per;
        const uint64_t pol_w = p.w_keep == 2 ? policy_evict_last() : (p.w_keep == 1 ? policy_evict_normal()
                                                                                     : policy_evict_first());
        const int n_pre = min(p.stages, nkb);
        for (int i = 0; i < n_pre; ++i) {
          mbar_arrive_expect_tx(&full[i], full_bytes);
          tma_load_2d(&maps.w, &full[i], smem + i * stage_bytes, i * kBlockK, g * p.w_gs + p.w_r0 + mt * kBlockM, pol_w);
          if constexpr (WHILO)
            tma_load_2d(&maps.wl, &full[i], smem + i * stage_bytes + kATileBytes, i * kBlockK,
                        g * p.w_gs + p.w_r0 + mt * kBlockM, pol_w);
        }
      }
    }
    tma_prefetch_desc(&maps.x64);
    tma_prefetch_desc(&maps.x16);
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      tmem_alloc_2sm(tmem_slot, kPersistTmemCols);
      tmem_relinquish_2sm();
    } else {
      tmem_alloc(tmem_slot, kPersistTmemCols);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // peer barriers initialised before any remote complete_tx / arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();

  auto decode = [&](int u, int& g, int& mt, int& nt) {
    g = u / units_per_group;
    const int r = u % units_per_group;
    nt = r / m_per;
    mt = pair ? 2 * (r % m_per) + static_cast<int>(crank) : r % m_per;
  };

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = p.w_keep == 2 ? policy_evict_last() : (p.w_keep == 1 ? policy_evict_normal()
                                                                                     : policy_evict_first());
      const uint64_t pol_x = policy_evict_last();
      auto load_w = [&](int s, int kb, int wrow) {
        uint8_t* sa = smem + s * stage_bytes;
        if constexpr (PAIR) {
          tma_load_2d_2sm(&maps.w, &full[s], sa, kb * kBlockK, wrow, pol_w);
          if constexpr (WHILO) tma_load_2d_2sm(&maps.wl, &full[s], sa + kATileBytes, kb * kBlockK, wrow, pol_w);
        } else {
          tma_load_2d(&maps.w, &full[s], sa, kb * kBlockK, wrow, pol_w);
          if constexpr (WHILO) tma_load_2d(&maps.wl, &full[s], sa + kATileBytes, kb * kBlockK, wrow, pol_w);
        }
      };
      auto load_x = [&](int s, int kb, int xrow) {
        uint8_t* sb = smem + s * stage_bytes + a_bytes;
        for (int term = 0; term < (HILO ? 2 : 1); ++term, sb += x_bytes) {
          const CUtensorMap* m64 = term ? &maps.xl64 : &maps.x64;
          const CUtensorMap* m16 = term ? &maps.xl16 : &maps.x16;
          int r = 0;
          if constexpr (PAIR) {
            for (; r + 64 <= x_rows; r += 64) tma_load_2d_2sm(m64, &full[s], sb + r * 128, kb * kBlockK, xrow + r, pol_x);
            for (; r < x_rows; r += 16) tma_load_2d_2sm(m16, &full[s], sb + r * 128, kb * kBlockK, xrow + r, pol_x);
          } else {
            for (; r + 64 <= x_rows; r += 64) tma_load_2d(m64, &full[s], sb + r * 128, kb * kBlockK, xrow + r, pol_x);
            for (; r < x_rows; r += 16) tma_load_2d(m16, &full[s], sb + r * 128, kb * kBlockK, xrow + r, pol_x);
          }
        }
      };
      int s = 0;
      uint32_t ph = 0;
      bool first = true;
      for (int u = u_first; u < units; u += u_stride) {
        int g, mt, nt;
        decode(u, g, mt, nt);
        const int wrow = g * p.w_gs + p.w_r0 + mt * kBlockM;
        const int xrow = g * p.x_group_rows + nt * p.bn + (int)crank * x_rows;
        int kb = 0;
        if (first) {  // weight prefetch of the first stages before the dependency wait
          const int n_pre = min(p.stages, nkb);
          if constexpr (PAIR)  // (single CTA: already issued at entry)
            for (int i = 0; i < n_pre; ++i) {
              if (leader) mbar_arrive_expect_tx(&full[i], full_bytes);
              load_w(i, i, wrow);
            }
          if (tr) tr[2] = globaltimer();
          pdl_wait();
          for (int i = 0; i < n_pre; ++i) load_x(i, i, xrow);
          kb = n_pre;
          s = n_pre % p.stages;
          ph = (n_pre == p.stages) ? 1u : 0u;
          first = false;
        }
        for (; kb < nkb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], full_bytes);
          load_w(s, kb, wrow);
          load_x(s, kb, xrow);
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      if (first) pdl_wait();  // no work: still honour the dependency
    }
  } else if (warp == 1) {
    if (leader && elect_one()) {
      const uint32_t idesc = umma_idesc_f16(pair ? 2 * kBlockM : kBlockM, p.bn);
      int s = 0;
      uint32_t ph = 0;
      int j = 0;
      unsigned long long w_acc = 0, w_full = 0;  // trace: ns the MMA thread waited on each barrier kind
      for (int u = u_first; u < units; u += u_stride, ++j) {
        const int b = j & 1;
        unsigned long long t0 = tr ? globaltimer() : 0ull;
        mbar_wait(&acc_empty[b], ((j >> 1) & 1) ^ 1);  // epilogue(s) drained this accumulator
        if (tr) w_acc += globaltimer() - t0;
        tc_fence_after();
        const uint32_t acc = tmem + static_cast<uint32_t>(b * 256);
        for (int kb = 0; kb < nkb; ++kb) {
          if (tr) t0 = globaltimer();
          mbar_wait(&full[s], ph);
          if (tr) w_full += globaltimer() - t0;
          tc_fence_after();
          if (tr && j == 0 && kb == 0) tr[4] = globaltimer();
          const uint32_t sa = smem_u32(smem + s * stage_bytes);
          const uint64_t adesc = umma_sdesc_sw128(sa);
          const uint64_t aldesc = umma_sdesc_sw128(sa + kATileBytes);      // weight lo term (whilo)
          const uint64_t bdesc = umma_sdesc_sw128(sa + a_bytes);
          const uint64_t ldesc = umma_sdesc_sw128(sa + a_bytes + x_bytes);  // token lo term (hilo)
          if constexpr (PAIR) {
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k) {
              umma_f16_ss_2sm(acc, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              if constexpr (HILO) umma_f16_ss_2sm(acc, adesc + 2 * k, ldesc + 2 * k, idesc, 1u);
              if constexpr (WHILO) umma_f16_ss_2sm(acc, aldesc + 2 * k, bdesc + 2 * k, idesc, 1u);
            }
            umma_commit_2sm_mc(&empty[s], 0x3);
          } else {
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k) {
              umma_f16_ss(acc, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              if constexpr (HILO) umma_f16_ss(acc, adesc + 2 * k, ldesc + 2 * k, idesc, 1u);
              if constexpr (WHILO) umma_f16_ss(acc, aldesc + 2 * k, bdesc + 2 * k, idesc, 1u);
            }
            umma_commit(&empty[s]);
          }
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
        if constexpr (PAIR) umma_commit_2sm_mc(&acc_full[b], 0x3);
        else umma_commit(&acc_full[b]);
      }
      if (tr) {
        tr[5] = globaltimer();
        tr[1] = w_full;
        tr[3] = w_acc;
      }
    }
    __syncwarp();
  } else {
    const int e = warp - 2;
    const int q = warp & 3;
    const int wg = e >> 2;            // warp group 0..3: 16-column chunks wg, wg + 4, ...
    const int n_chunks = p.bn >> 4;   // bn is a multiple of 16
    OutT* stage = reinterpret_cast<OutT*>(staging + e * 16 * kRowBytes);
    const int t_rows = p.t_dev ? __ldg(p.t_dev) : p.t_rows;
    const long long lo_off = OUT_F32 ? 0 : p.out_lo_off;
    // accumulator release: local barrier, or the leader's through the cluster window
    uint32_t acc_empty_leader0 = 0u;
    if constexpr (PAIR) acc_empty_leader0 = mapa_shared(smem_u32(&acc_empty[0]), 0);
    auto release = [&](int b) {  // after this warp's last TMEM read of the tile
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) mbar_arrive_cluster(acc_empty_leader0 + (uint32_t)(b * sizeof(uint64_t)));
        else mbar_arrive(&acc_empty[b]);
      }
    };
    int j = 0;
    for (int u = u_first; u < units; u += u_stride, ++j) {
      int g, mt, nt;
      decode(u, g, mt, nt);
      const int b = j & 1;
      const int m0 = mt * kBlockM, n0 = nt * p.bn;
      const int feat = m0 + q * 32 + lane;
      const float bias = p.bias ? __ldg(p.bias + (long long)g * p.bias_group_stride + feat) : 0.f;
      OutT* out = reinterpret_cast<OutT*>(p.out) + (long long)g * p.out_group_stride + m0 + q * 32;
      mbar_wait(&acc_full[b], (j >> 1) & 1);
      tc_fence_after();
      if (tr && j == 0 && warp == 2 && lane == 0) tr[6] = globaltimer();
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * 256);
      // chunks holding live tokens only (graph replay: the live length inside the bucket)
      const int live = t_rows - n0;
      const int live_chunks = live <= 0 ? 0 : min(n_chunks, (live + 15) >> 4);
      bool released = false;
      for (int ci = wg; ci < live_chunks; ci += 4) {
        const int c = ci * 16;
        uint32_t r[16];
        tmem_ld8_nowait(taddr + c, r);
        tmem_ld8_nowait(taddr + c + 8, r + 8);
        tmem_wait_ld();
        if (ci + 4 >= live_chunks) {
          release(b);
          released = true;
        }
        float y[16];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) y[jj] = apply_act<ACT>(__uint_as_float(r[jj]) + bias);
        warp_store_rows<OutT, 16>(y, 16, stage, out, n0 + c, t_rows, p.out_ld, false);
        if (lo_off && m0 >= p.lo_from)
          warp_store_rows<OutT, 16>(y, 16, stage, out + lo_off, n0 + c, t_rows, p.out_ld, true);
      }
      if (!released) release(b);  // no (live) chunk for this warp in this tile
    }
    if (tr && warp == 2 && lane == 0) tr[7] = globaltimer();
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // no CTA leaves while its peer may still signal into it
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_2sm(tmem, kPersistTmemCols);
    else tmem_dealloc(tmem, kPersistTmemCols);
  }
}

template <int ACT, bool OUT_F32, bool HILO, bool WHILO>
static void launch_persistent_t(const GemmMapsW& maps, const GemmParams& p, int groups, cudaStream_t stream) {
  static int n_sm = 0;
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(gemm_persistent_kernel<ACT, OUT_F32, false, HILO, WHILO>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(gemm_persistent_kernel<ACT, OUT_F32, true, HILO, WHILO>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  GemmParams q = p;
  q.groups = groups;
  q.cluster = gemm_persistent_pair(p.t_rows, p.m_tiles, groups) ? 2 : 1;
  const int units = groups * p.m_tiles * p.n_tiles;  // per-CTA tiles (a pair takes two at once)
  int grid = units < n_sm ? units : n_sm;
  if (q.cluster == 2) grid &= ~1;
  q.trace = trace_ptr_advance(grid);
  const int row_bytes = 32 * (OUT_F32 ? 4 : 2);
  const int x_rows = q.cluster == 2 ? p.bn / 2 : p.bn;
  const size_t smem = static_cast<size_t>(q.stages) *
                          (kATileBytes * (WHILO ? 2 : 1) + x_rows * 128 * (HILO ? 2 : 1)) +
                      kPEpiWarps * 16 * row_bytes + 1024 + 256;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = q.cluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  const MapsOf<WHILO>& m = maps;  // the BERT instantiations get the plain maps (no weight-lo map)
  if (q.cluster == 2) cudaLaunchKernelEx(&cfg, gemm_persistent_kernel<ACT, OUT_F32, true, HILO, WHILO>, m, q);
  else cudaLaunchKernelEx(&cfg, gemm_persistent_kernel<ACT, OUT_F32, false, HILO, WHILO>, m, q);
}

// CTA pairs (cta_group::2) halve each CTA's token-tile traffic (both (hi, lo) terms): from 256 tokens
// (batch-1 L = 448 / 512: 227 / 237 us against 249 / 258 with single-CTA tiles and the fused MLP;
// equal at 256-384; mixed below: profiles/r2_pair_threshold.txt).
bool gemm_persistent_pair(int t_rows, int m_tiles, int groups) {
  return t_rows >= 256 && m_tiles % 2 == 0 && groups * m_tiles >= 4;
}

// Tile policy of the persistent path: pick the token-tile count that minimises the makespan
// ceil(units / CTAs) x (fixed + bn) (bn <= 256), so projections with few feature tiles (O, FFN2:
// 6 per student) still fill every SM; ring as deep as the smem left after staging.
// Every operand is an (hi, lo) pair: two token terms per stage and two MMAs per k-slice.
void gemm_configure_persistent(int t_rows, bool out_f32, int units_per_tile, int n_ctas, bool pair, int* bn,
                               int* n_tiles, int* stages, int gran_override) {
  // Cost of a tiling = rounds x per-unit time, in cycles per 64-wide k-block of one CTA:
  //   MMA      2 * 2 * bn                          (two 128 x bn x 64 MMAs at 8192 flop/clk)
  //   operands 3 * (128 + 2 * token rows staged)   (L2 -> SM at ~42 B/clk per SM, 12.4 TB/s / 148)
  // plus ~200 cycles of per-unit fill / drain. Pairs stage half the token tile per CTA and run
  // units_per_tile / 2 units on n_ctas / 2 pairs.
  const int ctas = pair ? n_ctas / 2 : n_ctas;
  const int upt = pair ? units_per_tile / 2 : units_per_tile;
  // the tile count is chosen on 32-column tiles (the model was fitted there); the chosen tile is then
  // trimmed to a 16-column multiple (MMA N step; the epilogue deals 16-column chunks round-robin)
  // unless the caller needs 32 (pairs stage bn / 2 rows per CTA in 16-row TMA boxes; the fused MLP)
  const int gran = 32;
  const int trim = gran_override ? gran_override : (pair ? 32 : 16);
  int best_tiles = (t_rows + 255) / 256;
  long long best_cost = 0x7fffffffffffll;
  for (int tiles = (t_rows + 255) / 256; tiles <= (t_rows + 63) / 64; ++tiles) {
    const int per = (t_rows + tiles - 1) / tiles;
    const int b = ((per + gran - 1) / gran) * gran;
    if (b > 256) continue;
    const int x = pair ? b / 2 : b;
    const long long rounds = (upt * (long long)tiles + ctas - 1) / ctas;
    const long long unit = std::max(4LL * b, 3LL * (128 + 2 * x)) + 200;
    const long long cost = rounds * unit;
    if (cost < best_cost) {
      best_cost = cost;
      best_tiles = tiles;
    }
  }
  const int tiles = best_tiles;
  const int per = (t_rows + tiles - 1) / tiles;
  int b = ((per + gran - 1) / gran) * gran;
  // trim only where it does not add TMA boxes per token term (64- and 16-row boxes: 33 tokens stay
  // one 64-row box rather than three 16-row boxes — measured slower)
  auto boxes = [](int rows) { return rows / 64 + (rows % 64) / 16; };
  const int bt = ((per + trim - 1) / trim) * trim;
  if (bt < b && boxes(bt) <= boxes(b)) b = bt;
  *bn = b;
  *n_tiles = tiles;
  const int staging = kPEpiWarps * 16 * 32 * (out_f32 ? 4 : 2);
  int st = (224 * 1024 - staging) / (kATileBytes + (pair ? b / 2 : b) * 128 * 2);
  if (st > 8) st = 8;
  if (st < 2) st = 2;
  *stages = st;
}

// Operand modes are template parameters (a runtime branch in the MMA-issue loop measured 2-7 us
// per batch-1 request): token (hi, lo) pair or hi only; the weight-lo operand is instantiated for
// the dense kind's tanh projections only.
template <int ACT, bool OUT_F32>
static void launch_persistent_x(const GemmMapsW& maps, const GemmParams& p, int groups, cudaStream_t stream) {
  if (p.hilo) launch_persistent_t<ACT, OUT_F32, true, false>(maps, p, groups, stream);
  else launch_persistent_t<ACT, OUT_F32, false, false>(maps, p, groups, stream);
}
template <bool OUT_F32>
static void launch_persistent_w(const GemmMapsW& maps, const GemmParams& p, int groups, cudaStream_t stream) {
  if (p.hilo) launch_persistent_t<ACT_TANH, OUT_F32, true, true>(maps, p, groups, stream);
  else launch_persistent_t<ACT_TANH, OUT_F32, false, true>(maps, p, groups, stream);
}

void launch_gemm_persistent(const GemmMapsW& maps, const GemmParams& p, int groups, cudaStream_t stream) {
  const bool f32 = p.out_f32 != 0;
  if (p.whilo) {
    if (f32) launch_persistent_w<true>(maps, p, groups, stream);
    else launch_persistent_w<false>(maps, p, groups, stream);
  } else if (p.act == ACT_GELU) {
    if (f32) launch_persistent_x<ACT_GELU, true>(maps, p, groups, stream);
    else launch_persistent_x<ACT_GELU, false>(maps, p, groups, stream);
  } else if (p.act == ACT_TANH) {
    if (f32) launch_persistent_x<ACT_TANH, true>(maps, p, groups, stream);
    else launch_persistent_x<ACT_TANH, false>(maps, p, groups, stream);
  } else {
    if (f32) launch_persistent_x<ACT_NONE, true>(maps, p, groups, stream);
    else launch_persistent_x<ACT_NONE, false>(maps, p, groups, stream);
  }
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

static unsigned long long* g_trace = nullptr;
static size_t g_trace_used = 0;
static std::vector<int> g_trace_counts;
void set_gemm_trace(unsigned long long* buf) {
  g_trace = buf;
  g_trace_used = 0;
  g_trace_counts.clear();
}
static unsigned long long* trace_ptr_advance(int ctas, int aux_kind) {
  if (!g_trace) return nullptr;
  unsigned long long* p = g_trace + 8 * g_trace_used;
  g_trace_used += (size_t)ctas;
  // GEMMs: the CTA count; other kernels: -(kind * 100000 + CTA count)
  g_trace_counts.push_back(aux_kind ? -(aux_kind * 100000 + ctas) : ctas);
  return p;
}
unsigned long long* trace_alloc_aux(int ctas, int kind) { return trace_ptr_advance(ctas, kind); }

int gemm_trace_counts(int* out, int max) {
  const int n = static_cast<int>(g_trace_counts.size());
  for (int i = 0; i < n && i < max; ++i) out[i] = g_trace_counts[i];
  return n;
}

// stage = weight tile + both token terms (the smem size does not depend on hilo being used)
size_t gemm_smem_bytes(int bn, int stages, int whilo) {
  return static_cast<size_t>(stages) * (kATileBytes * (whilo ? 2 : 1) + 2 * bn * 128) + 1024 /*align*/ +
         256 /*barriers*/;
}

int gemm_whilo_stages(int x_rows, bool persistent, bool out_f32) {
  const int stage = 2 * kATileBytes + 2 * x_rows * 128;
  if (persistent) {
    const int staging = kPEpiWarps * 16 * 32 * (out_f32 ? 4 : 2);
    return std::max(2, std::min(8, (224 * 1024 - staging) / stage));
  }
  return std::max(2, std::min(6, (110 * 1024) / stage));
}

void gemm_configure_tiles(int t_rows, int* bn, int* n_tiles, int* stages) {
  // token-tile cap: 64 up to 128 tokens (two tiles at 65-128 tokens: more CTAs stream the split-K
  // weights, -4..-6 us at 96-128 measured in-graph), else 128
  const int max_bn = t_rows <= 128 ? 64 : 128;
  int tiles = (t_rows + max_bn - 1) / max_bn;
  if (tiles < 1) tiles = 1;
  const int per = (t_rows + tiles - 1) / tiles;
  int b = ((per + 15) / 16) * 16;
  if (b < 16) b = 16;
  *bn = b;
  *n_tiles = tiles;
  // ~110 KiB per CTA so that two CTAs (e.g. the tail of one projection and the prefetching head
  // of the next, or two tiles of one projection) share an SM: smem 2 x <= 111 KiB, TMEM <= 2 x 128 cols.
  int st = (110 * 1024) / (kATileBytes + 2 * b * 128);
  if (st > 6) st = 6;
  if (st < 2) st = 2;
  *stages = st;
}

template <int ACT, bool OUT_F32, bool HILO, bool WHILO>
static void launch_gemm_t(const GemmMapsW& maps, const GemmParams& p, int groups, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_kernel<ACT, OUT_F32, HILO, WHILO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.m_tiles * p.n_tiles * p.splits, groups);
  cfg.blockDim = dim3(64 + 32 * p.epi_warps);
  cfg.dynamicSmemBytes = gemm_smem_bytes(p.bn, p.stages, WHILO);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GemmParams q = p;
  q.trace = g_trace ? g_trace + 8 * g_trace_used : nullptr;
  if (g_trace) {
    g_trace_used += (size_t)cfg.gridDim.x * cfg.gridDim.y;
    g_trace_counts.push_back(static_cast<int>(cfg.gridDim.x * cfg.gridDim.y));
  }
  const MapsOf<WHILO>& m = maps;
  cudaLaunchKernelEx(&cfg, gemm_kernel<ACT, OUT_F32, HILO, WHILO>, m, q);
}

// Epilogue warps of the small-T kernel: 4 (192 threads) unless the launch has several wide token
// tiles (measured in-graph: 4 warps -1..-3 us at 96-192 tokens, 8 warps better at 256 = 2 x 128).
int gemm_epi_warps(int bn, int n_tiles) { return (bn <= 96 || n_tiles == 1) ? 4 : 8; }

template <int ACT, bool OUT_F32>
static void launch_gemm_x(const GemmMapsW& maps, const GemmParams& p, int groups, cudaStream_t stream) {
  if (p.hilo) launch_gemm_t<ACT, OUT_F32, true, false>(maps, p, groups, stream);
  else launch_gemm_t<ACT, OUT_F32, false, false>(maps, p, groups, stream);
}
template <bool OUT_F32>
static void launch_gemm_w(const GemmMapsW& maps, const GemmParams& p, int groups, cudaStream_t stream) {
  if (p.hilo) launch_gemm_t<ACT_TANH, OUT_F32, true, true>(maps, p, groups, stream);
  else launch_gemm_t<ACT_TANH, OUT_F32, false, true>(maps, p, groups, stream);
}

void launch_gemm(const GemmMapsW& maps, const GemmParams& p, int groups, cudaStream_t stream) {
  const bool f32 = p.out_f32 || p.splits > 1;
  const int act = p.splits > 1 ? ACT_NONE : p.act;
  if (p.whilo) {  // dense kind: tanh projections, one split
    if (f32) launch_gemm_w<true>(maps, p, groups, stream);
    else launch_gemm_w<false>(maps, p, groups, stream);
  } else if (act == ACT_GELU) {
    if (f32) launch_gemm_x<ACT_GELU, true>(maps, p, groups, stream);
    else launch_gemm_x<ACT_GELU, false>(maps, p, groups, stream);
  } else if (act == ACT_TANH) {
    if (f32) launch_gemm_x<ACT_TANH, true>(maps, p, groups, stream);
    else launch_gemm_x<ACT_TANH, false>(maps, p, groups, stream);
  } else {
    if (f32) launch_gemm_x<ACT_NONE, true>(maps, p, groups, stream);
    else launch_gemm_x<ACT_NONE, false>(maps, p, groups, stream);
  }
}

}  // namespace sp
