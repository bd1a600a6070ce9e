// sp_attn_tc2.cu — single-pass varlen attention on 5th-gen tensor cores (head_dim 64, L <= 512).
//
// attn_tc2_kernel<TRACE, SPLIT>: one CTA per (student, sequence, head, 128-query block), two CTAs
// per SM (320 threads at SPLIT = 2, 256 TMEM columns); one's softmax runs while the other waits on
// its MMAs or loads:
//   softmax warps: 4 * SPLIT; thread = query row = TMEM lane (warp w owns lanes 32(w%4)..+31) and
//              128 / SPLIT key columns of each chunk; running max m and sum l per row (online
//              softmax, log2 domain), row maxima / sums of the SPLIT column groups via smem
//   warp 4*SPLIT     TMA producer: Q once, then 128-key K/V chunks through a 2-stage ring
//   warp 4*SPLIT+1   TMEM allocation + MMA issue (one elected lane)
// TMEM: S = Q K^T of the current chunk in columns [0, 128) (fp32), P = exp2(S - m) as packed fp16
// in [128, 192), O in [192, 256). O += P V reads P straight from TMEM (tcgen05.mma A operand in
// tensor memory), so P never touches shared memory.
//   chunk j: MMA S_j -> softmax reads S_j to registers and frees S (the MMA of S_{j+1} overlaps
//   the exponentials) -> row max -> P_j = exp2(S*c - m) -> waits PV_{j-1} -> writes P_j -> MMA
//   O += P_j V_j.
// Lazy rescale: the running max m is only raised when a chunk's max exceeds it by more than
// 2^8 (P <= 256 stays exact in fp16, l in fp32); then the thread rescales its O row in TMEM
// (after PV_{j-1} completed) — rare after the first chunk. Keys past the sequence end are masked;
// query rows past it are not stored.
// attn_tc3_kernel (below): the same algorithm with 64-key chunks and P written over its own scores
// (128 TMEM columns), three CTAs per SM — one wave for up to 512 tokens.
// No reference counterpart; semantics = oracle/bert.py:attention.
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"
#include "sp_device.cuh"

#include <cstdlib>

namespace sp {

namespace {

constexpr int kTile = 128 * 64 * 2;  // 128 rows x 64 fp16 = 16 KiB
// SPLIT softmax warps per TMEM lane quadrant, each owning 128 / SPLIT key columns of a chunk
template <int SPLIT>
struct Tc2Cfg {
  static constexpr int kSoftWarps = 4 * SPLIT;
  static constexpr int kThreads = 32 * (kSoftWarps + 2);
  static constexpr int kProd = kSoftWarps, kMma = kSoftWarps + 1;
  static constexpr int kCols = 128 / SPLIT;  // S columns per softmax thread
  static constexpr int kGroups = kCols / 32;
  static constexpr int kMinBlocks = 2;
};
constexpr uint32_t kColS = 0, kColP = 128, kColO = 192;
constexpr float kRescaleLog2 = 8.f;

__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

}  // namespace

// TRACE (debug, tools/trace_attn.py): 16 %globaltimer stamps per CTA into `tr`.
template <bool TRACE, int SPLIT>
__global__ void __launch_bounds__(Tc2Cfg<SPLIT>::kThreads, Tc2Cfg<SPLIT>::kMinBlocks)
    attn_tc2_kernel(const __grid_constant__ CUtensorMap map_qkv, half* __restrict__ ctx, const int* __restrict__ cu,
                    int n_heads, int hidden, long long group_rows, float scale_log2, unsigned long long* tr,
                    long long lo_off) {
  using C = Tc2Cfg<SPLIT>;
  constexpr int kSoftWarps = C::kSoftWarps, kProd = C::kProd, kMma = C::kMma, NG = C::kGroups;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kTile;      // [2] stages
  uint8_t* sV = sK + 2 * kTile;  // [2] stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * kTile);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* s_free = bars + 6;
  uint64_t* p_full = bars + 7;
  uint64_t* pv_done = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  float* xch = reinterpret_cast<float*>(bars + 10);  // SPLIT = 2: [2 chunk parities][2 halves][128 rows]

  if (TRACE) tr += 16ull * (blockIdx.x + gridDim.x * (blockIdx.y + (unsigned long long)gridDim.y * blockIdx.z));
  if (TRACE && threadIdx.x == 0) tr[0] = globaltimer();
  pdl_launch_dependents();
  // grid (student x head, sequence, query tile): the query tile is the slowest index, so the CTAs
  // of the last (partial, mostly dead-warp) tiles of every head are dispatched last and fill the
  // second wave instead of full tiles (4 tiles per head at L > 384 vs 296 CTA slots)
  const int b = blockIdx.y;
  const int s0 = __ldg(cu + b);  // request input: read before the dependency wait
  const int L = __ldg(cu + b + 1) - s0;
  const int q0 = blockIdx.z * 128;
  if (q0 >= L) return;
  const int g = blockIdx.x / n_heads;
  const int h = blockIdx.x % n_heads;
  const int n_chunks = (L + 127) >> 7;
  const int row_base = static_cast<int>(g * group_rows + s0);
  const int warp = warp_id();
  const int lane = lane_id();

  if (warp == kProd && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, kSoftWarps);
    mbar_init(p_full, kSoftWarps);
    mbar_init(pv_done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&map_qkv);
  }
  if (warp == kMma) {
    tmem_alloc(tmem_slot, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (TRACE && threadIdx.x == 0) tr[1] = globaltimer();

  if (warp == kProd) {
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();
      pdl_wait();  // qkv is the previous kernel's output
      mbar_arrive_expect_tx(q_full, kTile);
      tma_load_2d(&map_qkv, q_full, sQ, h * 64, row_base + q0, pol);
      for (int j = 0; j < n_chunks; ++j) {
        const int st = j & 1;
        if (j >= 2) mbar_wait(&kv_empty[st], ((j >> 1) - 1) & 1);
        if (TRACE && j < 4) tr[10 + j] = globaltimer();
        mbar_arrive_expect_tx(&kv_full[st], 2 * kTile);
        tma_load_2d(&map_qkv, &kv_full[st], sK + st * kTile, hidden + h * 64, row_base + j * 128, pol);
        tma_load_2d(&map_qkv, &kv_full[st], sV + st * kTile, 2 * hidden + h * 64, row_base + j * 128, pol);
      }
    }
    __syncwarp();
  } else if (warp == kMma) {
    if (elect_one()) {
      const uint32_t idesc_s = umma_idesc_f16(128, 128);
      const uint32_t idesc_o = umma_idesc_f16(128, 64) | (1u << 16);  // B (= V) is MN-major
      const uint64_t qdesc = umma_sdesc_sw128(smem_u32(sQ));
      mbar_wait(q_full, 0);
      auto issue_s = [&](int j) {
        mbar_wait(&kv_full[j & 1], (j >> 1) & 1);
        if (j >= 1) mbar_wait(s_free, (j - 1) & 1);  // softmax holds S_{j-1} in registers
        tc_fence_after();
        const uint64_t kdesc = umma_sdesc_sw128(smem_u32(sK + (j & 1) * kTile));
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_f16_ss(tmem + kColS, qdesc + 2 * k, kdesc + 2 * k, idesc_s, k > 0 ? 1u : 0u);
        umma_commit(s_full);
      };
      issue_s(0);
      if (tr) tr[2] = globaltimer();
      for (int j = 0; j < n_chunks; ++j) {
        if (j + 1 < n_chunks) issue_s(j + 1);  // next scores while the softmax works on chunk j
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const uint8_t* vb = sV + (j & 1) * kTile;
#pragma unroll
        for (int k = 0; k < 8; ++k)  // 16 keys per step: P columns 8k.. (2 fp16 each), V rows 16k..
          umma_f16_ts(tmem + kColO, tmem + kColP + 8 * k, umma_sdesc_sw128(smem_u32(vb + k * 2048)), idesc_o,
                      (j > 0 || k > 0) ? 1u : 0u);
        umma_commit(pv_done);
        umma_commit(&kv_empty[j & 1]);
      }
    }
    __syncwarp();
  } else {
    // softmax: thread = query row q0 + row = TMEM lane row; with SPLIT = 2 the two warps of a lane
    // quadrant take one half of the chunk's key columns each and exchange row maxima through smem
    const int quad = warp & 3, hf = warp >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t col0 = static_cast<uint32_t>(hf * C::kCols);
    float m = 0.f, l = 0.f;
    // A warp whose 32 query rows all lie past the sequence end (the tail tile of a head) skips
    // the TMEM traffic and the exponentials; it still takes part in every barrier phase. Its P
    // lanes keep stale values: the O rows they feed are never stored.
    const bool live = q0 + quad * 32 < L;
    for (int j = 0; j < n_chunks; ++j) {
      mbar_wait(s_full, j & 1);
      if (!live) {
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);
        if (j >= 1) mbar_wait(pv_done, (j - 1) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        continue;
      }
      tc_fence_after();
      if (TRACE && threadIdx.x == 0 && j < 4) tr[2 + j] = globaltimer();
      uint32_t r[NG][32];
#pragma unroll
      for (int c = 0; c < NG; ++c) tmem_ld32_nowait(tmem + lane_base + kColS + col0 + 32 * c, r[c]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);  // S may be overwritten by the next chunk's MMA
      const int valid = L - j * 128 - static_cast<int>(col0);  // keys of this warp's columns inside the sequence
      if (valid < C::kCols) {  // last chunk only
#pragma unroll
        for (int c = 0; c < NG; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (32 * c + i >= valid) r[c][i] = __float_as_uint(-INFINITY);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < NG; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(r[c][i]));
      if constexpr (SPLIT == 2) {
        float* x = xch + (j & 1) * 256;
        x[hf * 128 + row] = mx;
        named_barrier_sync(1 + quad, 64);
        mx = fmaxf(mx, x[(hf ^ 1) * 128 + row]);
      }
      mx *= scale_log2;
      float alpha = 1.f;
      if (j == 0) {
        m = mx;
      } else if (mx > m + kRescaleLog2) {
        alpha = ex2(m - mx);
        m = mx;
        l *= alpha;
      }
      const float neg_m = -m;
      uint32_t pk[NG * 16];
#pragma unroll
      for (int c = 0; c < NG; ++c) {
        float ps = 0.f;
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float p0 = ex2(fmaf(__uint_as_float(r[c][i]), scale_log2, neg_m));
          const float p1 = ex2(fmaf(__uint_as_float(r[c][i + 1]), scale_log2, neg_m));
          ps += p0 + p1;
          __half2 hp = __floats2half2_rn(p0, p1);
          pk[c * 16 + (i >> 1)] = *reinterpret_cast<uint32_t*>(&hp);
        }
        l += ps;
      }
      if (j >= 1) {
        mbar_wait(pv_done, (j - 1) & 1);  // PV_{j-1} has read P and updated O
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {  // rare: rescale this warp's share of its O rows
#pragma unroll
          for (int c = 0; c < 2 / SPLIT; ++c) {
            uint32_t o[32];
            const uint32_t oc = tmem + lane_base + kColO + 32 * (hf + c);
            tmem_ld32_nowait(oc, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(oc, o);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NG / 2; ++c) {
        uint32_t w32[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) w32[i] = pk[c * 32 + i];
        tmem_st32(tmem + lane_base + kColP + col0 / 2 + 32 * c, w32);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (TRACE && threadIdx.x == 0 && j < 4) tr[6 + j] = globaltimer();
    }
    // epilogue: O / l -> fp16 -> ctx (this warp's 64 / SPLIT columns of one row per thread)
    if constexpr (SPLIT == 2) {  // row sums of the two column halves
      float* x = xch + 512;
      if (live) x[hf * 128 + row] = l;
      named_barrier_sync(1 + quad, 64);
      if (live) l += x[(hf ^ 1) * 128 + row];
    }
    mbar_wait(pv_done, (n_chunks - 1) & 1);
    if (TRACE && threadIdx.x == 0) tr[14] = globaltimer();
    if (!live) goto done;
    tc_fence_after();
    {
      constexpr int OC = 64 / SPLIT;  // output columns of this thread
      uint32_t o[OC];
#pragma unroll
      for (int c = 0; c < OC / 32; ++c)
        tmem_ld32_nowait(tmem + lane_base + kColO + hf * OC + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(o + 32 * c));
      tmem_wait_ld();
      if (q0 + row < L) {
        const float inv = 1.f / l;
        uint4* out = reinterpret_cast<uint4*>(ctx + (static_cast<long long>(row_base) + q0 + row) * hidden + h * 64 +
                                              hf * OC);
        uint4* out_lo = reinterpret_cast<uint4*>(reinterpret_cast<half*>(out) + lo_off);
#pragma unroll
        for (int v = 0; v < OC / 8; ++v) {
          uint32_t w[4], l[4];  // (hi, lo) pair
#pragma unroll
          for (int i = 0; i < 4; ++i)
            split_half2(__uint_as_float(o[v * 8 + 2 * i]) * inv, __uint_as_float(o[v * 8 + 2 * i + 1]) * inv, w[i],
                        l[i]);
          out[v] = make_uint4(w[0], w[1], w[2], w[3]);
          out_lo[v] = make_uint4(l[0], l[1], l[2], l[3]);
        }
      }
    }
  }
done:
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
  if (TRACE && threadIdx.x == 0) tr[15] = globaltimer();
}

size_t attn_tc2_smem_bytes() { return 1024 + 5 * kTile + 128 + 3 * 1024; }

static unsigned long long* g_attn_trace = nullptr;
void set_attn_trace(unsigned long long* buf) { g_attn_trace = buf; }

template <int SPLIT>
static void launch_tc2_t(const CUtensorMap& map_qkv, half* ctx, long long lo_off, const int* cu_seqlens, dim3 grid,
                         int n_heads, int hidden, long long group_rows, float scale_log2, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_tc2_kernel<false, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(attn_tc2_smem_bytes()));
    cudaFuncSetAttribute(attn_tc2_kernel<true, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(attn_tc2_smem_bytes()));
    attr_set = true;
  }
  const dim3 block(Tc2Cfg<SPLIT>::kThreads);
  if (g_attn_trace)
    launch_pdl(attn_tc2_kernel<true, SPLIT>, grid, block, attn_tc2_smem_bytes(), stream, map_qkv, ctx, cu_seqlens,
               n_heads, hidden, group_rows, scale_log2, g_attn_trace, lo_off);
  else
    launch_pdl(attn_tc2_kernel<false, SPLIT>, grid, block, attn_tc2_smem_bytes(), stream, map_qkv, ctx, cu_seqlens,
               n_heads, hidden, group_rows, scale_log2, static_cast<unsigned long long*>(nullptr), lo_off);
}

// Two softmax warps per TMEM lane quadrant (SPLIT = 2: each thread owns a 64-key half of its row;
// -1.5..2 us per layer at L > 384 against one thread per full row).
void launch_attention_tc2(const CUtensorMap& map_qkv, half* ctx, long long lo_off, const int* cu_seqlens, int n_seqs,
                          int max_len, int groups, int n_heads, int hidden, long long group_rows, cudaStream_t stream) {
  if (n_seqs <= 0 || max_len <= 0 || groups <= 0) return;
  const float scale_log2 = 1.4426950408889634f / 8.0f;  // log2(e) / sqrt(64)
  dim3 grid(groups * n_heads, n_seqs, (max_len + 127) / 128);
  launch_tc2_t<2>(map_qkv, ctx, lo_off, cu_seqlens, grid, n_heads, hidden, group_rows, scale_log2, stream);
}


// ---------------------------------------------------------------------------------------------
// Variant "tc3": 64-key chunks, three CTAs per SM (192 threads <= 113 registers, 51 KiB smem,
// 128 TMEM columns: S in [0, 64) with P written back over its first 32 columns, O in [64, 128)).
// With P aliased into S the next chunk's scores are issued after O += P V (in-order tensor pipe),
// so a CTA's chunks are serial; the third resident CTA per SM supplies the overlap, and up to 444
// CTAs (L <= 512: 4 query tiles x 96 heads = 384) run in one wave. Because S_j is issued after
// PV_{j-1}, scores ready implies the previous PV finished: the softmax may rescale O right away.
// Thread = query row (4 softmax warps), 64 keys per chunk; producer warp, MMA warp.
// D (head_dim) = 64: 128-byte rows, SWIZZLE_128B; D = 32 (the tiny config): 64-byte rows,
// SWIZZLE_64B, half the K steps of S = Q K^T and an N = 32 P V product.
namespace {
constexpr int kT3Threads = 192;
constexpr uint32_t k3ColS = 0, k3ColO = 64;
template <int D>
struct T3 {
  static constexpr int kQ = 128 * D * 2;   // query tile
  static constexpr int kKv = 64 * D * 2;   // one 64-key chunk of K (or V)
  static __device__ __forceinline__ uint64_t desc(uint32_t a) {
    return D == 64 ? umma_sdesc_sw128(a) : umma_sdesc_sw64(a);
  }
};
}  // namespace

// QLO: V is an (hi, lo) fp16 pair (the lo tile at map row + lo_rows) and P is split into (hi, lo)
// too: O += Ph Vh + Ph Vl + Pl Vh (three MMAs per 16-key step), so the context carries ~22-bit
// operands like the projections. The fp16 rounding of V and P dominated the adaptive-prefix cases
// whose logits cancel (tools/diag_prefix.py: V 0.7-3.0e-3, P 0.1-1.3e-3 of max|z|; Q and K
// together <= 4.8e-4 there, but 9.6e-4 in K32 seed 146's k=30 prefix: hence QKLO, the default).
// QKLO (implies QLO): Q and K are (hi, lo) pairs too: S = Qh Kh + Ql Kh + Qh Kl. 99 KiB of shared
// memory per CTA (two CTAs per SM): +0 us up to L=384, +14 us at L=512 (two waves, len_probe).
template <int D, bool QLO, bool QKLO = false, int NS = 2>
__global__ void __launch_bounds__(kT3Threads, 3)
    attn_tc3_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                    half* __restrict__ ctx, const int* __restrict__ cu, int n_heads, int hidden, long long group_rows,
                    float scale_log2, long long lo_off, unsigned long long* trace, long long lo_rows) {
  // debug trace (8 stamps per CTA): entry, dependency released, first S issued, scores seen by the
  // softmax, last P V issued, P V done seen by the epilogue, end
  unsigned long long* tr =
      trace ? trace + 8ull * ((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  static_assert(D == 64 || D == 32, "head_dim 64 or 32");
  constexpr int kKv64 = T3<D>::kKv;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  static_assert(QLO || !QKLO, "QKLO implies QLO");
  uint8_t* sQ = smem;                 // 16 KiB (D = 64) / 8 KiB
  uint8_t* sQl = sQ + T3<D>::kQ;      // QKLO: Q lo
  uint8_t* sK = sQl + (QKLO ? T3<D>::kQ : 0);  // [2] x 8 / 4 KiB
  static_assert(NS == 1 || NS == 2, "K/V ring of one or two 64-key stages");
  uint8_t* sV = sK + NS * kKv64;      // [NS] x 8 / 4 KiB
  uint8_t* sVl = sV + NS * kKv64;     // QLO: [NS] V lo
  uint8_t* sKl = sVl + (QLO ? NS * kKv64 : 0);  // QKLO: [NS] K lo
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKl + (QKLO ? NS * kKv64 : 0));
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* p_full = bars + 6;
  uint64_t* pv_done = bars + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  pdl_launch_dependents();
  const int b = blockIdx.y;
  const int s0 = __ldg(cu + b);  // request input: read before the dependency wait
  const int L = __ldg(cu + b + 1) - s0;
  const int q0 = blockIdx.z * 128;
  if (q0 >= L) return;
  const int g = blockIdx.x / n_heads;
  const int h = blockIdx.x % n_heads;
  const int n_chunks = (L + 63) >> 6;
  const int row_base = static_cast<int>(g * group_rows + s0);
  const int warp = warp_id();
  const int lane = lane_id();
  constexpr int kProd3 = 4, kMma3 = 5;

  if (warp == kProd3 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(pv_done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_kv);
  }
  if (warp == kMma3) {
    tmem_alloc(tmem_slot, 128);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProd3) {
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();
      pdl_wait();  // qkv is the previous kernel's output
      if (tr) tr[1] = globaltimer();
      mbar_arrive_expect_tx(q_full, (QKLO ? 2 : 1) * T3<D>::kQ);
      tma_load_2d(&map_q, q_full, sQ, h * D, row_base + q0, pol);
      if constexpr (QKLO) tma_load_2d(&map_q, q_full, sQl, h * D, (int)(row_base + q0 + lo_rows), pol);
      for (int j = 0; j < n_chunks; ++j) {
        const int st = j % NS;
        if (j >= NS) mbar_wait(&kv_empty[st], (j / NS - 1) & 1);
        mbar_arrive_expect_tx(&kv_full[st], (QKLO ? 4 : QLO ? 3 : 2) * kKv64);
        tma_load_2d(&map_kv, &kv_full[st], sK + st * kKv64, hidden + h * D, row_base + j * 64, pol);
        tma_load_2d(&map_kv, &kv_full[st], sV + st * kKv64, 2 * hidden + h * D, row_base + j * 64, pol);
        if constexpr (QLO)
          tma_load_2d(&map_kv, &kv_full[st], sVl + st * kKv64, 2 * hidden + h * D, (int)(row_base + j * 64 + lo_rows),
                      pol);
        if constexpr (QKLO)
          tma_load_2d(&map_kv, &kv_full[st], sKl + st * kKv64, hidden + h * D, (int)(row_base + j * 64 + lo_rows),
                      pol);
      }
    }
    __syncwarp();
  } else if (warp == kMma3) {
    if (elect_one()) {
      const uint32_t idesc_s = umma_idesc_f16(128, 64);
      const uint32_t idesc_o = umma_idesc_f16(128, D) | (1u << 16);  // B (= V) is MN-major
      const uint64_t qdesc = T3<D>::desc(smem_u32(sQ));
      mbar_wait(q_full, 0);
      auto issue_s = [&](int j) {
        mbar_wait(&kv_full[j % NS], (j / NS) & 1);
        tc_fence_after();
        const uint64_t kdesc = T3<D>::desc(smem_u32(sK + (j % NS) * kKv64));
#pragma unroll
        for (int k = 0; k < D / 16; ++k)
          umma_f16_ss(tmem + k3ColS, qdesc + 2 * k, kdesc + 2 * k, idesc_s, k > 0 ? 1u : 0u);
        if constexpr (QKLO) {
          const uint64_t qldesc = T3<D>::desc(smem_u32(sQl));
          const uint64_t kldesc = T3<D>::desc(smem_u32(sKl + (j % NS) * kKv64));
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            umma_f16_ss(tmem + k3ColS, qldesc + 2 * k, kdesc + 2 * k, idesc_s, 1u);
            umma_f16_ss(tmem + k3ColS, qdesc + 2 * k, kldesc + 2 * k, idesc_s, 1u);
          }
        }
        umma_commit(s_full);
      };
      issue_s(0);
      if (tr) tr[2] = globaltimer();
      for (int j = 0; j < n_chunks; ++j) {
        mbar_wait(p_full, j & 1);  // P_j is in TMEM columns [0, 32)
        tc_fence_after();
        const uint8_t* vb = sV + (j % NS) * kKv64;
        const uint8_t* vbl = sVl + (j % NS) * kKv64;
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 16 keys per step: P columns 8k.. (2 fp16 each), V rows 16k..
          const uint64_t vdesc = T3<D>::desc(smem_u32(vb + k * 16 * D * 2));
          umma_f16_ts(tmem + k3ColO, tmem + k3ColS + 8 * k, vdesc, idesc_o, (j > 0 || k > 0) ? 1u : 0u);
          if constexpr (QLO) {  // P lo at columns 32 + 8k
            umma_f16_ts(tmem + k3ColO, tmem + k3ColS + 8 * k, T3<D>::desc(smem_u32(vbl + k * 16 * D * 2)), idesc_o, 1u);
            umma_f16_ts(tmem + k3ColO, tmem + k3ColS + 32 + 8 * k, vdesc, idesc_o, 1u);
          }
        }
        umma_commit(pv_done);
        umma_commit(&kv_empty[j % NS]);
        if (j + 1 < n_chunks) issue_s(j + 1);  // after PV_j in the tensor pipe: P_j is consumed first
      }
      if (tr) tr[4] = globaltimer();
    }
    __syncwarp();
  } else {
    const int row = warp * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    const bool live = q0 + warp * 32 < L;
    float m = 0.f, l = 0.f;
    for (int j = 0; j < n_chunks; ++j) {
      mbar_wait(s_full, j & 1);  // also: PV_{j-1} has completed (issued before S_j)
      if (tr && j == 0 && threadIdx.x == 0) tr[3] = globaltimer();
      if (!live) {
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        continue;
      }
      tc_fence_after();
      uint32_t r[2][32];
      tmem_ld32_nowait(tmem + lane_base + k3ColS, r[0]);
      tmem_ld32_nowait(tmem + lane_base + k3ColS + 32, r[1]);
      tmem_wait_ld();
      const int valid = L - j * 64;
      if (valid < 64) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (32 * c + i >= valid) r[c][i] = __float_as_uint(-INFINITY);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(r[c][i]));
      mx *= scale_log2;
      float alpha = 1.f;
      if (j == 0) {
        m = mx;
      } else if (mx > m + kRescaleLog2) {
        alpha = ex2(m - mx);
        m = mx;
        l *= alpha;
      }
      const float neg_m = -m;
      float ps = 0.f;
      if constexpr (QLO) {  // P = hi + lo: hi packed into columns [0, 32), lo into [32, 64), 8 at a time
#pragma unroll
        for (int g4 = 0; g4 < 4; ++g4) {
          uint32_t pk[8], pl[8];
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const int c = g4 >> 1, e = (g4 & 1) * 16 + i;
            const float p0 = ex2(fmaf(__uint_as_float(r[c][e]), scale_log2, neg_m));
            const float p1 = ex2(fmaf(__uint_as_float(r[c][e + 1]), scale_log2, neg_m));
            ps += p0 + p1;
            split_half2(p0, p1, pk[i >> 1], pl[i >> 1]);
          }
          tmem_st8(tmem + lane_base + k3ColS + 8 * g4, pk);
          tmem_st8(tmem + lane_base + k3ColS + 32 + 8 * g4, pl);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 2; ++c) {  // P over the (already read) scores, 16 packed columns at a time
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float p0 = ex2(fmaf(__uint_as_float(r[c][i]), scale_log2, neg_m));
            const float p1 = ex2(fmaf(__uint_as_float(r[c][i + 1]), scale_log2, neg_m));
            ps += p0 + p1;
            __half2 hp = __floats2half2_rn(p0, p1);
            pk[i >> 1] = *reinterpret_cast<uint32_t*>(&hp);
          }
          tmem_st16(tmem + lane_base + k3ColS + 16 * c, pk);
        }
      }
      l += ps;
      if (j >= 1 && __any_sync(0xffffffffu, alpha != 1.f)) {  // rare: rescale this warp's O rows
#pragma unroll
        for (int c = 0; c < D / 16; ++c) {
          uint32_t o[16];
          tmem_ld16_nowait(tmem + lane_base + k3ColO + 16 * c, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st16(tmem + lane_base + k3ColO + 16 * c, o);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(pv_done, (n_chunks - 1) & 1);
    if (tr && threadIdx.x == 0) tr[5] = globaltimer();
    if (live) {
      tc_fence_after();
      const float inv = 1.f / l;
      uint4* out = reinterpret_cast<uint4*>(ctx + (static_cast<long long>(row_base) + q0 + row) * hidden + h * D);
      uint4* out_lo = reinterpret_cast<uint4*>(ctx + lo_off + (static_cast<long long>(row_base) + q0 + row) * hidden +
                                               h * D);
#pragma unroll
      for (int c = 0; c < D / 16; ++c) {  // 16 output columns at a time
        uint32_t o[16];
        tmem_ld16_nowait(tmem + lane_base + k3ColO + 16 * c, o);
        tmem_wait_ld();
        if (q0 + row < L) {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            uint32_t w[4], l[4];  // (hi, lo) pair
#pragma unroll
            for (int i = 0; i < 4; ++i)
              split_half2(__uint_as_float(o[v * 8 + 2 * i]) * inv, __uint_as_float(o[v * 8 + 2 * i + 1]) * inv,
                          w[i], l[i]);
            out[2 * c + v] = make_uint4(w[0], w[1], w[2], w[3]);
            out_lo[2 * c + v] = make_uint4(l[0], l[1], l[2], l[3]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[7] = globaltimer();
  if (warp == kMma3) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

size_t attn_tc3_smem_bytes(int head_dim, bool qlo, bool qklo, int ns) {
  return 1024 + (size_t)(qklo ? 2 : 1) * 128 * head_dim * 2 +
         (qklo ? 4 : qlo ? 3 : 2) * (size_t)ns * 64 * head_dim * 2 + 128;
}

constexpr int kTc3OneStageFrom = 384;

template <int D, bool QLO, bool QKLO = false, int NS = 2>
static void launch_tc3_t(const CUtensorMap& map_q, const CUtensorMap& map_kv, half* ctx, long long lo_off,
                         const int* cu_seqlens, int n_seqs, int max_len, int groups, int n_heads, int hidden,
                         long long group_rows, long long lo_rows, cudaStream_t stream) {
  static bool attr_set = false;
  const size_t smem = attn_tc3_smem_bytes(D, QLO, QKLO, NS);
  if (!attr_set) {
    cudaFuncSetAttribute(attn_tc3_kernel<D, QLO, QKLO, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr_set = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  dim3 grid(groups * n_heads, n_seqs, (max_len + 127) / 128);
  unsigned long long* tr = trace_alloc_aux(static_cast<int>(grid.x * grid.y * grid.z), 2);
  launch_pdl(attn_tc3_kernel<D, QLO, QKLO, NS>, grid, dim3(kT3Threads), smem, stream, map_q, map_kv, ctx, cu_seqlens, n_heads,
             hidden, group_rows, scale_log2, lo_off, tr, lo_rows);
}

void launch_attention_tc3(const CUtensorMap& map_q, const CUtensorMap& map_kv, half* ctx, long long lo_off,
                          const int* cu_seqlens, int n_seqs, int max_len, int groups, int n_heads, int hidden,
                          long long group_rows, cudaStream_t stream, long long lo_rows, bool qk_lo) {
  if (n_seqs <= 0 || max_len <= 0 || groups <= 0) return;
  const bool d32 = hidden / n_heads == 32;
  static const int stages = [] {  // A/B: SP_TC3_STAGES=1|2 forces the K/V ring depth of the QKLO kernel
    const char* v = getenv("SP_TC3_STAGES");
    return v == nullptr ? 0 : atoi(v);
  }();
  // QKLO at two stages is 99 KiB (two CTAs per SM): above 384 tokens (four query tiles per head) a
  // one-stage ring keeps three CTAs per SM and one wave
  const bool one_stage = stages == 1 || (stages == 0 && max_len > kTc3OneStageFrom);
  if (lo_rows && qk_lo && one_stage) {
    if (d32) launch_tc3_t<32, true, true, 1>(map_q, map_kv, ctx, lo_off, cu_seqlens, n_seqs, max_len, groups, n_heads,
                                             hidden, group_rows, lo_rows, stream);
    else launch_tc3_t<64, true, true, 1>(map_q, map_kv, ctx, lo_off, cu_seqlens, n_seqs, max_len, groups, n_heads,
                                         hidden, group_rows, lo_rows, stream);
  } else if (lo_rows && qk_lo) {
    if (d32) launch_tc3_t<32, true, true>(map_q, map_kv, ctx, lo_off, cu_seqlens, n_seqs, max_len, groups, n_heads,
                                          hidden, group_rows, lo_rows, stream);
    else launch_tc3_t<64, true, true>(map_q, map_kv, ctx, lo_off, cu_seqlens, n_seqs, max_len, groups, n_heads, hidden,
                                      group_rows, lo_rows, stream);
  } else if (lo_rows) {
    if (d32) launch_tc3_t<32, true>(map_q, map_kv, ctx, lo_off, cu_seqlens, n_seqs, max_len, groups, n_heads, hidden,
                                    group_rows, lo_rows, stream);
    else launch_tc3_t<64, true>(map_q, map_kv, ctx, lo_off, cu_seqlens, n_seqs, max_len, groups, n_heads, hidden,
                                group_rows, lo_rows, stream);
  } else {
    if (d32) launch_tc3_t<32, false>(map_q, map_kv, ctx, lo_off, cu_seqlens, n_seqs, max_len, groups, n_heads, hidden,
                                     group_rows, 0, stream);
    else launch_tc3_t<64, false>(map_q, map_kv, ctx, lo_off, cu_seqlens, n_seqs, max_len, groups, n_heads, hidden,
                                 group_rows, 0, stream);
  }
}

}  // namespace sp
