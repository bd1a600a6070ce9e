// sp_attn_tc.cu — unpadded varlen attention on 5th-gen tensor cores (head_dim 64, L <= 512).
//
// One CTA per (student, sequence, head, 128-query block). Q, K and V tiles of the packed
// sequence are TMA-loaded (128-byte swizzle) straight from the qkv projection output and stay
// resident in shared memory (L <= 512 -> at most four 128-key chunks).
//
//   pass 1: S = Q K^T per 128-key chunk (tcgen05.mma M=128 N=128 K=64, S in TMEM); each of the
//           128 softmax threads owns one query row = one TMEM lane and keeps its running max.
//   pass 2: S is recomputed, P = exp2(S*scale - max) is written as fp16 into shared memory in the
//           UMMA K-major swizzled layout, row sums accumulate in fp32, and O += P V runs on the
//           tensor core (V is the MN-major B operand) with O in TMEM.
// With the exact row max known before any exponential, O never needs rescaling and every score
// costs one exp2. Keys past the sequence end are masked; query rows past it are not stored.
//
// Warp roles (160 threads): warps 0-3 softmax/epilogue (warp w = TMEM lanes 32w..32w+31),
// warp 4 TMEM allocation + TMA + MMA issue (one elected lane).
// No reference counterpart; semantics = oracle/bert.py:attention.
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"
#include "sp_device.cuh"

namespace sp {

static constexpr int kTileBytes = 128 * 64 * 2;  // 128 rows x 64 fp16 = 16 KiB
static constexpr int kMaxChunks = 4;

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 16 softmax warps (4 per TMEM lane quadrant, each owning 32 of a chunk's 128 key columns) + one
// control warp (TMEM allocation, TMA, MMA issue). S is double-buffered in TMEM so the MMA of chunk
// j+1 overlaps the softmax of chunk j; P is double-buffered in smem.
constexpr int kTcSoftWarps = 16;
constexpr int kTcThreads = 32 * (kTcSoftWarps + 1);

__device__ __forceinline__ float tc_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(kTcThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap map_qkv, half* __restrict__ ctx, const int* __restrict__ cu,
                   int n_heads, int hidden, long long group_rows, float scale_log2, int max_chunks, long long lo_off) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kTileBytes;
  uint8_t* sV = sK + max_chunks * kTileBytes;
  uint8_t* sP = sV + max_chunks * kTileBytes;  // [2 buffers][2 halves of 64 keys] x 16 KiB
  float* red = reinterpret_cast<float*>(sP + 4 * kTileBytes);  // [128 rows][4 column quarters]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 128 * 4);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;          // [kMaxChunks]
  uint64_t* s_full = kv_full + kMaxChunks;  // [2]
  uint64_t* s_free = s_full + 2;            // [2]
  uint64_t* p_full = s_free + 2;            // [2]
  uint64_t* pv_done = p_full + 2;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  pdl_launch_dependents();
  const int b = blockIdx.y;
  const int s0 = __ldg(cu + b);
  const int L = __ldg(cu + b + 1) - s0;
  const int q0 = blockIdx.x * 128;
  if (q0 >= L) return;
  const int g = blockIdx.z / n_heads;
  const int h = blockIdx.z % n_heads;
  const int n_chunks = (L + 127) >> 7;
  const int row_base = static_cast<int>(g * group_rows + s0);
  const int warp = warp_id();
  const int lane = lane_id();
  constexpr int kCtl = kTcSoftWarps;  // control warp

  if (warp == kCtl && lane == 0) {
    mbar_init(q_full, 1);
    for (int j = 0; j < kMaxChunks; ++j) mbar_init(&kv_full[j], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], kTcSoftWarps);
      mbar_init(&p_full[i], kTcSoftWarps);
      mbar_init(&pv_done[i], 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&map_qkv);
  }
  if (warp == kCtl) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t O_t = tmem + 256;  // S buffers at columns [0, 128) and [128, 256)

  if (warp == kCtl) {
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();
      pdl_wait();  // qkv is the previous kernel's output
      mbar_arrive_expect_tx(q_full, kTileBytes);
      tma_load_2d(&map_qkv, q_full, sQ, h * 64, row_base + q0, pol);
      for (int j = 0; j < n_chunks; ++j) {
        mbar_arrive_expect_tx(&kv_full[j], 2 * kTileBytes);
        tma_load_2d(&map_qkv, &kv_full[j], sK + j * kTileBytes, hidden + h * 64, row_base + j * 128, pol);
        tma_load_2d(&map_qkv, &kv_full[j], sV + j * kTileBytes, 2 * hidden + h * 64, row_base + j * 128, pol);
      }
      const uint32_t idesc_s = umma_idesc_f16(128, 128);
      const uint32_t idesc_o = umma_idesc_f16(128, 64) | (1u << 16);  // B (= V) is MN-major
      const uint64_t qdesc = umma_sdesc_sw128(smem_u32(sQ));
      mbar_wait(q_full, 0);
      int u = 0;  // S buffer uses
      auto issue_s = [&](int j) {
        const int sb = u & 1;
        if (u >= 2) mbar_wait(&s_free[sb], ((u >> 1) - 1) & 1);  // softmax released this buffer
        mbar_wait(&kv_full[j], 0);
        tc_fence_after();
        const uint64_t kdesc = umma_sdesc_sw128(smem_u32(sK + j * kTileBytes));
        const uint32_t S_t = tmem + static_cast<uint32_t>(sb * 128);
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_f16_ss(S_t, qdesc + 2 * k, kdesc + 2 * k, idesc_s, k > 0 ? 1u : 0u);
        umma_commit(&s_full[sb]);
        ++u;
      };
      for (int j = 0; j < n_chunks; ++j) issue_s(j);  // pass 1: row maxima
      issue_s(0);                                     // pass 2: P = exp2(S - m), O += P V
      for (int j = 0; j < n_chunks; ++j) {
        if (j + 1 < n_chunks) issue_s(j + 1);  // next scores while the softmax works on chunk j
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        uint8_t* pb = sP + (j & 1) * 2 * kTileBytes;
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 16 keys per step: P half k/4 (+32 B per step), V 2 x 8-key atoms
          const uint64_t pdesc = umma_sdesc_sw128(smem_u32(pb + (k >> 2) * kTileBytes)) + 2 * (k & 3);
          const uint64_t vdesc = umma_sdesc_sw128(smem_u32(sV + j * kTileBytes + k * 2048));
          umma_f16_ss(O_t, pdesc, vdesc, idesc_o, (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&pv_done[j & 1]);
      }
    }
    __syncwarp();
  } else {
    // softmax warp w: TMEM lanes 32*(w%4).. (query rows), key columns 32*(w/4).. of each chunk
    const int quad = warp & 3, wq = warp >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const int named = 1, nthr = 32 * kTcSoftWarps;
    int u = 0;
    float m = -INFINITY;
    for (int j = 0; j < n_chunks; ++j) {  // pass 1: partial row max over this warp's columns
      const int sb = u & 1;
      mbar_wait(&s_full[sb], (u >> 1) & 1);
      tc_fence_after();
      uint32_t r[32];
      tmem_ld32_nowait(tmem + static_cast<uint32_t>(sb * 128 + wq * 32) + lane_base, r);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[sb]);
      ++u;
      float v[32];
      const int key0 = j * 128 + wq * 32;
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = key0 + i < L ? __uint_as_float(r[i]) : -INFINITY;
#pragma unroll
      for (int w = 16; w > 0; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) v[i] = fmaxf(v[i], v[i + w]);
      m = fmaxf(m, v[0]);
    }
    red[row * 4 + wq] = m;
    named_barrier_sync(named, nthr);
    m = fmaxf(fmaxf(red[row * 4 + 0], red[row * 4 + 1]), fmaxf(red[row * 4 + 2], red[row * 4 + 3]));
    const float neg_m = -m * scale_log2;
    named_barrier_sync(named, nthr);  // red is reused for the row sums
    float l = 0.f;
    const uint32_t prow = static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128);
    for (int j = 0; j < n_chunks; ++j) {  // pass 2
      const int sb = u & 1;
      mbar_wait(&s_full[sb], (u >> 1) & 1);
      tc_fence_after();
      uint32_t r[32];
      tmem_ld32_nowait(tmem + static_cast<uint32_t>(sb * 128 + wq * 32) + lane_base, r);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[sb]);
      ++u;
      if (j >= 2) mbar_wait(&pv_done[j & 1], ((j >> 1) - 1) & 1);  // P buffer j&1 consumed by P V (j-2)
      const int key0 = j * 128 + wq * 32;
      float p[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) p[i] = key0 + i < L ? tc_exp2(fmaf(__uint_as_float(r[i]), scale_log2, neg_m)) : 0.f;
      float ps[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) ps[i] = p[2 * i] + p[2 * i + 1];
#pragma unroll
      for (int w = 8; w > 0; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) ps[i] += ps[i + w];
      l += ps[0];
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        __half2 hp = __floats2half2_rn(p[2 * i], p[2 * i + 1]);
        packed[i] = *reinterpret_cast<uint32_t*>(&hp);
      }
      // keys wq*32 .. +31 of the chunk -> half wq/2, 16-byte chunks (wq&1)*4 .. +3, XOR-swizzled by row
      uint8_t* half_base = sP + (j & 1) * 2 * kTileBytes + (wq >> 1) * kTileBytes + prow;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int chunk = ((wq & 1) * 4 + q) ^ (row & 7);
        *reinterpret_cast<uint4*>(half_base + chunk * 16) =
            make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
      }
      fence_proxy_async_smem();  // P written through the generic proxy, read by the tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[j & 1]);
    }
    red[row * 4 + wq] = l;
    named_barrier_sync(named, nthr);
    l = (red[row * 4 + 0] + red[row * 4 + 1]) + (red[row * 4 + 2] + red[row * 4 + 3]);
    // epilogue: O[row][wq*16 .. +15] / l -> fp16 -> ctx
    mbar_wait(&pv_done[(n_chunks - 1) & 1], ((n_chunks - 1) >> 1) & 1);
    tc_fence_after();
    uint32_t o[16];
    tmem_ld8_nowait(O_t + lane_base + static_cast<uint32_t>(wq * 16), o);
    tmem_ld8_nowait(O_t + lane_base + static_cast<uint32_t>(wq * 16 + 8), o + 8);
    tmem_wait_ld();
    if (q0 + row < L) {
      const float inv = 1.f / l;
      half* out = ctx + (static_cast<long long>(row_base) + q0 + row) * hidden + h * 64 + wq * 16;
      uint32_t w8[8], l8[8];  // (hi, lo) pair, lo at out + lo_off
#pragma unroll
      for (int i = 0; i < 8; ++i)
        split_half2(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv, w8[i], l8[i]);
      *reinterpret_cast<uint4*>(out) = make_uint4(w8[0], w8[1], w8[2], w8[3]);
      *reinterpret_cast<uint4*>(out + 8) = make_uint4(w8[4], w8[5], w8[6], w8[7]);
      *reinterpret_cast<uint4*>(out + lo_off) = make_uint4(l8[0], l8[1], l8[2], l8[3]);
      *reinterpret_cast<uint4*>(out + lo_off + 8) = make_uint4(l8[4], l8[5], l8[6], l8[7]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kCtl) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

size_t attn_tc_smem_bytes(int max_len) {
  const int chunks = (max_len + 127) / 128;
  return 1024 + kTileBytes * (1 + 2 * chunks + 4) + 128 * 4 * 4 + 256;
}

void launch_attention_tc(const CUtensorMap& map_qkv, half* ctx, long long lo_off, const int* cu_seqlens, int n_seqs,
                         int max_len, int groups, int n_heads, int hidden, long long group_rows, cudaStream_t stream) {
  if (n_seqs <= 0 || max_len <= 0 || groups <= 0) return;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  const int chunks = (max_len + 127) / 128;
  const float scale_log2 = 1.4426950408889634f / 8.0f;  // log2(e) / sqrt(64)
  dim3 grid((max_len + 127) / 128, n_seqs, groups * n_heads);
  launch_pdl(attn_tc_kernel, grid, dim3(kTcThreads), attn_tc_smem_bytes(max_len), stream, map_qkv, ctx, cu_seqlens, n_heads,
             hidden, group_rows, scale_log2, chunks, lo_off);
}

}  // namespace sp
