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

namespace sp {

static constexpr int kTileBytes = 128 * 64 * 2;  // 128 rows x 64 fp16 = 16 KiB
static constexpr int kMaxChunks = 4;

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__global__ void __launch_bounds__(160, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap map_qkv, half* __restrict__ ctx, const int* __restrict__ cu,
                   int n_heads, int hidden, long long group_rows, float scale_log2, int max_chunks) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kTileBytes;
  uint8_t* sV = sK + max_chunks * kTileBytes;
  uint8_t* sP = sV + max_chunks * kTileBytes;  // two 64-key halves of the 128 x 128 P tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * kTileBytes);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;  // [kMaxChunks]
  uint64_t* s_full = kv_full + kMaxChunks;
  uint64_t* s_free = s_full + 1;
  uint64_t* p_full = s_free + 1;
  uint64_t* pv_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);

  pdl_wait();
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

  if (warp == 4 && lane == 0) {
    mbar_init(q_full, 1);
    for (int j = 0; j < kMaxChunks; ++j) mbar_init(&kv_full[j], 1);
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);
    mbar_init(p_full, 4);
    mbar_init(pv_done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&map_qkv);
  }
  if (warp == 4) {
    tmem_alloc(tmem_slot, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t S_t = tmem;        // columns [0, 128): scores of the current chunk
  const uint32_t O_t = tmem + 128;  // columns [128, 192): output accumulator

  if (warp == 4) {
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();
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
      int use = 0;
      auto issue_s = [&](int j) {
        mbar_wait(&kv_full[j], 0);
        if (use > 0) mbar_wait(s_free, (use - 1) & 1);  // softmax finished reading the previous S
        tc_fence_after();
        const uint64_t kdesc = umma_sdesc_sw128(smem_u32(sK + j * kTileBytes));
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_f16_ss(S_t, qdesc + 2 * k, kdesc + 2 * k, idesc_s, k > 0 ? 1u : 0u);
        umma_commit(s_full);
        ++use;
      };
      for (int j = 0; j < n_chunks; ++j) issue_s(j);  // pass 1: row maxima
      for (int j = 0; j < n_chunks; ++j) {            // pass 2: P V
        issue_s(j);
        mbar_wait(p_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // 16 keys per step: P half k/4 (+32 B per step), V 2 x 8-key atoms
          const uint64_t pdesc = umma_sdesc_sw128(smem_u32(sP + (k >> 2) * kTileBytes)) + 2 * (k & 3);
          const uint64_t vdesc = umma_sdesc_sw128(smem_u32(sV + j * kTileBytes + k * 2048));
          umma_f16_ss(O_t, pdesc, vdesc, idesc_o, (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(pv_done);
      }
    }
    __syncwarp();
  } else {
    // softmax: thread t owns query row t (TMEM lane t)
    const int t = threadIdx.x;
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    float m = -INFINITY;
    int use = 0;
    for (int j = 0; j < n_chunks; ++j) {
      mbar_wait(s_full, use & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32_nowait(S_t + lane_base + c * 32, r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int key = j * 128 + c * 32 + i;
          if (key < L) m = fmaxf(m, __uint_as_float(r[i]) * scale_log2);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);
      ++use;
    }
    float l = 0.f;
    const uint32_t prow = static_cast<uint32_t>((t >> 3) * 1024 + (t & 7) * 128);
    for (int j = 0; j < n_chunks; ++j) {
      mbar_wait(s_full, use & 1);
      tc_fence_after();
      if (j > 0) mbar_wait(pv_done, (j - 1) & 1);  // the previous P V consumed the P buffer
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32_nowait(S_t + lane_base + c * 32, r);
        tmem_wait_ld();
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const int key = j * 128 + c * 32 + i;
          const float p0 = key < L ? exp2f(__uint_as_float(r[i]) * scale_log2 - m) : 0.f;
          const float p1 = key + 1 < L ? exp2f(__uint_as_float(r[i + 1]) * scale_log2 - m) : 0.f;
          l += p0 + p1;
          __half2 hp = __floats2half2_rn(p0, p1);
          packed[i >> 1] = *reinterpret_cast<uint32_t*>(&hp);
        }
        // keys c*32 .. c*32+31 -> half c/2, 16-byte chunks (c&1)*4 .. +3, XOR-swizzled by row
        uint8_t* half_base = sP + (c >> 1) * kTileBytes + prow;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = ((c & 1) * 4 + q) ^ (t & 7);
          *reinterpret_cast<uint4*>(half_base + chunk * 16) =
              make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();  // P written through the generic proxy, read by the tensor core
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(s_free);
        mbar_arrive(p_full);
      }
      ++use;
    }
    // epilogue: O row t / l -> fp16 -> ctx
    mbar_wait(pv_done, (n_chunks - 1) & 1);
    tc_fence_after();
    uint32_t o0[32], o1[32];
    tmem_ld32_nowait(O_t + lane_base, o0);
    tmem_ld32_nowait(O_t + lane_base + 32, o1);
    tmem_wait_ld();
    if (q0 + t < L) {
      const float inv = 1.f / l;
      half* out = ctx + (static_cast<long long>(row_base) + q0 + t) * hidden + h * 64;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t* src = q < 4 ? o0 + q * 8 : o1 + (q - 4) * 8;
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __half2 hv = __floats2half2_rn(__uint_as_float(src[2 * i]) * inv, __uint_as_float(src[2 * i + 1]) * inv);
          w[i] = *reinterpret_cast<uint32_t*>(&hv);
        }
        *reinterpret_cast<uint4*>(out + q * 8) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

size_t attn_tc_smem_bytes(int max_len) {
  const int chunks = (max_len + 127) / 128;
  return 1024 + kTileBytes * (1 + 2 * chunks + 2) + 128;
}

void launch_attention_tc(const CUtensorMap& map_qkv, half* ctx, const int* cu_seqlens, int n_seqs, int max_len,
                         int groups, int n_heads, int hidden, long long group_rows, cudaStream_t stream) {
  if (n_seqs <= 0 || max_len <= 0 || groups <= 0) return;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  const int chunks = (max_len + 127) / 128;
  const float scale_log2 = 1.4426950408889634f / 8.0f;  // log2(e) / sqrt(64)
  dim3 grid((max_len + 127) / 128, n_seqs, groups * n_heads);
  launch_pdl(attn_tc_kernel, grid, dim3(160), attn_tc_smem_bytes(max_len), stream, map_qkv, ctx, cu_seqlens, n_heads,
             hidden, group_rows, scale_log2, chunks);
}

}  // namespace sp
