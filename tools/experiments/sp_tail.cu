// sp_tail.cu — the last encoder layer on the CLS rows + pooler + boosting head, ONE launch.
//
// Only the CLS row of the last layer reaches the pooler, so after the last QKV
// projection a request of n_seqs <= kTailMaxRows sequences needs, per student, a chain of
// matrix-vector products on n_seqs rows: CLS-query attention, O (+ bias + residual, LayerNorm 1),
// FFN1 (+ GELU), FFN2 (+ bias + residual, LayerNorm 2), the tanh pooler — then the boosting sum
// over students and the classifier (distill.py:169-178, :512). As separate kernels these are
// eight dependent launches (~55 us at batch-1 for 94 MB of weights, 14.5 us of HBM time).
//
// Here each student is one thread-block CLUSTER of C CTAs (C = 16 for K <= 8 students: one
// cluster per GPC). CTA r of the cluster owns 1/C of every matrix's output rows; its weight rows
// are contiguous in HBM, so one producer warp streams the CTA's whole share of all four matrices
// (O, FFN1, FFN2, pooler: ~737 KB at H = 768) through a ring of 16 KiB 1-D bulk copies from the
// moment the CTA starts — weights never depend on activations, so the HBM stream runs through
// the dependency waits. Eight compute warps:
//   A  attention of the CLS query for the heads h = r, r + C, ... (fp32: scores, softmax, P V);
//   B  y1 = W_o ctx + b_o + x_CLS   (rows of this CTA), then LayerNorm 1 on the full vector;
//   C  f  = gelu(W_1 x1 + b_1);
//   D  y2 = W_2 f + b_2 + x1,       then LayerNorm 2;
//   E  p  = tanh(W_p x2 + b_p)  -> the student's pooled representation (global scratch).
// After each of A-D a CTA pushes its slice of the vector into every CTA of the cluster
// (st.shared::cluster) and arrives on their phase mbarrier (release, cluster scope); consumers wait
// on their local one (acquire), so a phase boundary is a DSMEM exchange, not a kernel boundary.
// The last CTA of the grid (atomic ticket) runs the head: rep = sum_m alpha_m p_m in student
// order, logits = W_c rep (+ b_c once).
//
// Every activation is fp32 and every product fp16 weight x fp32 activation accumulated in fp32:
// more precise than the tensor-core path (no operand rounding at all).
#include <algorithm>
#include <cstdlib>

#include "sp_kernels.cuh"
#include "sp_ptx.cuh"
#include "sp_device.cuh"

namespace sp {

__device__ unsigned long long* g_tail_trace_dev = nullptr;  // debug timeline (sp_debug_set_tail_trace)
__device__ int g_tail_skip_mma = 0;  // debug: consume the weight ring without computing (streaming-only timing)

namespace {

constexpr int kTailWarps = 8;                    // compute warps
constexpr int kTailThreads = 32 * (kTailWarps + 1);  // + one producer warp
constexpr int kTailStage = 16384;               // bytes per ring slot

__device__ __forceinline__ void bulk_load_1d(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  const long long t0 = clock64();
  while (!mbar_try_wait_cluster(addr, parity)) {
    if (clock64() - t0 > 8000000000LL) __trap();
  }
}

__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

__device__ __forceinline__ void fence_acq_rel_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }

// One matrix of the chain: this CTA's share (n_rows output rows) of a [out][k_in] matrix, repacked
// by tail_pack_weights into mma.sync m16n8k16 A-operand fragments: 16-row tiles, 16-column k-steps,
// per (tile, k-step) 32 lanes x 16 bytes in register order, so a lane's A fragment is ONE 16-byte
// shared load (no ldmatrix, no bank conflicts). Order: [tile group][k-step][tile][lane][8 halves];
// a tile group holds tg <= 32 tiles (16 KiB per k-step); a ring slot = kc k-steps of one group.
struct TailMat {
  const half* base;  // this CTA's share
  int n_rows, k_in, n_tiles, tg, n_tg, ks, kc, n_kc;
};

__device__ __host__ __forceinline__ void tail_geom(int n_rows, int k_in, int& tg, int& n_tg, int& kc, int& n_kc) {
  const int n_tiles = n_rows / 16;
  n_tg = (n_tiles + 31) / 32;
  while (n_tiles % n_tg) ++n_tg;
  tg = n_tiles / n_tg;
  const int ks = k_in / 16;
  kc = kTailStage / (tg * 512);
  if (kc < 1) kc = 1;
  if (kc > ks) kc = ks;
  n_kc = (ks + kc - 1) / kc;
}

__device__ __forceinline__ TailMat tail_mat(int mi, const TailParams& p, int g, int C, int rank) {
  const int H = p.hidden, F = p.ffn;
  const int out = mi == 1 ? F : H, k_in = mi == 2 ? F : H;
  const long long mat_off = mi == 0 ? 0 : (mi == 1 ? (long long)H * H : (mi == 2 ? (long long)H * H + (long long)F * H
                                                                                 : (long long)H * H + 2LL * F * H));
  TailMat m;
  m.n_rows = out / C;
  m.k_in = k_in;
  m.base = p.wt + (long long)g * (2LL * H * H + 2LL * F * H) + mat_off + (long long)rank * m.n_rows * k_in;
  m.n_tiles = m.n_rows / 16;
  m.ks = k_in / 16;
  tail_geom(m.n_rows, k_in, m.tg, m.n_tg, m.kc, m.n_kc);
  return m;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// One tile group of a matrix on the tensor cores (mma.sync m16n8k16, fp16 x fp16 -> fp32):
// D[16 rows][8] += A[16 rows][16 k] B[16 k][8], A = weight fragments from the ring, B = the input
// vector(s) as columns: n = 2 b is row b's fp16 hi term, n = 2 b + 1 its lo term (xs, [R][2][k_in]),
// so D[r][2b] + D[r][2b+1] = W x_b with ~22-bit operands and fp32 accumulation. Warp w takes the
// group's tiles w, w + 8, ... (TPW per warp). Returns in acc[t] the fragment of tile w + 8 t.
template <int TPW, int R>
__device__ __forceinline__ void tail_group(const TailMat& m, int gi, uint32_t xs_s, uint32_t ring_s, uint64_t* full,
                                           uint64_t* empty, int n_st, int& s, uint32_t& ph, float (&acc)[TPW][4],
                                           unsigned long long* wait_ns) {
  const int warp = warp_id(), lane = lane_id();
#pragma unroll
  for (int t = 0; t < TPW; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  const int n = lane >> 2;  // B column of this lane
  const bool bcol = n < 2 * R;
  const uint32_t xrow = xs_s + 2u * (uint32_t)((n >> 1) * 2 * m.k_in + (n & 1) * m.k_in) + 4u * (lane & 3);
  for (int c = 0; c < m.n_kc; ++c) {
    const int kb = c * m.kc, ke = min(kb + m.kc, m.ks);
    const unsigned long long t0 = wait_ns ? globaltimer() : 0ull;
    mbar_wait(&full[s], ph);
    if (wait_ns) *wait_ns += globaltimer() - t0;
    const uint32_t slot = ring_s + (uint32_t)(s * kTailStage) + 16u * lane;
#pragma unroll 2
    for (int k = kb; k < (g_tail_skip_mma ? kb : ke); ++k) {
      const uint32_t b0 = bcol ? lds32(xrow + 32u * k) : 0u;
      const uint32_t b1 = bcol ? lds32(xrow + 32u * k + 16u) : 0u;
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const int tile = warp + kTailWarps * t;
        if (tile < m.tg) {
          const uint4 a = lds128(slot + 512u * (uint32_t)((k - kb) * m.tg + tile));
          asm volatile(
              "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
              "{%0,%1,%2,%3};"
              : "+f"(acc[t][0]), "+f"(acc[t][1]), "+f"(acc[t][2]), "+f"(acc[t][3])
              : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == n_st) {
      s = 0;
      ph ^= 1;
    }
  }
}

// Compute warps of the CTA (256 threads) synchronise among themselves (named barrier 1).
__device__ __forceinline__ void compute_sync() { named_barrier_sync(1, 32 * kTailWarps); }

// LayerNorm of R rows of `hidden` floats in place (one warp per row; fp32 statistics).
__device__ __forceinline__ void tail_layer_norm(float* v, int R, int hidden, const float* gamma, const float* beta,
                                                float eps) {
  const int warp = warp_id(), lane = lane_id();
  for (int b = warp; b < R; b += kTailWarps) {
    float* x = v + (long long)b * hidden;
    float s = 0.f;
    for (int j = lane; j < hidden; j += 32) s += x[j];
    const float mean = warp_sum(s) / hidden;
    float q = 0.f;
    for (int j = lane; j < hidden; j += 32) {
      const float d = x[j] - mean;
      q += d * d;
    }
    const float rstd = rsqrtf(warp_sum(q) / hidden + eps);
    for (int j = lane; j < hidden; j += 32) x[j] = (x[j] - mean) * rstd * __ldg(gamma + j) + __ldg(beta + j);
  }
}

}  // namespace

template <int R>
__global__ void __launch_bounds__(kTailThreads, 1) tail_kernel(const TailParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int H = p.hidden, F = p.ffn;
  const int n_st = p.stages;
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + n_st * kTailStage);
  uint64_t* empty = full + n_st;
  uint64_t* ph_bar = empty + n_st;  // [4] phases A..D
  int* flag = reinterpret_cast<int*>(ph_bar + 4);
  float* ctx = reinterpret_cast<float*>(flag + 4);  // [R][H]
  float* y1 = ctx + R * H;                          // [R][H]  -> x1 after LayerNorm 1
  float* fv = y1 + R * H;                           // [R][F]
  float* y2 = fv + R * F;                           // [R][H]  -> x2 after LayerNorm 2
  float* sc = y2 + R * H;                           // [2][max_len] attention scores (two head groups)
  float* red = sc + 2 * p.max_len;                  // 2 x ([4][64] PV partials + [16] statistics)
  float* ebias = red + 2 * (kTailWarps / 2 * 64 + 16);  // this CTA's bias slices: O | FFN1 | FFN2 | pooler

  const int C = p.cluster;
  const int rank = (int)cluster_ctarank();
  const int g = blockIdx.x / C;  // student
  const int warp = warp_id(), lane = lane_id();
  const int n_o = H / C, n_1 = F / C;
  float* res = ebias + 3 * n_o + n_1;  // [R][n_o] residual slice (the CLS rows of the layer input)
  half* xs = reinterpret_cast<half*>(res + R * n_o);  // [R][2][k_in] the GEMV input as (hi, lo) fp16

  unsigned long long* tr = g_tail_trace_dev ? g_tail_trace_dev + 16ull * blockIdx.x : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  if (threadIdx.x == 0) {
    for (int s = 0; s < n_st; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTailWarps);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&ph_bar[i], C);
    fence_barrier_init();
  }
  __syncthreads();
  cluster_sync();  // every CTA's barriers initialised before any remote arrive
  pdl_launch_dependents();

  if (warp == kTailWarps) {
    // ------------------------------------------------------------ weight producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int mi = 0; mi < 4; ++mi) {
        const TailMat m = tail_mat(mi, p, g, C, rank);
        for (int gi = 0; gi < m.n_tg; ++gi)
          for (int c = 0; c < m.n_kc; ++c) {
            const int kw = min(m.kc, m.ks - c * m.kc);
            const uint32_t bytes = (uint32_t)(kw * m.tg * 512);
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], bytes);
            bulk_load_1d(ring + s * kTailStage,
                         m.base + ((long long)gi * m.ks + (long long)c * m.kc) * m.tg * 256, bytes, &full[s], pol);
            if (++s == n_st) {
              s = 0;
              ph ^= 1;
            }
          }
        if (tr) tr[10 + mi] = globaltimer();  // last chunk of matrix mi issued
      }
    }
  } else {
    // ------------------------------------------------------------ compute warps
    const int tid = threadIdx.x;  // 0..255
    const int n_rows = p.n_seqs;  // == R
    for (int i = tid; i < 3 * n_o + n_1; i += 32 * kTailWarps) {  // weights: before the dependency wait
      const int seg = i < n_o ? 0 : (i < n_o + n_1 ? 1 : (i < 2 * n_o + n_1 ? 2 : 3));
      const int off = seg == 0 ? i : (seg == 1 ? i - n_o : (seg == 2 ? i - n_o - n_1 : i - 2 * n_o - n_1));
      const float* bsrc = seg == 0 ? p.b_o + (long long)g * H + rank * n_o
                                   : (seg == 1 ? p.b_1 + (long long)g * F + rank * n_1
                                               : (seg == 2 ? p.b_2 + (long long)g * H + rank * n_o
                                                           : p.b_p + (long long)g * H + rank * n_o));
      ebias[i] = __ldg(bsrc + off);
    }
    pdl_wait();                   // qkv and the residual stream come from the previous kernels
    if (tr && tid == 0) tr[1] = globaltimer();
    for (int i = tid; i < R * n_o; i += 32 * kTailWarps) {
      const int b = i / n_o, j = i - b * n_o;
      res[i] = p.x32[(long long)g * p.x_gs + (long long)__ldg(p.cu + b) * H + rank * n_o + j];
    }

    // push this CTA's slice [j0, j0 + n) of every row of vector v (row stride ld) to every CTA,
    // then arrive on their phase barrier
    auto publish = [&](float* v, int ld, int j0, int n, int phase) {
      compute_sync();
      const int v4 = n / 4;
      for (int i = tid; i < (C - 1) * R * v4; i += 32 * kTailWarps) {
        const int q = i / (R * v4);
        const int rem = i - q * (R * v4);
        const int b = rem / v4, e = rem - b * v4;
        const int dst = (rank + 1 + q) % C;
        float* src = v + (long long)b * ld + j0 + 4 * e;
        st_cluster_v4(mapa_shared(smem_u32(src), dst), *reinterpret_cast<const float4*>(src));
      }
      compute_sync();
      if (tid == 0) {
        fence_acq_rel_cluster();
        for (int q = 0; q < C; ++q) mbar_arrive_cluster(mapa_shared(smem_u32(&ph_bar[phase]), q));
      }
      mbar_wait_cluster(&ph_bar[phase], 0);
    };

    // ---- A: attention of the CLS query, heads h = rank, rank + C, ...: units (row, head) dealt to
    // two groups of four warps (named barriers 2 and 3), so two heads' global-load round trips
    // overlap. Scores in fp32, exact exp, P V over fp16 V rows.
    const int D = H / p.n_heads;
    const float scale = rsqrtf((float)D);
    const long long row3 = 3LL * H;
    {
      constexpr int kGW = kTailWarps / 2;  // warps per group
      const int grp = warp / kGW, gt = tid - grp * 32 * kGW, gw = warp - grp * kGW;
      float* gsc = sc + grp * p.max_len;
      float* gred = red + grp * (kGW * 64 + 16);
      int n_mine = 0;
      for (int h = rank; h < p.n_heads; h += C) ++n_mine;
      for (int u = grp; u < n_mine * R; u += 2) {
        const int b = u / n_mine, h = rank + (u % n_mine) * C;
        const int c0 = __ldg(p.cu + b), L = __ldg(p.cu + b + 1) - c0;
        const half* base = p.qkv + (long long)g * p.qkv_gs + (long long)c0 * row3 + h * D;
        float mx = -INFINITY;
        for (int j = gt; j < L; j += 32 * kGW) {
          const half* kr = base + (long long)j * row3 + H;
          float sco = 0.f;
          for (int v = 0; v < D; v += 8) {
            const uint4 qu = *reinterpret_cast<const uint4*>(base + v);
            const uint4 ku = *reinterpret_cast<const uint4*>(kr + v);
            const __half2* qh = reinterpret_cast<const __half2*>(&qu);
            const __half2* kh = reinterpret_cast<const __half2*>(&ku);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float2 a2 = __half22float2(qh[t]), k2 = __half22float2(kh[t]);
              sco = fmaf(a2.x, k2.x, sco);
              sco = fmaf(a2.y, k2.y, sco);
            }
          }
          sco *= scale;
          gsc[j] = sco;
          mx = fmaxf(mx, sco);
        }
        mx = warp_max(mx);
        if (lane == 0) gred[kGW * 64 + gw] = mx;
        named_barrier_sync(2 + grp, 32 * kGW);
        mx = gred[kGW * 64];
        for (int w = 1; w < kGW; ++w) mx = fmaxf(mx, gred[kGW * 64 + w]);
        float sum = 0.f;
        for (int j = gt; j < L; j += 32 * kGW) {
          const float e = __expf(gsc[j] - mx);
          gsc[j] = e;
          sum += e;
        }
        sum = warp_sum(sum);
        named_barrier_sync(2 + grp, 32 * kGW);  // max slots read; gsc complete
        if (lane == 0) gred[kGW * 64 + 8 + gw] = sum;
        // P V: warp gw takes keys gw, gw + 4, ...; lane owns dims lane and lane + 32 (D <= 64)
        float a0 = 0.f, a1 = 0.f;
        const half* vb = base + 2 * H;
        for (int j = gw; j < L; j += kGW) {
          const float pj = gsc[j];
          const half* vr = vb + (long long)j * row3;
          a0 = fmaf(pj, __half2float(vr[lane]), a0);
          if (D > 32) a1 = fmaf(pj, __half2float(vr[lane + 32]), a1);
        }
        gred[gw * 64 + lane] = a0;
        if (D > 32) gred[gw * 64 + lane + 32] = a1;
        named_barrier_sync(2 + grp, 32 * kGW);
        if (gt < D) {
          float tot = 0.f, o = 0.f;
          for (int w = 0; w < kGW; ++w) tot += gred[kGW * 64 + 8 + w];
          for (int w = 0; w < kGW; ++w) o += gred[w * 64 + gt];
          ctx[(long long)b * H + h * D + gt] = o / tot;
        }
        named_barrier_sync(2 + grp, 32 * kGW);  // gred / gsc reused by the group's next unit
      }
    }
    // every CTA's heads into every CTA (the heads of this CTA: one D-wide slice each)
    compute_sync();
    {
      const int v4 = D / 4;
      int n_mine = 0;
      for (int h = rank; h < p.n_heads; h += C) ++n_mine;
      for (int i = tid; i < (C - 1) * R * n_mine * v4; i += 32 * kTailWarps) {
        int t = i;
        const int e = t % v4;
        t /= v4;
        const int hh = t % n_mine;
        t /= n_mine;
        const int b = t % R;
        const int q = t / R;
        const int dst = (rank + 1 + q) % C;
        float* src = ctx + (long long)b * H + (rank + hh * C) * D + 4 * e;
        st_cluster_v4(mapa_shared(smem_u32(src), dst), *reinterpret_cast<const float4*>(src));
      }
      compute_sync();
      if (tid == 0) {
        fence_acq_rel_cluster();
        for (int q = 0; q < C; ++q) mbar_arrive_cluster(mapa_shared(smem_u32(&ph_bar[0]), q));
      }
      mbar_wait_cluster(&ph_bar[0], 0);
    }
    if (tr && tid == 0) tr[2] = globaltimer();

    // ---- B..E: matrix-vector products from the weight ring (tensor cores, mma.sync)
    int s = 0;
    uint32_t ph = 0;
#pragma unroll 1
    for (int mi = 0; mi < 4; ++mi) {
      const TailMat m = tail_mat(mi, p, g, C, rank);
      const float* vin = mi == 0 ? ctx : (mi == 1 ? y1 : (mi == 2 ? fv : y2));
      const float* eb = ebias + (mi == 0 ? 0 : (mi == 1 ? n_o : (mi == 2 ? n_o + n_1 : 2 * n_o + n_1)));
      const int j0 = rank * m.n_rows;  // first output feature of this CTA
      // the input vector(s) as fp16 (hi, lo) pairs: xs[b][0][k] = hi, xs[b][1][k] = lo
      for (int u = tid; u < R * m.k_in / 2; u += 32 * kTailWarps) {
        const int b = (2 * u) / m.k_in, k = 2 * u - b * m.k_in;
        uint32_t hi, lo;
        split_half2(vin[(long long)b * m.k_in + k], vin[(long long)b * m.k_in + k + 1], hi, lo);
        reinterpret_cast<uint32_t*>(xs + (long long)(2 * b) * m.k_in + k)[0] = hi;
        reinterpret_cast<uint32_t*>(xs + (long long)(2 * b + 1) * m.k_in + k)[0] = lo;
      }
      compute_sync();
      unsigned long long wsum = 0;
      unsigned long long* wns = (tr && tid == 0) ? &wsum : nullptr;  // trace: warp 0's waits on the ring
      const uint32_t xs_s = smem_u32(xs), ring_s = smem_u32(ring);
      const int tpw = (m.tg + kTailWarps - 1) / kTailWarps;
      for (int gi = 0; gi < m.n_tg; ++gi) {
        float accv[4][4];
        if (tpw <= 1) {
          float a1[1][4];
          tail_group<1, R>(m, gi, xs_s, ring_s, full, empty, n_st, s, ph, a1, wns);
#pragma unroll
          for (int e = 0; e < 4; ++e) accv[0][e] = a1[0][e];
        } else if (tpw == 2) {
          float a2[2][4];
          tail_group<2, R>(m, gi, xs_s, ring_s, full, empty, n_st, s, ph, a2, wns);
#pragma unroll
          for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) accv[t][e] = a2[t][e];
        } else if (tpw == 3) {
          float a3[3][4];
          tail_group<3, R>(m, gi, xs_s, ring_s, full, empty, n_st, s, ph, a3, wns);
#pragma unroll
          for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) accv[t][e] = a3[t][e];
        } else {
          tail_group<4, R>(m, gi, xs_s, ring_s, full, empty, n_st, s, ph, accv, wns);
        }
        // epilogue: lane with lane % 4 == b holds row b's (hi, lo) columns for rows lane / 4 and + 8
        const int b = lane & 3;
        if (b < n_rows) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int tile = warp + kTailWarps * t;
            if (t < tpw && tile < m.tg) {
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {
                const int i = (gi * m.tg + tile) * 16 + (lane >> 2) + 8 * hf;  // row of the CTA's share
                const int j = j0 + i;
                const float z = accv[t][2 * hf] + accv[t][2 * hf + 1] + eb[i];
                if (mi == 0) {  // O + bias + residual (the CLS token row of the layer input)
                  y1[(long long)b * H + j] = z + res[b * n_o + i];
                } else if (mi == 1) {
                  fv[(long long)b * F + j] = gelu_erf_exact(z);
                } else if (mi == 2) {
                  y2[(long long)b * H + j] = z + y1[(long long)b * H + j];
                } else {
                  const float pv = tanhf(z);
                  p.pooled[((long long)g * R + b) * H + j] = pv;
                  if (p.finals) p.finals[((long long)g * n_rows + b) * H + j] = pv;
                }
              }
            }
          }
        }
      }
      compute_sync();  // every row of the matrix written before the exchange
      if (tr && tid == 0) {
        tr[3 + mi] = globaltimer();  // matrix mi done (before its exchange)
        tr[14 + (mi & 1)] += wsum;   // ns warp 0 waited for weight chunks: [14] O + FFN2, [15] FFN1 + pooler
      }
      if (mi == 0) {
        publish(y1, H, j0, m.n_rows, 1);
        tail_layer_norm(y1, R, H, p.g1 + (long long)g * H, p.be1 + (long long)g * H, p.eps);
        compute_sync();
      } else if (mi == 1) {
        publish(fv, F, j0, m.n_rows, 2);
      } else if (mi == 2) {
        publish(y2, H, j0, m.n_rows, 3);
        tail_layer_norm(y2, R, H, p.g2 + (long long)g * H, p.be2 + (long long)g * H, p.eps);
        compute_sync();
      }
    }

    if (tr && tid == 0) tr[7] = globaltimer();
    // ---- head: the last CTA of the grid sums the students in order and applies the classifier
    __threadfence();
    compute_sync();
    if (tid == 0) flag[0] = (atomicAdd(p.counter, 1) == (int)gridDim.x - 1);
    compute_sync();
    if (flag[0]) {
      __threadfence();
      float* rep = ctx;  // reuse: [R][H]
      for (int i = tid; i < n_rows * H; i += 32 * kTailWarps) {
        const int b = i / H, j = i - b * H;
        float r = 0.f;
        for (int m = 0; m < p.groups; ++m)  // student order (distill.py:174-177)
          r += __ldg(p.alpha + m) * __ldcg(p.pooled + ((long long)m * R + b) * H + j);
        rep[i] = r;
        if (p.rep) p.rep[(long long)b * H + j] = r;
      }
      compute_sync();
      for (int b = 0; b < n_rows; ++b)
        for (int c = warp; c < p.n_classes; c += kTailWarps) {
          float z = 0.f;
          for (int j = lane; j < H; j += 32) z += __ldg(p.w_cls + (long long)c * H + j) * rep[(long long)b * H + j];
          z = warp_sum(z);
          if (lane == 0) {
            if (p.add_bias) z += __ldg(p.b_cls + c);
            p.logits[(long long)b * p.n_classes + c] = z;
          }
        }
      compute_sync();
      if (tid == 0) {
        *p.counter = 0;  // for the next launch
        if (p.ready_flag != nullptr) {  // batch-1 host path: logits in mapped memory, then the flag
          __threadfence_system();
          *reinterpret_cast<volatile int*>(p.ready_flag) = __ldg(p.seq_src);
        }
      }
    }
  }
  __syncwarp();
  cluster_sync();  // no CTA leaves while a peer may still write into its shared memory
  if (tr && threadIdx.x == 0) tr[8] = globaltimer();
}

// Shared memory besides the weight ring (vectors, scores, partials, bias / residual slices).
static size_t tail_fixed_bytes(int hidden, int ffn, int rows, int max_len) {
  return 1024 + 64 * 8 + 16 +
         sizeof(float) * ((size_t)rows * (3 * hidden + ffn) + 2 * max_len + kTailWarps * 64 + 32 + 3 * hidden + ffn +
                          (size_t)rows * hidden) +
         sizeof(half) * (size_t)rows * 2 * std::max(hidden, ffn) + 16;
}

int tail_stages(int hidden, int ffn, int rows, int max_len) {
  const size_t budget = 227 * 1024 - tail_fixed_bytes(hidden, ffn, rows, max_len);
  static const int cap = getenv("SP_TAIL_STAGES") ? atoi(getenv("SP_TAIL_STAGES")) : 8;  // probe only
  return std::max(2, std::min(cap, (int)(budget / kTailStage)));
}

size_t tail_smem_bytes(int hidden, int ffn, int rows, int max_len) {
  return tail_fixed_bytes(hidden, ffn, rows, max_len) + (size_t)tail_stages(hidden, ffn, rows, max_len) * kTailStage;
}

// Cluster size: the largest C in {16, 8, 4, 2, 1} that divides H and F, and with which the GPU can
// hold every student's cluster at once (cudaOccupancyMaxActiveClusters), else with the most CTAs.
int tail_cluster_size(int groups, int hidden, int ffn, int rows, int max_len) {
  const size_t smem = tail_smem_bytes(hidden, ffn, rows, max_len);
  int best = 1;
  if (hidden % kTailWarps || ffn % kTailWarps) return 1;
  for (int C : {16, 8, 4, 2}) {
    if (hidden % (16 * C) || ffn % (16 * C)) continue;  // 16-row mma tiles per CTA
    void (*fn)(TailParams) = rows == 1 ? tail_kernel<1> : tail_kernel<2>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (C > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(groups * C);
    cfg.blockDim = dim3(kTailThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (n >= groups) return C;
    if (n > 0 && best == 1) best = C;  // fallback: several waves of clusters
  }
  return best;
}

// Transposed per-CTA slices of the last layer's O, FFN1, FFN2 and pooler matrices (see TailMat):
// wt[g] = [O | FFN1 | FFN2 | pooler], each = C slices of n = out / C rows, each slice = row blocks
// of rb rows stored [k_in][rb]. One-time at group creation (a plain elementwise gather).
__global__ void tail_pack_kernel(const half* __restrict__ w_o, const half* __restrict__ w_1,
                                 const half* __restrict__ w_2, const half* __restrict__ w_p, half* __restrict__ wt,
                                 int S, int H, int F, int C) {
  const long long per_student = 2LL * H * H + 2LL * F * H;
  const long long total = (long long)S * per_student;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(idx / per_student);
    long long e = idx - (long long)g * per_student;
    int mi = 0;
    const long long sizes[4] = {(long long)H * H, (long long)F * H, (long long)H * F, (long long)H * H};
    while (e >= sizes[mi]) e -= sizes[mi++];
    const int out = mi == 1 ? F : H, k_in = mi == 2 ? F : H;
    const int n = out / C;
    int tg, n_tg, kc, n_kc;
    tail_geom(n, k_in, tg, n_tg, kc, n_kc);
    const int ks = k_in / 16;
    const long long slice = (long long)n * k_in;
    const int rank = (int)(e / slice);
    long long r2 = e - (long long)rank * slice;
    const long long per_group = (long long)ks * tg * 256;
    const int gi = (int)(r2 / per_group);
    r2 -= (long long)gi * per_group;
    const int k = (int)(r2 / (tg * 256));
    r2 -= (long long)k * tg * 256;
    const int tile = (int)(r2 / 256);
    r2 -= (long long)tile * 256;
    const int lane = (int)(r2 / 8), el = (int)(r2 % 8);
    // m16n8k16 A fragment (row-major): a0 = (r, c), a1 = (r + 8, c), a2 = (r, c + 8), a3 = (r + 8, c + 8),
    // r = lane / 4, c = 2 (lane % 4) + {0, 1}
    const int reg = el >> 1;
    const int row = (lane >> 2) + ((reg & 1) ? 8 : 0);
    const int col = 2 * (lane & 3) + (el & 1) + ((reg & 2) ? 8 : 0);
    const long long src_row = (long long)rank * n + (long long)(gi * tg + tile) * 16 + row;
    const half* src = mi == 0 ? w_o : (mi == 1 ? w_1 : (mi == 2 ? w_2 : w_p));
    wt[idx] = src[(long long)g * out * k_in + src_row * k_in + (long long)k * 16 + col];
  }
}

void tail_pack_weights(const half* w_o, const half* w_1, const half* w_2, const half* w_p, half* wt, int S, int H,
                       int F, int C, cudaStream_t stream) {
  tail_pack_kernel<<<1184, 256, 0, stream>>>(w_o, w_1, w_2, w_p, wt, S, H, F, C);
}

void set_tail_trace(unsigned long long* buf) {
  cudaMemcpyToSymbol(g_tail_trace_dev, &buf, sizeof(buf));
  int skip = (getenv("SP_TAIL_SKIP_MMA") != nullptr);  // debug probe only (tools/trace_tail.py)
  cudaMemcpyToSymbol(g_tail_skip_mma, &skip, sizeof(skip));
}

bool launch_tail(const TailParams& p0, cudaStream_t stream) {
  if (p0.n_seqs < 1 || p0.n_seqs > kTailMaxRows) return false;
  TailParams p = p0;
  const int C = p.cluster;
  const size_t smem = tail_smem_bytes(p.hidden, p.ffn, p.n_seqs, p.max_len);
  void (*fn)(TailParams) = p.n_seqs == 1 ? tail_kernel<1> : tail_kernel<2>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (C > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.groups * C);
  cfg.blockDim = dim3(kTailThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = C;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, fn, p) == cudaSuccess;
}

}  // namespace sp
