// sp_request.cu — a whole short request (<= 128 tokens) of the BERT student group in ONE
// persistent kernel: embedding + LN, every layer's QKV / attention / O + LN / FFN1 + GELU /
// FFN2 + LN, the pooler and the boosting-sum head (distill.py:169-178, :512).
//
// Why: at batch-1 the multi-kernel path is a chain of 17 dependent launches. Each projection
// refills its TMA ring from cold HBM only after its predecessor drains (2.5-4 us per launch) and,
// e.g., 192 FFN1 tiles do not divide over 148 SMs, so a 236 MB weight stream (BERT-base, K=8)
// reaches ~37% of HBM bandwidth at L=16. Here one CTA per SM runs every stage:
//   * warp 0 (weight producer) streams the weight k-blocks of every projection of every layer
//     through a TMA ring in one fixed order. Weights never depend on activations, so while
//     attention, LayerNorm and epilogues run the ring keeps filling with the next projection;
//   * warp 10 (activation producer) TMA-loads the token-side k-blocks of each item once their
//     producers published them (dataflow counters in global memory, acquire/release);
//   * warp 1 issues tcgen05.mma (swap-AB: 128 weight rows x T tokens, fp32 accumulators in TMEM,
//     two buffers so epilogue i overlaps MMA i+1);
//   * warps 2-9 (compute) run the epilogues (bias / erf-GELU / tanh), the embedding gather,
//     attention (mma.sync, K/V staged in smem) and the residual LayerNorms.
// Every projection is cut into chunks — a 128-feature tile times a 1/sp slice of its k-blocks —
// and each CTA takes a contiguous run of chunks, so all 148 SMs stream weights in every
// projection. QKV and FFN1 keep whole tiles (their bias / GELU epilogue needs the full sum); the
// O, FFN2 and pooler projections are split sp ways and their fp32 partial sums are added, in fixed
// order, by the stage that consumes them (LayerNorm rows, the head) — no cross-CTA fixups.
// A counter per (stage, student) replaces kernel boundaries: a student's next stage starts as soon
// as that student's inputs exist, with no grid-wide barrier.
//
// Counters live in one of two banks that alternate between consecutive requests (a device-side
// epoch picks the bank); each launch zeroes the other bank, which the previous request used.
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"
#include "sp_device.cuh"

namespace sp {

namespace {

constexpr int kRqWarps = 11;
constexpr int kRqThreads = 32 * kRqWarps;
constexpr int kRqComputeThreads = 256;  // warps 2..9
constexpr int kWBytes = 128 * 64 * 2;   // one weight k-block: 128 rows x 64 fp16
constexpr int kBarCompute = 1;          // named barrier of the compute warps
constexpr int kRqMaxStages = 16;
constexpr int kRqTmemCols = 256;        // two 128-column accumulators

enum { K_QKV = 0, K_O = 1, K_F1 = 2, K_F2 = 3, K_POOL = 4 };

struct RqPhase {
  int idx, kind, layer;
  int n_out, nkb, tps, sp, kpc, chunks, ncols, x_rows;
  const CUtensorMap *w, *x64, *x16;
};

// Split-K factor of a projection: whole tiles for QKV / FFN1 (bias + activation epilogue);
// otherwise the sp in 1..kReqMaxSplit dividing nkb that minimises the busiest CTA's k-blocks.
__device__ __forceinline__ int rq_split(int kind, int tiles, int nkb, int G) {
  if (kind == K_QKV || kind == K_F1) return 1;
  int best = 1, best_cost = 0x7fffffff;
  for (int s = 1; s <= kReqMaxSplit; ++s) {
    if (nkb % s) continue;
    const int cost = ((tiles * s + G - 1) / G) * (nkb / s);
    if (cost < best_cost) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

__device__ __forceinline__ RqPhase rq_phase(const ReqParams& p, const ReqMaps& m, int idx, int tpad, int ppad) {
  RqPhase f;
  f.idx = idx;
  if (idx < 4 * p.n_layers) {
    f.layer = idx >> 2;
    f.kind = idx & 3;
  } else {
    f.layer = p.n_layers - 1;
    f.kind = K_POOL;
  }
  const int H = p.hidden;
  f.nkb = H / 64;
  f.ncols = tpad;
  f.x_rows = p.t_cap;
  switch (f.kind) {
    case K_QKV:
      f.n_out = 3 * H;
      f.x64 = &m.x16_64;
      f.x16 = &m.x16_16;
      break;
    case K_O:
      f.n_out = H;
      f.x64 = &m.ctx_64;
      f.x16 = &m.ctx_16;
      break;
    case K_F1:
      f.n_out = p.ffn;
      f.x64 = &m.x16_64;
      f.x16 = &m.x16_16;
      break;
    case K_F2:
      f.n_out = H;
      f.nkb = p.ffn / 64;
      f.x64 = &m.ffn_64;
      f.x16 = &m.ffn_16;
      break;
    default:
      f.n_out = H;
      f.x64 = &m.cls_64;
      f.x16 = &m.cls_16;
      f.ncols = ppad;
      f.x_rows = p.b_cap;
      break;
  }
  f.w = f.kind == K_POOL ? &m.w_pool : &m.w[f.layer][f.kind];
  f.tps = f.n_out / 128;
  f.sp = rq_split(f.kind, p.k * f.tps, f.nkb, gridDim.x);
  f.kpc = f.nkb / f.sp;
  f.chunks = p.k * f.tps * f.sp;
  return f;
}

// CTA c owns chunks [lo(c), lo(c+1)), lo(c) = floor(c * chunks / G).
__device__ __forceinline__ int rq_lo(int n, int G, int c) { return (int)((long long)c * n / G); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Generic-proxy writes / reads vs the TMA (async proxy) reads of the same global memory.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Spin until *p >= target (acquire). Traps after ~4 s instead of hanging the GPU on a bug.
__device__ __forceinline__ void wait_ge(const int* p, int target) {
  if (ld_acquire(p) >= target) return;
  const long long t0 = clock64();
  while (ld_acquire(p) < target) {
    __nanosleep(32);
    if (clock64() - t0 > 8000000000LL) __trap();
  }
}

// Optional timeline (sp_debug_set_request_trace): 128 globaltimer stamps per CTA.
//   [64 + 5*phase + step]  ns spent by compute warp 0 in epilogue step (acc wait, TMEM->global,
//                  arrival sync, fixup sum, completion signal) of GEMM phase `phase`
//   [0]            kernel entry
//   [1 + stage]    compute warps leave stage (embed, then per layer QKV-epi, attention, O-epi,
//                  LN1, FFN1-epi, FFN2-epi, LN2; then pooler-epi, head)
//   [20 + phase]   activation producer: first dependency of GEMM phase `phase` satisfied
//   [40 + phase]   weight producer has issued every load of GEMM phase `phase`
//   [52 + phase]   MMA issuer: last accumulator of GEMM phase `phase` committed
__device__ __forceinline__ void rq_stamp(const ReqParams& p, int idx) {
  if (p.trace) p.trace[(size_t)blockIdx.x * 128 + idx] = globaltimer();
}

struct RqClock {
  const ReqParams* p;
  int base;
  unsigned long long t;
  bool on;
  __device__ void start(const ReqParams& pp, int phase, bool enable) {
    p = &pp;
    base = 64 + 5 * phase;
    on = enable && pp.trace != nullptr;
    if (on) t = globaltimer();
  }
  __device__ void lap(int step) {
    if (!on) return;
    const unsigned long long n = globaltimer();
    p->trace[(size_t)blockIdx.x * 128 + base + step] += n - t;
    t = n;
  }
};

// ------------------------------------------------------------------------------ row stages
// mode 0: embedding gather + LN (writes rows stage 0); mode 1: LN1 of layer l (after O);
// mode 2: LN2 of layer l (after FFN2; CLS rows copied on the last layer). Row r = (student, token)
// of the k*T rows; CTA c owns rows [c*R/G, (c+1)*R/G) in every row stage, warp-per-row.
template <int NC>
__device__ __noinline__ void rq_rows(const ReqParams& p, int mode, int l, int T, int sp, int* bank, int cw,
                                     int lane) {
  const int H = p.hidden;
  const int R = p.k * T;
  const int G = gridDim.x, c = blockIdx.x;
  const int lo = rq_lo(R, G, c), hi = rq_lo(R, G, c + 1);
  const int wait_phase = mode == 1 ? 4 * l + K_O : 4 * l + K_F2;
  const bool last_ln = mode == 2 && l == p.n_layers - 1;
  for (int r = lo + cw; r < hi; r += 8) {
    const int st = r / T, t = r - st * T;
    const long long row = ((long long)st * p.t_cap + t) * H;
    float v[NC][4];
    const float *gam, *bet;
    if (mode == 0) {
      const int id = __ldg(p.ids + t);
      const int b = seq_of(p.cu, p.n_seqs, t);
      const int ps = t - __ldg(p.cu + b);
      const half* wr = p.word + st * p.word_gs + (long long)id * H;
      const half* pr = p.pos + st * p.pos_gs + (long long)ps * H;
      const half* tr = p.type + (long long)st * H;
      uint2 wa[NC], pa[NC], ta[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const int f = q * 128 + lane * 4;
        wa[q] = __ldg(reinterpret_cast<const uint2*>(wr + f));
        pa[q] = __ldg(reinterpret_cast<const uint2*>(pr + f));
        ta[q] = __ldg(reinterpret_cast<const uint2*>(tr + f));
      }
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        float a[4], bb[4], cc[4];
        h4_to_f4(wa[q], a);
        h4_to_f4(pa[q], bb);
        h4_to_f4(ta[q], cc);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[q][j] = a[j] + bb[j] + cc[j];
      }
      gam = p.emb_g + (long long)st * H;
      bet = p.emb_b + (long long)st * H;
    } else {
      if (lane == 0) wait_ge(&bank[kReqOffDone + wait_phase * kReqMaxStudents + st], (H / 128) * sp);
      __syncwarp();
      const long long ls = (long long)l * p.s_total + st;
      const float* bias = (mode == 1 ? p.b_o : p.b_f2) + ls * H;
      gam = (mode == 1 ? p.ln1_g : p.ln2_g) + ls * H;
      bet = (mode == 1 ? p.ln1_b : p.ln2_b) + ls * H;
      float4 pr[kReqMaxSplit][NC], rs[NC], bs[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const int f = q * 128 + lane * 4;
        rs[q] = __ldcg(reinterpret_cast<const float4*>(p.x32 + row + f));
        bs[q] = __ldg(reinterpret_cast<const float4*>(bias + f));
#pragma unroll
        for (int k = 0; k < kReqMaxSplit; ++k)
          if (k < sp) pr[k][q] = __ldcg(reinterpret_cast<const float4*>(p.pre + k * p.part_ss + row + f));
      }
      // same association as reduce_ln_kernel: (residual + bias) + split partials in order
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        v[q][0] = rs[q].x + bs[q].x;
        v[q][1] = rs[q].y + bs[q].y;
        v[q][2] = rs[q].z + bs[q].z;
        v[q][3] = rs[q].w + bs[q].w;
#pragma unroll
        for (int k = 0; k < kReqMaxSplit; ++k)
          if (k < sp) {
            v[q][0] += pr[k][q].x;
            v[q][1] += pr[k][q].y;
            v[q][2] += pr[k][q].z;
            v[q][3] += pr[k][q].w;
          }
      }
    }
    half* cls_row = nullptr;
    if (last_ln) {
      const int b = seq_of(p.cu, p.n_seqs, t);
      if (__ldg(p.cu + b) == t) cls_row = p.cls16 + ((long long)st * p.b_cap + b) * H;
    }
    layer_norm_store<NC>(v, gam, bet, p.eps, H, p.x32 + row, p.x16 + row, cls_row);
  }
  fence_proxy_async_global();  // x16 / cls16 rows are read next by TMA
  named_barrier_sync(kBarCompute, kRqComputeThreads);
  if (cw == 0 && lane == 0 && hi > lo) {
    __threadfence();
    const int ridx = mode == 0 ? 0 : (mode == 1 ? 2 * l + 1 : 2 * l + 2);
    for (int st = lo / T; st <= (hi - 1) / T; ++st) {
      const int n = min(hi, (st + 1) * T) - max(lo, st * T);
      red_release_add(&bank[kReqOffRows + ridx * kReqMaxStudents + st], n);
    }
  }
}

// ------------------------------------------------------------------------------ attention
// One item = (student, head, sequence); L <= 128 keys. Eight warps of 16 query rows; K and V of
// the item staged in smem by cp.async; Q fragments loaded straight from global (L2).
template <int D>
__device__ __noinline__ void rq_attention(const ReqParams& p, int l, int* bank, half* sK, half* sV, int cw, int lane) {
  constexpr int LD = D + 8, VPR = D / 8;
  const int H = p.hidden, nh = p.n_heads;
  const int items = p.k * nh * p.n_seqs;
  const long long rs = 3LL * H;
  const int gr = lane >> 2, tq = lane & 3;
  const int ctid = cw * 32 + lane;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int st = it / (nh * p.n_seqs);
    const int rem = it - st * nh * p.n_seqs;
    const int h = rem / p.n_seqs, b = rem - (rem / p.n_seqs) * p.n_seqs;
    if (ctid == 0) wait_ge(&bank[kReqOffDone + (4 * l + K_QKV) * kReqMaxStudents + st], 3 * H / 128);
    named_barrier_sync(kBarCompute, kRqComputeThreads);
    const int s0 = __ldg(p.cu + b);
    const int L = __ldg(p.cu + b + 1) - s0;
    const half* base = p.qkv + ((long long)st * p.t_cap + s0) * rs + h * D;
    const int Lp = (L + 63) & ~63;
    for (int i = ctid; i < Lp * VPR; i += kRqComputeThreads) {
      const int r = i / VPR, c8 = (i - r * VPR) * 8;
      const bool ok = r < L;
      const half* rowp = base + (long long)(ok ? r : 0) * rs + c8;
      cp_async16(sK + r * LD + c8, rowp + H, ok ? 16u : 0u);
      cp_async16(sV + r * LD + c8, rowp + 2 * H, ok ? 16u : 0u);
    }
    cp_async_commit();
    cp_async_wait<0>();
    named_barrier_sync(kBarCompute, kRqComputeThreads);
    const int q0 = cw * 16;
    if (q0 < L) {
      // A fragments of Q (16 rows x D) straight from global: a0 = Q[g][2t..], a1 = Q[g+8][2t..],
      // a2 = Q[g][2t+8..], a3 = Q[g+8][2t+8..] per 16-wide k slice
      uint32_t qa[D / 16][4];
      const int r0 = q0 + gr, r1 = r0 + 8;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int cc = kk * 16 + 2 * tq;
        qa[kk][0] = r0 < L ? __ldcg(reinterpret_cast<const unsigned int*>(base + (long long)r0 * rs + cc)) : 0u;
        qa[kk][1] = r1 < L ? __ldcg(reinterpret_cast<const unsigned int*>(base + (long long)r1 * rs + cc)) : 0u;
        qa[kk][2] = r0 < L ? __ldcg(reinterpret_cast<const unsigned int*>(base + (long long)r0 * rs + cc + 8)) : 0u;
        qa[kk][3] = r1 < L ? __ldcg(reinterpret_cast<const unsigned int*>(base + (long long)r1 * rs + cc + 8)) : 0u;
      }
      float o[D / 8][4];
#pragma unroll
      for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      float m_run[2] = {-INFINITY, -INFINITY};
      float l_run[2] = {0.f, 0.f};
      for (int k0 = 0; k0 < Lp; k0 += 64) {
        const half* cK = sK + k0 * LD;
        const half* cV = sV + k0 * LD;
        float s[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
          for (int kk = 0; kk < D / 16; kk += 2) {
            uint32_t kf[4];
            const int r = nt * 8 + (lane & 7);
            const int c = kk * 16 + (lane >> 3) * 8;
            ldmatrix_x4(kf, cK + r * LD + c);
            mma_16816(s[nt], qa[kk], kf[0], kf[1]);
            if (kk + 1 < D / 16) mma_16816(s[nt], qa[kk + 1], kf[2], kf[3]);
          }
        }
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int key = k0 + nt * 8 + 2 * tq + (e & 1);
            float x = s[nt][e] * p.scale_log2;
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
        for (int nt = 0; nt < 8; ++nt) {
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
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
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
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 1);
        l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 2);
      }
      const float inv0 = 1.f / l_run[0], inv1 = 1.f / l_run[1];
      half* out = p.ctx + ((long long)st * p.t_cap + s0) * H + h * D;
#pragma unroll
      for (int dt = 0; dt < D / 8; ++dt) {
        const int c = dt * 8 + 2 * tq;
        if (r0 < L)
          *reinterpret_cast<__half2*>(out + (long long)r0 * H + c) = __floats2half2_rn(o[dt][0] * inv0, o[dt][1] * inv0);
        if (r1 < L)
          *reinterpret_cast<__half2*>(out + (long long)r1 * H + c) = __floats2half2_rn(o[dt][2] * inv1, o[dt][3] * inv1);
      }
    }
    fence_proxy_async_global();  // ctx is read next by TMA
    named_barrier_sync(kBarCompute, kRqComputeThreads);  // K/V smem free; all ctx rows stored
    if (ctid == 0) {
      __threadfence();
      red_release_add(&bank[kReqOffAtt + l * kReqMaxStudents + st], 1);
    }
  }
}

// ------------------------------------------------------------------------------ epilogues
// Where one chunk's outputs go (hoisted out of the per-element loops).
struct RqOut {
  void* base;         // element (col, feat) at base + col * col_stride + feat
  long long col_stride;
  const float* bias;  // [feat] or null
  int mode;           // 0: half(v + b)  1: half(gelu(v + b))  3: f32 raw partial
};

__device__ __forceinline__ RqOut rq_out(const ReqParams& p, const RqPhase& f, int st, int split) {
  const int H = p.hidden;
  const long long ls = (long long)f.layer * p.s_total + st;
  RqOut o;
  switch (f.kind) {
    case K_QKV:
      o = {p.qkv + (long long)st * p.t_cap * 3 * H, 3LL * H, p.b_qkv + ls * 3 * H, 0};
      break;
    case K_F1:
      o = {p.ffn_act + (long long)st * p.t_cap * p.ffn, (long long)p.ffn, p.b_f1 + ls * p.ffn, 1};
      break;
    case K_POOL:
      o = {p.pool_part + split * p.pool_ss + (long long)st * p.rows_cap * H, (long long)H, nullptr, 3};
      break;
    default:  // O, FFN2: raw split partial; bias + residual + LN happen in the row stage
      o = {p.pre + split * p.part_ss + (long long)st * p.t_cap * H, (long long)H, nullptr, 3};
      break;
  }
  return o;
}

__device__ __forceinline__ void rq_put(const RqOut& o, int col, int feat, float v, float bias) {
  const long long e = col * o.col_stride + feat;
  if (o.mode == 0) static_cast<half*>(o.base)[e] = __float2half_rn(v + bias);
  else if (o.mode == 1) static_cast<half*>(o.base)[e] = __float2half_rn(gelu_erf(v + bias));
  else static_cast<float*>(o.base)[e] = v;
}

__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Pooler finish (sum of the sp split partials + b_pool, tanh) + boosting sum in student order
// (distill.py:174-177) + shared classifier (+ bias once).
__device__ __noinline__ void rq_head(const ReqParams& p, int sp, int cw, int lane, float (*red)[4]) {
  const int ctid = cw * 32 + lane;
  const int H = p.hidden;
  for (int b = 0; b < p.n_seqs; ++b) {
    for (int c0 = 0; c0 < p.n_classes; c0 += 4) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j = ctid; j < H; j += kRqComputeThreads) {
        float r = 0.f;
        for (int s0 = 0; s0 < p.k; s0 += 8) {  // all loads of 8 students x sp splits in flight
          float v[8][kReqMaxSplit], bp[8], al[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const bool ok = s0 + i < p.k;
            const float* src = p.pool_part + ((long long)(s0 + i) * p.rows_cap + b) * H + j;
#pragma unroll
            for (int k = 0; k < kReqMaxSplit; ++k) v[i][k] = (ok && k < sp) ? __ldcg(src + k * p.pool_ss) : 0.f;
            bp[i] = ok ? __ldg(p.b_pool + (long long)(s0 + i) * H + j) : 0.f;
            al[i] = ok ? __ldg(p.alpha + s0 + i) : 0.f;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (s0 + i < p.k) {
              float t = v[i][0];
#pragma unroll
              for (int k = 1; k < kReqMaxSplit; ++k)
                if (k < sp) t += v[i][k];
              r += al[i] * tanhf(t + bp[i]);
            }
          }
        }
        if (p.rep && c0 == 0) p.rep[(long long)b * H + j] = r;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (c0 + q < p.n_classes) acc[q] += __ldg(p.w_cls + (long long)(c0 + q) * H + j) * r;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = warp_sum(acc[q]);
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < 4; ++q) red[cw][q] = acc[q];
      named_barrier_sync(kBarCompute, kRqComputeThreads);
      if (ctid < 4 && c0 + ctid < p.n_classes) {
        float z = 0.f;
        for (int w = 0; w < 8; ++w) z += red[w][ctid];
        if (p.add_bias) z += __ldg(p.b_cls + c0 + ctid);
        p.logits[(long long)b * p.n_classes + c0 + ctid] = z;
      }
      named_barrier_sync(kBarCompute, kRqComputeThreads);
    }
  }
}

// Publish `n` finished chunks of student st in phase f (and count pooler chunks toward the head).
// Returns 1 if this publication completed the pooler (this CTA runs the head).
__device__ __forceinline__ int rq_publish(const ReqParams& p, const RqPhase& f, int* bank, int st, int n,
                                          volatile int* bcast, int cw, int lane) {
  fence_proxy_async_global();  // outputs are read next by TMA (or by other CTAs' warps)
  named_barrier_sync(kBarCompute, kRqComputeThreads);
  if (cw == 0 && lane == 0) {
    int head = 0;
    if (f.kind == K_POOL) {
      const int old = atom_add_acq_rel(&bank[kReqOffPoolTotal], n);
      head = (old + n == f.chunks) ? 1 : 0;
    } else {
      red_release_add(&bank[kReqOffDone + f.idx * kReqMaxStudents + st], n);
    }
    *bcast = head;
  }
  named_barrier_sync(kBarCompute, kRqComputeThreads);
  return *bcast;
}

// The compute warps' epilogues of one projection: TMEM -> (bias / GELU) -> global per chunk, then
// one publication per student. Returns true if this CTA completed the pooler (the head runs
// here). One out-of-line copy serves every projection (a megakernel executes each stage once per
// request; inlined copies would run from a cold instruction cache every time).
__device__ __noinline__ bool rq_epilogues(const ReqParams& p, const RqPhase f, int T, int* bank, uint32_t tmem,
                                          uint64_t* acc_full, uint64_t* acc_empty, int* jp, volatile int* bcast,
                                          int cw, int lane) {
  const int G = gridDim.x, c = blockIdx.x;
  const int lo = rq_lo(f.chunks, G, c), hi = rq_lo(f.chunks, G, c + 1);
  const int q = (cw + 2) & 3;  // TMEM lane quadrant = warp id % 4
  const int half_cols = f.ncols >> 1;
  const int c_begin = (cw >> 2) * half_cols;
  const int live = f.kind == K_POOL ? p.n_seqs : T;
  int j = *jp;
  bool do_head = false;
  RqClock clk;
  clk.start(p, f.idx, cw == 0 && lane == 0);
  int pend_st = -1, pend_n = 0;
  for (int ch = lo; ch < hi; ++ch) {
    const int tile = ch / f.sp, split = ch - tile * f.sp;
    const int st = tile / f.tps, mt = tile - st * f.tps;
    if (st != pend_st && pend_n > 0) {
      do_head |= rq_publish(p, f, bank, pend_st, pend_n, bcast, cw, lane) != 0;
      pend_n = 0;
    }
    pend_st = st;
    const int feat = mt * 128 + q * 32 + lane;
    const RqOut o = rq_out(p, f, st, split);
    const float bias = o.bias ? __ldg(o.bias + feat) : 0.f;
    const int b = j & 1;
    mbar_wait(&acc_full[b], (j >> 1) & 1);
    tc_fence_after();
    clk.lap(0);
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * 128);
    for (int cc = c_begin; cc < c_begin + half_cols; cc += 8) {
      uint32_t r[8];
      tmem_ld8_nowait(taddr + cc, r);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (cc + e < live) rq_put(o, cc + e, feat, __uint_as_float(r[e]), bias);
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&acc_empty[b]);
    clk.lap(1);
    ++pend_n;
    ++j;
  }
  if (pend_n > 0) do_head |= rq_publish(p, f, bank, pend_st, pend_n, bcast, cw, lane) != 0;
  clk.lap(4);
  *jp = j;
  return do_head;
}

template <int NC, int D>
__global__ void __launch_bounds__(kRqThreads, 1)
    request_kernel(const __grid_constant__ ReqMaps m, const __grid_constant__ ReqParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int G = gridDim.x, c = blockIdx.x;
  const int warp = warp_id(), lane = lane_id();
  const int T = __ldg(p.cu + p.n_seqs);
  const int tpad = (T + 15) & ~15;
  const int ppad = (p.n_seqs + 15) & ~15;
  const int stage_bytes = kWBytes + tpad * 128;
  int stages = p.ring_bytes / stage_bytes;
  if (stages > kRqMaxStages) stages = kRqMaxStages;
  constexpr int LD = D + 8;
  half* sK = reinterpret_cast<half*>(smem + p.ring_bytes);
  half* sV = sK + 128 * LD;
  uint64_t* full = reinterpret_cast<uint64_t*>(sV + 128 * LD);
  uint64_t* empty = full + kRqMaxStages;
  uint64_t* acc_full = empty + kRqMaxStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  volatile int* bcast = reinterpret_cast<volatile int*>(tmem_slot + 1);
  float(*red)[4] = reinterpret_cast<float(*)[4]>(tmem_slot + 4);

  const int epoch = *reinterpret_cast<volatile const int*>(p.epoch);
  int* bank = p.banks + (epoch & 1) * kReqBankInts;
  {  // zero the bank the NEXT request will use (the previous request's; it has completed)
    int* other = p.banks + ((epoch & 1) ^ 1) * kReqBankInts;
    for (int i = c * kRqThreads + threadIdx.x; i < kReqBankInts; i += G * kRqThreads) other[i] = 0;
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kRqMaxStages; ++s) {
      mbar_init(&full[s], 2);  // weight producer + activation producer
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, kRqTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_phases = 4 * p.n_layers + 1;

  if (warp == 0) {
    // ---------------------------------------------------------------- weight producer
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();  // streamed once per request
      int s = 0;
      uint32_t ph = 0;
      for (int pi = 0; pi < n_phases; ++pi) {
        const RqPhase f = rq_phase(p, m, pi, tpad, ppad);
        const int lo = rq_lo(f.chunks, G, c), hi = rq_lo(f.chunks, G, c + 1);
        for (int ch = lo; ch < hi; ++ch) {
          const int tile = ch / f.sp, split = ch - tile * f.sp;
          const int st = tile / f.tps;
          const int w_row = st * f.n_out + (tile - st * f.tps) * 128;
          for (int kb = split * f.kpc; kb < (split + 1) * f.kpc; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], kWBytes);
            tma_load_2d(f.w, &full[s], smem + s * stage_bytes, kb * 64, w_row, pol);
            if (++s == stages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
        rq_stamp(p, 40 + pi);
      }
    }
  } else if (warp == kRqWarps - 1) {
    // ---------------------------------------------------------------- activation producer
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();  // re-read by every feature tile of the student
      int s = 0;
      uint32_t ph = 0;
      for (int pi = 0; pi < n_phases; ++pi) {
        const RqPhase f = rq_phase(p, m, pi, tpad, ppad);
        const int lo = rq_lo(f.chunks, G, c), hi = rq_lo(f.chunks, G, c + 1);
        const uint32_t x_bytes = (uint32_t)f.ncols * 128u;
        int dep_st = -1;
        for (int ch = lo; ch < hi; ++ch) {
          const int tile = ch / f.sp, split = ch - tile * f.sp;
          const int st = tile / f.tps;
          if (st != dep_st) {  // this student's input of the projection must be published
            const int* dep;
            int target;
            switch (f.kind) {
              case K_QKV:
                dep = &bank[kReqOffRows + (2 * f.layer) * kReqMaxStudents + st];
                target = T;
                break;
              case K_O:
                dep = &bank[kReqOffAtt + f.layer * kReqMaxStudents + st];
                target = p.n_heads * p.n_seqs;
                break;
              case K_F1:
                dep = &bank[kReqOffRows + (2 * f.layer + 1) * kReqMaxStudents + st];
                target = T;
                break;
              case K_F2:  // every FFN1 tile of the student (whole tiles, GELU applied)
                dep = &bank[kReqOffDone + (f.idx - 1) * kReqMaxStudents + st];
                target = p.ffn / 128;
                break;
              default:
                dep = &bank[kReqOffRows + (2 * p.n_layers) * kReqMaxStudents + st];
                target = T;
                break;
            }
            wait_ge(dep, target);
            fence_proxy_async_global();
            if (dep_st < 0) rq_stamp(p, 20 + pi);
            dep_st = st;
          }
          const int xrow = st * f.x_rows;
          for (int kb = split * f.kpc; kb < (split + 1) * f.kpc; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], x_bytes);
            uint8_t* sb = smem + s * stage_bytes + kWBytes;
            int r = 0;
            for (; r + 64 <= f.ncols; r += 64) tma_load_2d(f.x64, &full[s], sb + r * 128, kb * 64, xrow + r, pol);
            for (; r < f.ncols; r += 16) tma_load_2d(f.x16, &full[s], sb + r * 128, kb * 64, xrow + r, pol);
            if (++s == stages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      int j = 0;
      for (int pi = 0; pi < n_phases; ++pi) {
        const RqPhase f = rq_phase(p, m, pi, tpad, ppad);
        const uint32_t idesc = umma_idesc_f16(128, f.ncols);
        const int lo = rq_lo(f.chunks, G, c), hi = rq_lo(f.chunks, G, c + 1);
        for (int ch = lo; ch < hi; ++ch) {
          const int split = ch % f.sp;
          const int b = j & 1;
          mbar_wait(&acc_empty[b], ((j >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t acc = tmem + (uint32_t)(b * 128);
          for (int kk = 0; kk < f.kpc; ++kk) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + s * stage_bytes);
            const uint64_t adesc = umma_sdesc_sw128(sa);
            const uint64_t bdesc = umma_sdesc_sw128(sa + kWBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_f16_ss(acc, adesc + 2 * k, bdesc + 2 * k, idesc, (kk > 0 || k > 0) ? 1u : 0u);
            umma_commit(&empty[s]);
            if (++s == stages) {
              s = 0;
              ph ^= 1;
            }
          }
          (void)split;
          umma_commit(&acc_full[b]);
          ++j;
        }
        rq_stamp(p, 52 + pi);
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- compute warps
    const int cw = warp - 2;
    const bool stamp = cw == 0 && lane == 0;
    int j = 0;
    if (stamp) rq_stamp(p, 0);
    rq_rows<NC>(p, 0, 0, T, 1, bank, cw, lane);
    if (stamp) rq_stamp(p, 1);
    for (int l = 0; l < p.n_layers; ++l) {
      const int sb = 2 + 7 * l;
      rq_epilogues(p, rq_phase(p, m, 4 * l + K_QKV, tpad, ppad), T, bank, tmem, acc_full, acc_empty, &j, bcast, cw, lane);
      if (stamp) rq_stamp(p, sb + 0);
      rq_attention<D>(p, l, bank, sK, sV, cw, lane);
      if (stamp) rq_stamp(p, sb + 1);
      rq_epilogues(p, rq_phase(p, m, 4 * l + K_O, tpad, ppad), T, bank, tmem, acc_full, acc_empty, &j, bcast, cw, lane);
      if (stamp) rq_stamp(p, sb + 2);
      rq_rows<NC>(p, 1, l, T, rq_phase(p, m, 4 * l + K_O, tpad, ppad).sp, bank, cw, lane);
      if (stamp) rq_stamp(p, sb + 3);
      rq_epilogues(p, rq_phase(p, m, 4 * l + K_F1, tpad, ppad), T, bank, tmem, acc_full, acc_empty, &j, bcast, cw, lane);
      if (stamp) rq_stamp(p, sb + 4);
      rq_epilogues(p, rq_phase(p, m, 4 * l + K_F2, tpad, ppad), T, bank, tmem, acc_full, acc_empty, &j, bcast, cw, lane);
      if (stamp) rq_stamp(p, sb + 5);
      rq_rows<NC>(p, 2, l, T, rq_phase(p, m, 4 * l + K_F2, tpad, ppad).sp, bank, cw, lane);
      if (stamp) rq_stamp(p, sb + 6);
    }
    const RqPhase fp = rq_phase(p, m, 4 * p.n_layers, tpad, ppad);
    const bool head = rq_epilogues(p, fp, T, bank, tmem, acc_full, acc_empty, &j, bcast, cw, lane);
    if (stamp) rq_stamp(p, 2 + 7 * p.n_layers);
    if (head) rq_head(p, fp.sp, cw, lane, red);
    if (stamp) rq_stamp(p, 3 + 7 * p.n_layers);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kRqTmemCols);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const int old = atomicAdd(&bank[0], 1);
    if (old == G - 1) atomicExch(p.epoch, epoch + 1);  // every CTA has read this epoch
  }
}

template <int NC, int D>
bool launch_request_t(const ReqMaps& m, const ReqParams& p, int grid, cudaStream_t stream) {
  int ring = 0;
  const int smem = request_smem_bytes(D, &ring);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(request_kernel<NC, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  ReqParams q = p;
  q.ring_bytes = ring;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRqThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: they wait on each other
  attrs[0].val.cooperative = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  prefer_max_smem(reinterpret_cast<const void*>(request_kernel<NC, D>));
  return cudaLaunchKernelEx(&cfg, request_kernel<NC, D>, m, q) == cudaSuccess;
}

}  // namespace

static_assert(sizeof(ReqMaps) + sizeof(ReqParams) <= 4000, "kernel parameter space");

int request_smem_bytes(int head_dim, int* ring_bytes) {
  const int total = 227 * 1024;
  const int kv = 2 * 128 * (head_dim + 8) * 2;
  const int tail = (2 * kRqMaxStages + 4) * 8 + 16 + 8 * 4 * 4 + 64;
  const int ring = ((total - 1024 - kv - tail) / 1024) * 1024;
  if (ring_bytes) *ring_bytes = ring;
  return 1024 + ring + kv + tail;
}

bool launch_request(const ReqMaps& m, const ReqParams& p, int grid, cudaStream_t stream) {
  const int nc = p.hidden / 128, d = p.hidden / p.n_heads;
  if (nc == 6 && d == 64) return launch_request_t<6, 64>(m, p, grid, stream);
  if (nc == 8 && d == 64) return launch_request_t<8, 64>(m, p, grid, stream);
  if (nc == 1 && d == 32) return launch_request_t<1, 32>(m, p, grid, stream);
  if (nc == 2 && d == 64) return launch_request_t<2, 64>(m, p, grid, stream);
  return false;
}

}  // namespace sp
