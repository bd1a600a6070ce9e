// sp_stream.cu — weight streamer: keeps HBM busy across the batch-1 kernel chain.
//
// A short request is a chain of ~17 dependent kernels, and HBM idles between the projections
// (attention, LayerNorm, each GEMM's fill and drain): at L=16 the 236 MB of BERT-base K=8 weights
// stream at ~37% of the HBM roofline although each projection's main loop runs near peak. The
// weights do not depend on the activations, so a small kernel on a side branch of the request
// (forked stream / graph branch) pulls the upcoming projections' weights into L2 in consumption
// order with bulk L2 prefetches, while the chain runs; the projections then read them from L2.
//
// Pacing: the projections add the weight bytes they have requested to state[0] (GemmParams.progress);
// the streamer keeps at most `window` bytes ahead of that, so prefetched lines are not evicted before
// use (L2 126 MB). state[1] is the progress value at the start of the request (advanced by `total`
// by the last streamer CTA to finish; requests are stream-ordered), state[2] counts finished CTAs.
// A bounded wait (max_wait_ns) makes any accounting mismatch cost speed, never a hang.
//
// Grid: a few one-warp CTAs (co-resident with the chain's kernels: 32 threads, no shared memory).
#include "sp_kernels.cuh"
#include "sp_ptx.cuh"

namespace sp {

// Relaxed poll: the value is only a pacing hint. (An acquire load here waits for the thread's
// outstanding bulk prefetches: ~2 us per chunk, measured.)
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(32) weight_stream_kernel(const __grid_constant__ StreamPlan plan,
                                                           unsigned long long* state) {
  if (threadIdx.x != 0) return;
  const unsigned long long base = ld_relaxed_u64(state + 1);
  const unsigned long long chunk = plan.chunk;
  const unsigned int G = gridDim.x;
  unsigned long long seg_off = 0;  // offset of segment i in the request's consumption order
  unsigned int ci = 0;             // global index of the segment's first chunk (chunks dealt round-robin)
  const unsigned long long t_start = globaltimer();
  bool waiting = true;
  unsigned long long seen = base;
  for (int i = 0; i < plan.n; ++i) {
    const uint8_t* ptr = static_cast<const uint8_t*>(plan.ptr[i]);
    const unsigned long long bytes = plan.bytes[i];
    const unsigned int n_chunks = static_cast<unsigned int>((bytes + chunk - 1) / chunk);
    // this CTA's first chunk of the segment: global index = blockIdx.x (mod G)
    for (unsigned int j = (blockIdx.x + G - ci % G) % G; j < n_chunks; j += G) {
      const unsigned long long off = (unsigned long long)j * chunk;
      const unsigned long long o = seg_off + off;
      const unsigned long long len = bytes - off < chunk ? bytes - off : chunk;
      if (o + len <= plan.skip) continue;  // the chain's first projection loads these itself
      while (waiting && seen - base + plan.window < o + len) {  // re-read only while behind
        __nanosleep(200);
        seen = ld_relaxed_u64(state);
        if (globaltimer() - t_start > plan.max_wait_ns) waiting = false;
      }
      bulk_prefetch_l2(ptr + off, static_cast<uint32_t>(len));
    }
    ci += n_chunks;
    seg_off += bytes;
  }
  __threadfence();
  if (atomicAdd(reinterpret_cast<unsigned int*>(state + 2), 1u) == gridDim.x - 1) {
    state[1] = base + plan.total;
    reinterpret_cast<unsigned int*>(state + 2)[0] = 0u;
    __threadfence();
  }
}

void launch_weight_stream(const StreamPlan& plan, unsigned long long* state, int ctas, cudaStream_t stream) {
  prefer_max_smem(reinterpret_cast<const void*>(weight_stream_kernel));
  weight_stream_kernel<<<ctas, 32, 0, stream>>>(plan, state);
}

}  // namespace sp
