// stream_probe.cu — HBM weight-streaming ceiling for the batch-1 projection shapes.
//
// Streams a [rows, cols] fp16 weight matrix into shared memory the way the projection GEMMs do
// (16 KiB stages through an mbarrier ring, no MMA) and reports GB/s per launch (L2 flushed before
// every launch). Block b = (m-tile, k-block) in m-major order; the blocks are dealt to CTAs in
// contiguous, equal ranges (stream-K style), so the CTA count is free.
//   mode 0: 2-D TMA box {64 cols x 128 rows}, 128-B swizzle, row-major [rows, cols] (today's layout)
//   mode 1: 1-D cp.async.bulk of 16 KiB contiguous blocks (pre-tiled layout: block b at b * 16 KiB)
//   mode 2: 2-D TMA, but CTA c owns whole m-tiles over full K (today's one-tile-per-CTA split)
//   mode 3: bulk L2 prefetch (cp.async.bulk.prefetch.L2) of the CTA's range in chunks of
//           stages x 16 KiB, no smem; mode 4: mode 3 then a mode-1 read of the same bytes (two
//           launches, timed together); mode 5: 2-D tensor L2 prefetch of each block
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/stream_probe.cu -lcuda -o /tmp/sp
//   /tmp/sp <rows> <cols> <ctas> <stages> <mode> [reps]
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);      \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void load2d(const CUtensorMap* m, uint64_t* b, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(m), "r"(su32(b)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void load1d(const void* src, uint64_t* b, void* dst, uint32_t bytes) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b))
               : "memory");
}

constexpr int kStage = 16384;

__global__ void stream_kernel(const __grid_constant__ CUtensorMap map, const uint8_t* tiled, int m_tiles, int kbs,
                              int stages, int mode, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  uint64_t* full = (uint64_t*)(smem + stages * kStage);
  if (threadIdx.x != 0) return;
  if (mode == 3 || mode == 5) {
    const long long nb = (long long)m_tiles * kbs;
    const long long q0 = nb * blockIdx.x / gridDim.x, q1 = nb * (blockIdx.x + 1) / gridDim.x;
    if (mode == 5) {
      for (long long b = q0; b < q1; ++b)
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(&map),
                     "r"((int)(b % kbs) * 64), "r"((int)(b / kbs) * 128) : "memory");
      return;
    }
    const long long step = stages;
    for (long long b = q0; b < q1; b += step) {
      const long long n = (q1 - b < step ? q1 - b : step) * kStage;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tiled + b * kStage), "r"((uint32_t)n) : "memory");
    }
    return;
  }
  for (int s = 0; s < stages; ++s) bar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long long nblocks = (long long)m_tiles * kbs;
  long long b0, b1;
  if (mode == 2) {  // whole m-tiles per CTA, round-robin
    b0 = 0;
    b1 = 0;
  } else {
    b0 = nblocks * blockIdx.x / gridDim.x;
    b1 = nblocks * (blockIdx.x + 1) / gridDim.x;
  }
  auto issue = [&](int s, long long b) {
    bar_expect(&full[s], kStage);
    const int mt = (int)(b / kbs), kb = (int)(b % kbs);
    if (mode == 1) load1d(tiled + b * kStage, &full[s], smem + s * kStage, kStage);
    else load2d(&map, &full[s], smem + s * kStage, kb * 64, mt * 128);
  };
  // block sequence
  long long cnt = 0;
  auto nth = [&](long long i) -> long long {
    if (mode != 2) return b0 + i;
    const long long tile = blockIdx.x + (i / kbs) * gridDim.x;
    return tile * kbs + i % kbs;
  };
  long long total = (mode == 2) ? (long long)((m_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * kbs : b1 - b0;
  if (mode == 2 && (int)blockIdx.x >= m_tiles) total = 0;
  int s = 0;
  uint32_t ph = 0;
  for (; cnt < total && cnt < stages; ++cnt) issue((int)cnt, nth(cnt));
  unsigned long long acc = 0;
  for (long long i = 0; i < total; ++i) {
    bar_wait(&full[s], ph);
    acc += smem[s * kStage + (i & 1023)];
    if (cnt < total) {
      issue(s, nth(cnt));
      ++cnt;
    }
    if (++s == stages) {
      s = 0;
      ph ^= 1;
    }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

// read the flush buffer after writing it: L2 ends holding CLEAN lines (a write-only flush leaves
// ~126 MB of dirty lines whose write-back then competes with the measured stream)
__global__ void read_kernel(const float4* p, long long n, float* sink) {
  float a = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = p[i];
    a += v.x + v.y + v.z + v.w;
  }
  if (a == 1234.5f) *sink = a;
}

int main(int argc, char** argv) {
  if (argc < 6) {
    std::printf("usage: %s rows cols ctas stages mode [reps]\n", argv[0]);
    return 1;
  }
  const long long rows = atoll(argv[1]), cols = atoll(argv[2]);
  const int ctas = atoi(argv[3]), stages = atoi(argv[4]), mode = atoi(argv[5]);
  const int reps = argc > 6 ? atoi(argv[6]) : 20;
  const size_t bytes = rows * cols * 2;
  void *w, *flush, *sink;
  CK(cudaMalloc(&w, bytes));
  CK(cudaMemset(w, 1, bytes));
  CK(cudaMalloc(&flush, 256ull << 20));
  CK(cudaMalloc(&sink, 64));
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  if (cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    std::printf("encode failed\n");
    return 1;
  }
  const int smem = (mode >= 3 ? 6 : stages) * kStage + 1024 + 8 * stages + 64;
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int r = 0; r < reps + 2; ++r) {
    CK(cudaMemsetAsync(flush, r, 256ull << 20));
    if (!getenv("DIRTY_FLUSH")) read_kernel<<<148 * 4, 256>>>((const float4*)flush, (256ll << 20) / 16, (float*)sink);
    cudaEventRecord(e0);
    stream_kernel<<<ctas, 32, smem>>>(map, (const uint8_t*)w, (int)(rows / 128), (int)(cols / 64), stages,
                                      mode == 4 ? 3 : mode, (unsigned long long*)sink);
    if (mode == 4)
      stream_kernel<<<148, 32, 6 * kStage + 2048>>>(map, (const uint8_t*)w, (int)(rows / 128), (int)(cols / 64), 6, 1,
                                                  (unsigned long long*)sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2) ts.push_back(ms);
  }
  CK(cudaGetLastError());
  std::sort(ts.begin(), ts.end());
  const float med = ts[ts.size() / 2];
  std::printf("rows=%lld cols=%lld MB=%.1f ctas=%d stages=%d mode=%d  median %.2f us  %.0f GB/s  (min %.2f us)\n",
              rows, cols, bytes / 1e6, ctas, stages, mode, med * 1e3, bytes / (med * 1e-3) / 1e9, ts[0] * 1e3);
  return 0;
}
