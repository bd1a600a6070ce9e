// mc_probe.cu — does TMA multicast within a cluster raise the operand bandwidth L2 can deliver?
//
// Every CTA streams, per k-block, a 16 KiB tile of its own (the weight slab of a projection CTA)
// and a shared 256-row x 64-col (32 KiB) tile (the token tile all m-tile CTAs of a student read).
//   mode 0: every CTA loads the shared tile itself (unicast, today's persistent GEMM)
//   mode 1: cluster of C CTAs; CTA r loads rows [r*256/C, (r+1)*256/C) and multicasts them to all
// A stage is refilled only once every CTA of the cluster released it (remote mbarrier arrives).
// Reports the operand bytes delivered into shared memory per second (chip-wide).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/mc_probe.cu -lcuda -o /tmp/mc
//   /tmp/mc <mode> <cluster> [kblocks]
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                   \
    }                                                                                 \
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
__device__ __forceinline__ void bar_arrive_remote(uint64_t* local_bar, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(local_bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void load2d(const CUtensorMap* m, uint64_t* b, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(m), "r"(su32(b)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void load2d_mc(const CUtensorMap* m, uint64_t* b, void* dst, int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(su32(dst)),
      "l"(m), "r"(su32(b)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int kW = 16384, kX = 32768, kStages = 4;

__global__ void mc_kernel(const __grid_constant__ CUtensorMap mw, const __grid_constant__ CUtensorMap mx, int kblocks,
                          int mode, int csz, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  uint64_t* full = (uint64_t*)(smem + kStages * (kW + kX));
  uint64_t* empty = full + kStages;
  const uint32_t rank = mode == 1 ? cluster_rank() : 0u;
  const int cl = blockIdx.x / csz;  // cluster index: the shared tile it reads
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], mode == 1 ? csz : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (mode == 1) cluster_sync_all();
  if (threadIdx.x == 0) {
    const int rows_per = 256 / csz;
    const uint16_t mask = (uint16_t)((1u << csz) - 1u);
    unsigned long long acc = 0;
    for (int kb = 0; kb < kblocks + kStages; ++kb) {
      const int s = kb % kStages;
      if (kb >= kStages) {  // consume k-block kb - kStages, release its stage cluster-wide
        bar_wait(&full[s], ((kb / kStages) - 1) & 1);
        acc += smem[s * (kW + kX) + (kb & 511)];
        if (mode == 1)
          for (int r = 0; r < csz; ++r) bar_arrive_remote(&empty[s], (uint32_t)r);
        else
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
      }
      if (kb < kblocks) {
        if (kb >= kStages) bar_wait(&empty[s], ((kb / kStages) - 1) & 1);
        uint8_t* st = smem + s * (kW + kX);
        bar_expect(&full[s], kW + kX);
        load2d(&mw, &full[s], st, (kb % 48) * 64, blockIdx.x * 128);
        if (mode == 1) {
          for (int r0 = (int)rank * rows_per; r0 < ((int)rank + 1) * rows_per; r0 += 16)
            load2d_mc(&mx, &full[s], st + kW + r0 * 128, (kb % 48) * 64, cl * 256 + r0, mask);
        } else {
          for (int r0 = 0; r0 < 256; r0 += 16) load2d(&mx, &full[s], st + kW + r0 * 128, (kb % 48) * 64, cl * 256 + r0);
        }
      }
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
  __syncthreads();
  if (mode == 1) cluster_sync_all();
}

static void make_map(CUtensorMap* m, void* p, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  if (cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, p, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    std::printf("encode failed\n");
    std::exit(1);
  }
}

int main(int argc, char** argv) {
  const int mode = atoi(argv[1]), csz = atoi(argv[2]);
  const int kblocks = argc > 3 ? atoi(argv[3]) : 480;
  const int grid = 144;  // divisible by 2, 4, 6, 8
  void *w, *x, *sink;
  const size_t wrows = (size_t)grid * 128, xrows = (size_t)(grid / csz) * 256 + 256;
  CK(cudaMalloc(&w, wrows * 3072 * 2));
  CK(cudaMalloc(&x, xrows * 3072 * 2));
  CK(cudaMemset(w, 0, wrows * 3072 * 2));
  CK(cudaMemset(x, 0, xrows * 3072 * 2));
  CK(cudaMalloc(&sink, 64));
  CUtensorMap mw, mx;
  make_map(&mw, w, wrows, 3072, 128);
  make_map(&mx, x, xrows, 3072, 16);
  const int smem = kStages * (kW + kX) + 1024 + 256;
  CK(cudaFuncSetAttribute(mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = mode == 1 ? csz : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(e0);
    CK(cudaLaunchKernelEx(&cfg, mc_kernel, mw, mx, kblocks, mode, csz, (unsigned long long*)sink));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2) ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  const double t = ts[ts.size() / 2] * 1e-3;
  const double bytes = (double)grid * kblocks * (kW + kX);
  std::printf("mode=%d cluster=%d kblocks=%d: %.1f us, delivered %.2f TB/s into smem (%.1f B/clk/SM @1.965GHz)\n",
              mode, csz, kblocks, t * 1e6, bytes / t / 1e12, bytes / t / 144 / 1.965e9);
  return 0;
}
