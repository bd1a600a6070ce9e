// chain_probe.cu — the floor of a chain of dependent kernels on this GPU.
//
// Times (CUDA events around a captured graph, 200 replays) a chain of N kernels where each kernel
// must see the previous kernel's writes:
//   mode 0: plain launches (stream order)
//   mode 1: programmatic dependent launch (launch_dependents at entry, griddepcontrol.wait before
//           reading the previous kernel's output) — what the engine's chain does
//   mode 2: one persistent kernel, phases separated by a grid-wide barrier (atomic arrive + spin
//           on a generation counter with acquire loads) — the megakernel alternative
// Each phase: every CTA reads one value the previous phase wrote and writes one value.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/experiments/chain_probe.cu -o /tmp/cp
//   /tmp/cp <ctas> <threads> <n_kernels>
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

__global__ void step_kernel(const float* in, float* out, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const float v = in[blockIdx.x];
  if (threadIdx.x == 0) out[blockIdx.x] = v + 1.f;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// grid barrier: count arrivals; the last arriver bumps the generation
__device__ void grid_sync(unsigned* count, unsigned* gen, unsigned n_ctas) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == n_ctas - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (ld_acquire(gen) == g) {
      }
    }
  }
  __syncthreads();
}

__global__ void persistent_kernel(float* buf, int n_phases, unsigned* count, unsigned* gen) {
  for (int p = 0; p < n_phases; ++p) {
    const float* in = buf + (size_t)(p & 1) * gridDim.x;
    float* out = buf + (size_t)((p + 1) & 1) * gridDim.x;
    const float v = in[(blockIdx.x + 1) % gridDim.x];  // a value another CTA wrote
    if (threadIdx.x == 0) out[blockIdx.x] = v + 1.f;
    grid_sync(count, gen, gridDim.x);
  }
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 148;
  const int threads = argc > 2 ? atoi(argv[2]) : 128;
  const int n = argc > 3 ? atoi(argv[3]) : 16;
  float* buf;
  unsigned* sync;
  CK(cudaMalloc(&buf, sizeof(float) * 2 * ctas));
  CK(cudaMemset(buf, 0, sizeof(float) * 2 * ctas));
  CK(cudaMalloc(&sync, 256));
  CK(cudaMemset(sync, 0, 256));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (int mode = 0; mode < 3; ++mode) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
    if (mode < 2) {
      for (int i = 0; i < n; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(threads);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = (mode == 1 && i > 0) ? 1 : 0;
        const float* in = buf + (size_t)(i & 1) * ctas;
        float* out = buf + (size_t)((i + 1) & 1) * ctas;
        CK(cudaLaunchKernelEx(&cfg, step_kernel, in, out, mode));
      }
    } else {
      persistent_kernel<<<ctas, threads, 0, st>>>(buf, n, sync, sync + 32);
    }
    CK(cudaStreamEndCapture(st, &graph));
    cudaGraphExec_t exec;
    CK(cudaGraphInstantiate(&exec, graph, 0));
    for (int r = 0; r < 20; ++r) CK(cudaGraphLaunch(exec, st));
    CK(cudaStreamSynchronize(st));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<float> ts;
    for (int r = 0; r < 200; ++r) {
      cudaEventRecord(e0, st);
      CK(cudaGraphLaunch(exec, st));
      cudaEventRecord(e1, st);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms * 1e3f);
    }
    std::sort(ts.begin(), ts.end());
    const char* names[3] = {"plain launches", "PDL launches", "persistent + grid barrier"};
    std::printf("ctas=%d threads=%d steps=%d %-26s median %.1f us  (%.2f us per step)\n", ctas, threads, n,
                names[mode], ts[ts.size() / 2], ts[ts.size() / 2] / n);
    CK(cudaGraphExecDestroy(exec));
    CK(cudaGraphDestroy(graph));
  }
  return 0;
}
