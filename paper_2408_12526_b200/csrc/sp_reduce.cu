// sp_reduce.cu — the device-side logit reduce of a sharded student group.
//
// Each rank holds K/n students and computes partial logits z_r = W_c sum_{m in r, m < k} alpha_m S_m
// (bias on rank 0 only). Instead of a collective, every rank STORES its [n_rows][C] partial into
// its slot of a mailbox that lives on the root's GPU (reached over NVLink through a CUDA-IPC
// mapping of the root's allocation) and then raises a per-rank sequence flag with release
// semantics; the root's combine kernel waits for every flag of the request and sums the slots in
// FIXED rank order (deterministic, independent of arrival order), writing the logits to device or
// host-mapped memory plus an optional host-visible completion flag. The paper models this
// exchange as a 0.2 ms gather (servesim.py:294-304); here it is two tiny kernels and
// 8 bytes per rank at batch-1 (C = 2).
//
// Mailbox layout (bytes): [0, 64) consumed sequence number (int64, written by the root); [64, 64 +
// 64 W) one 64-byte line per rank holding its latest published sequence number; then
// kBanks x W x max_rows x C floats. Request seq uses bank seq % kBanks; a publisher first waits
// until the root has consumed seq - kBanks, so at most kBanks requests are in flight per mailbox.
#include <cstdint>
#include <cstring>

#include "../../include/studentpar_b200.h"
#include "sp_kernels.cuh"

namespace sp {

namespace {

constexpr int kBanks = 4;

__device__ __forceinline__ long long ld_acquire_sys(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(long long* p, long long v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void spin_until_at_least(const long long* p, long long target) {
  const long long t0 = clock64();
  while (ld_acquire_sys(p) < target) {
    __nanosleep(32);
    if (clock64() - t0 > 20000000000LL) __trap();  // ~10 s: a peer that never publishes
  }
}

__host__ __device__ __forceinline__ size_t slots_offset(int world) { return 64 + 64 * (size_t)world; }

// slot of (request seq, rank): bank seq % kBanks, fixed stride cap = max_rows x C floats
__global__ void publish_kernel(uint8_t* mbox, const float* __restrict__ partial, int rank, int world, int n,
                               int cap, long long seq) {
  long long* consumed = reinterpret_cast<long long*>(mbox);
  long long* flag = reinterpret_cast<long long*>(mbox + 64 + 64 * (size_t)rank);
  if (threadIdx.x == 0 && seq > kBanks) spin_until_at_least(consumed, seq - kBanks);  // bank free
  __syncthreads();
  float* dst = reinterpret_cast<float*>(mbox + slots_offset(world)) + ((size_t)(seq % kBanks) * world + rank) * cap;
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = partial[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) st_release_sys(flag, seq);
}

__global__ void combine_kernel(uint8_t* mbox, int world, int n, int cap, int n_classes, long long seq,
                               const float* __restrict__ bias, float* out, int* out_flag) {
  long long* consumed = reinterpret_cast<long long*>(mbox);
  if (threadIdx.x < world) spin_until_at_least(reinterpret_cast<long long*>(mbox + 64 + 64 * (size_t)threadIdx.x), seq);
  __syncthreads();
  const float* src = reinterpret_cast<const float*>(mbox + slots_offset(world)) + (size_t)(seq % kBanks) * world * cap;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    float z = 0.f;
    for (int r = 0; r < world; ++r) z += __ldcv(src + (size_t)r * cap + i);  // rank order: deterministic
    if (bias) z += bias[i % n_classes];
    out[i] = z;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    st_release_sys(consumed, seq);
    if (out_flag) *reinterpret_cast<volatile int*>(out_flag) = (int)seq;
  }
}

}  // namespace

}  // namespace sp

extern "C" {

long long sp_reduce_mailbox_bytes(int32_t world, int32_t max_rows, int32_t n_classes) {
  if (world < 1 || max_rows < 1 || n_classes < 1) return -1;
  return (long long)sp::slots_offset(world) + (long long)sp::kBanks * world * max_rows * n_classes * 4;
}

int sp_reduce_publish(void* mailbox, const float* partial, int32_t rank, int32_t world, int32_t n_rows,
                      int32_t max_rows, int32_t n_classes, int64_t seq, void* stream) {
  if (!mailbox || !partial || rank < 0 || rank >= world || n_rows < 1 || n_rows > max_rows || n_classes < 1 || seq < 1)
    return sp::report_error(SP_EINVAL, "sp_reduce_publish: bad argument");
  sp::publish_kernel<<<1, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint8_t*>(mailbox), partial, rank, world, n_rows * n_classes, max_rows * n_classes, (long long)seq);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SP_OK : sp::report_error(SP_ECUDA, cudaGetErrorString(e));
}

int sp_reduce_combine(void* mailbox, int32_t world, int32_t n_rows, int32_t max_rows, int32_t n_classes, int64_t seq,
                      const float* bias, float* out, int32_t* out_flag, void* stream) {
  if (!mailbox || !out || world < 1 || world > 128 || n_rows < 1 || n_rows > max_rows || n_classes < 1 || seq < 1)
    return sp::report_error(SP_EINVAL, "sp_reduce_combine: bad argument");
  sp::combine_kernel<<<1, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint8_t*>(mailbox), world, n_rows * n_classes, max_rows * n_classes, n_classes, (long long)seq, bias,
      out, out_flag);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SP_OK : sp::report_error(SP_ECUDA, cudaGetErrorString(e));
}

int sp_mailbox_create(int32_t world, int32_t max_rows, int32_t n_classes, int32_t device, void** out) {
  if (!out) return sp::report_error(SP_EINVAL, "null output");
  *out = nullptr;
  const long long bytes = sp_reduce_mailbox_bytes(world, max_rows, n_classes);
  if (bytes < 0) return sp::report_error(SP_EINVAL, "sp_mailbox_create: bad shape");
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(out, (size_t)bytes);  // its own allocation: IPC maps it whole
  if (e == cudaSuccess) e = cudaMemset(*out, 0, (size_t)bytes);
  return e == cudaSuccess ? SP_OK : sp::report_error(SP_ECUDA, cudaGetErrorString(e));
}

int sp_mailbox_destroy(void* mailbox) {
  if (mailbox) cudaFree(mailbox);
  return SP_OK;
}

int sp_ipc_get_handle(const void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return SP_EINVAL;
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) return sp::report_error(SP_ECUDA, cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle_out, &h, sizeof(h));
  return SP_OK;
}

int sp_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return SP_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? SP_OK : sp::report_error(SP_ECUDA, cudaGetErrorString(e));
}

int sp_ipc_close_handle(void* dev_ptr) {
  if (!dev_ptr) return SP_EINVAL;
  const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? SP_OK : sp::report_error(SP_ECUDA, cudaGetErrorString(e));
}

}  // extern "C"
