// sp_torch.cpp — the thin PyTorch C++ extension over the engine's C ABI (torch.ops.studentpar.*).
//
// The hot calls of StudentGroup go through these ops instead of ctypes: the arguments arrive as
// tensors, the stream is torch's current CUDA stream of the tensors' device (no Python-side stream
// lookup), and a failing sp_* status becomes a RuntimeError carrying sp_last_error(). Every op is a
// direct call of one C-ABI entry point (include/studentpar_b200.h); there is no compute here.
#include <ATen/ATen.h>
#include <c10/cuda/CUDAStream.h>
#include <torch/library.h>

#include "../../include/studentpar_b200.h"

namespace {

sp_group* as_group(int64_t handle) {
  TORCH_CHECK(handle != 0, "studentpar: null group handle");
  return reinterpret_cast<sp_group*>(static_cast<intptr_t>(handle));
}

void check(int rc) {
  if (rc == SP_OK) return;
  const char* msg = sp_last_error();
  TORCH_CHECK_VALUE(rc != SP_EINVAL, "studentpar: ", msg ? msg : "invalid argument");
  TORCH_CHECK(false, "studentpar: CUDA engine failure: ", msg ? msg : "");
}

void check_dev(const at::Tensor& t, at::ScalarType dt, const char* name) {
  TORCH_CHECK(t.is_cuda(), "studentpar: ", name, " must be a CUDA tensor");
  TORCH_CHECK(t.scalar_type() == dt, "studentpar: ", name, " has the wrong dtype");
  TORCH_CHECK(t.is_contiguous(), "studentpar: ", name, " must be contiguous");
}

void* stream_of(const at::Tensor& t) {
  return static_cast<void*>(c10::cuda::getCurrentCUDAStream(t.device().index()).stream());
}

// sp_group_forward: ids int32 [T], cu int32 [B+1], logits f32 [B, C] (all on the group's device)
void group_forward(int64_t handle, const at::Tensor& ids, const at::Tensor& cu, int64_t n_seqs, int64_t n_tokens,
                   int64_t max_len, int64_t k, const at::Tensor& logits, bool add_bias) {
  as_group(handle);
  check_dev(ids, at::kInt, "ids");
  check_dev(cu, at::kInt, "cu_seqlens");
  check_dev(logits, at::kFloat, "logits");
  check(sp_group_forward(as_group(handle), ids.data_ptr<int32_t>(), cu.data_ptr<int32_t>(), (int32_t)n_seqs,
                         (int32_t)n_tokens, (int32_t)max_len, (int32_t)k, nullptr, logits.data_ptr<float>(),
                         add_bias ? 1 : 0, stream_of(ids)));
}

// sp_group_forward_graph: one sequence as its bucket's CUDA graph, device buffers
void group_forward_graph(int64_t handle, const at::Tensor& ids, const at::Tensor& cu, int64_t n_tokens, int64_t k,
                         const at::Tensor& logits, bool add_bias) {
  as_group(handle);
  check_dev(ids, at::kInt, "ids");
  check_dev(cu, at::kInt, "cu_seqlens");
  check_dev(logits, at::kFloat, "logits");
  check(sp_group_forward_graph(as_group(handle), ids.data_ptr<int32_t>(), cu.data_ptr<int32_t>(), (int32_t)n_tokens,
                               (int32_t)k, logits.data_ptr<float>(), add_bias ? 1 : 0, stream_of(logits)));
}

// sp_group_forward_host: HOST ids / cu_seqlens in, HOST logits out (the serving seam)
void group_forward_host(int64_t handle, const at::Tensor& ids, const at::Tensor& cu, int64_t k, const at::Tensor& out,
                        bool add_bias, int64_t device) {
  sp_group* g = as_group(handle);
  TORCH_CHECK(!ids.is_cuda() && !cu.is_cuda() && !out.is_cuda(), "studentpar: forward_host takes host tensors");
  TORCH_CHECK(ids.scalar_type() == at::kInt && cu.scalar_type() == at::kInt && out.scalar_type() == at::kFloat,
              "studentpar: ids / cu_seqlens int32, out float32");
  TORCH_CHECK(ids.is_contiguous() && cu.is_contiguous() && out.is_contiguous(), "studentpar: contiguous tensors");
  const int64_t n = cu.numel() - 1;
  TORCH_CHECK(n >= 1 && out.dim() == 2 && out.size(0) >= n, "studentpar: out must hold [n_seqs, C] logits");
  void* st = static_cast<void*>(c10::cuda::getCurrentCUDAStream(device).stream());
  check(sp_group_forward_host(g, ids.data_ptr<int32_t>(), cu.data_ptr<int32_t>(), (int32_t)n,
                              (int32_t)ids.numel(), (int32_t)k, out.data_ptr<float>(), add_bias ? 1 : 0, st));
}

}  // namespace

TORCH_LIBRARY(studentpar, m) {
  m.def("group_forward(int handle, Tensor ids, Tensor cu, int n_seqs, int n_tokens, int max_len, int k, "
        "Tensor(a!) logits, bool add_bias) -> ()",
        &group_forward);
  m.def("group_forward_graph(int handle, Tensor ids, Tensor cu, int n_tokens, int k, Tensor(a!) logits, "
        "bool add_bias) -> ()",
        &group_forward_graph);
  m.def("group_forward_host(int handle, Tensor ids, Tensor cu, int k, Tensor(a!) out, bool add_bias, int device) -> ()",
        &group_forward_host);
}
