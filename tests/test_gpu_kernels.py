"""Per-kernel numerics on the B200: each sm_100a kernel against a plain PyTorch reference of the same
op. The kernels take fp16 weights and (hi, lo) fp16 activation pairs with fp32 accumulation, so a
GEMM on an fp32 activation matches the float64 product to ~1e-6 relative."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _split(x):
    """fp32 tensor -> (hi, lo) fp16 pair, hi + lo = x to ~2^-22 relative (the engine's operand format)."""
    hi = x.half()
    lo = (x - hi.float()).half()
    return hi, lo


def _gemm_ref(w, x, bias, act, x_group_rows):
    G, N, K = w.shape
    T = x.shape[0] if x_group_rows == 0 else x_group_rows
    outs = []
    for g in range(G):
        xg = x if x_group_rows == 0 else x[g * x_group_rows:(g + 1) * x_group_rows]
        y = xg.double() @ w[g].double().T
        if bias is not None:
            y = y + bias[g]
        if act == 1:
            y = torch.tanh(y)
        elif act == 2:
            y = torch.nn.functional.gelu(y)
        outs.append(y)
    return torch.stack(outs)


@pytest.mark.parametrize("T", [1, 16, 20, 64, 100, 256, 300, 520])
@pytest.mark.parametrize("act", [0, 1, 2])
def test_gemm_matches_torch(cuda_lib, T, act):
    from paper_2408_12526_b200 import _lib

    torch.manual_seed(T * 3 + act)
    G, N, K = 3, 256, 192
    dev = "cuda"
    w = (torch.randn(G, N, K, device=dev) * 0.05).half()
    x = torch.randn(G * T, K, device=dev)
    xh, xl = _split(x)
    bias = torch.randn(G, N, device=dev) * 0.1
    out = torch.empty(G, T, N, device=dev, dtype=torch.float32)
    _lib.check(cuda_lib.sp_op_gemm(w.data_ptr(), xh.data_ptr(), xl.data_ptr(), G, N, K, T, T, G * T, bias.data_ptr(),
                                   act, out.data_ptr(), None, 1, 1, None))
    torch.cuda.synchronize()
    ref = _gemm_ref(w, x, bias, act, T)
    torch.testing.assert_close(out.double(), ref, rtol=2e-6, atol=2e-6)


@pytest.mark.parametrize("T", [16, 200])
def test_gemm_hilo_operand_removes_fp16_rounding(cuda_lib, T):
    """The lo term is what carries the precision: hi only is off by ~2e-4 of max|y| (fp16 rounding of
    the activation), hi + lo by ~3e-6 (fp32 accumulation over K = 768), on both the small-T and the
    persistent kernel."""
    from paper_2408_12526_b200 import _lib

    torch.manual_seed(T)
    G, N, K = 2, 256, 768
    w = (torch.randn(G, N, K, device="cuda") * 0.05).half()
    x = torch.randn(G * T, K, device="cuda")
    xh, xl = _split(x)
    ref = _gemm_ref(w, x, None, 0, T)
    errs = []
    for lo in (None, xl):
        out = torch.empty(G, T, N, device="cuda", dtype=torch.float32)
        _lib.check(cuda_lib.sp_op_gemm(w.data_ptr(), xh.data_ptr(), None if lo is None else lo.data_ptr(), G, N, K, T,
                                       T, G * T, None, 0, out.data_ptr(), None, 1, 1, None))
        torch.cuda.synchronize()
        errs.append(float((out.double() - ref).abs().max() / ref.abs().max()))
    assert errs[0] > 1e-4 and errs[1] < 1e-5 and errs[0] > 30 * errs[1], errs


@pytest.mark.parametrize("T", [5, 48, 130])
def test_gemm_fp16_out_shared_input(cuda_lib, T):
    """x_group_rows = 0: every student reads the same rows (dense kind input_proj)."""
    from paper_2408_12526_b200 import _lib

    torch.manual_seed(7)
    G, N, K = 4, 128, 64
    w = (torch.randn(G, N, K, device="cuda") * 0.1).half()
    x = torch.randn(T, K, device="cuda").half()
    out = torch.empty(2, G, T, N, device="cuda", dtype=torch.float16)  # (hi, lo) output planes
    _lib.check(cuda_lib.sp_op_gemm(w.data_ptr(), x.data_ptr(), None, G, N, K, T, 0, T, None, 1, out[0].data_ptr(),
                                   out[1].data_ptr(), 0, 1, None))
    torch.cuda.synchronize()
    ref = _gemm_ref(w, x, None, 1, 0)
    torch.testing.assert_close(out[0].double(), ref, rtol=2e-3, atol=2e-3)  # hi: fp16 rounding of the output
    torch.testing.assert_close(out[0].double() + out[1].double(), ref, rtol=2e-6, atol=2e-6)


@pytest.mark.parametrize("splits", [2, 3, 6])
def test_gemm_split_k_partials(cuda_lib, splits):
    from paper_2408_12526_b200 import _lib

    torch.manual_seed(splits)
    G, N, K, T = 2, 384, 768, 37
    w = (torch.randn(G, N, K, device="cuda") * 0.03).half()
    x = torch.randn(G * T, K, device="cuda")
    xh, xl = _split(x)
    part = torch.empty(splits, G, T, N, device="cuda", dtype=torch.float32)
    _lib.check(cuda_lib.sp_op_gemm(w.data_ptr(), xh.data_ptr(), xl.data_ptr(), G, N, K, T, T, G * T, None, 0,
                                   part.data_ptr(), None, 1, splits, None))
    torch.cuda.synchronize()
    ref = _gemm_ref(w, x, None, 0, T)
    torch.testing.assert_close(part.double().sum(0), ref, rtol=2e-6, atol=2e-6)


def _attn_ref(qkv, cu, G, nh, hd):
    H = nh * hd
    out = torch.zeros(qkv.shape[0], qkv.shape[1], H, device=qkv.device)
    for g in range(G):
        for b in range(len(cu) - 1):
            s, e = int(cu[b]), int(cu[b + 1])
            q = qkv[g, s:e, :H].float().view(e - s, nh, hd).transpose(0, 1)
            k = qkv[g, s:e, H:2 * H].float().view(e - s, nh, hd).transpose(0, 1)
            v = qkv[g, s:e, 2 * H:].float().view(e - s, nh, hd).transpose(0, 1)
            p = torch.softmax(q @ k.transpose(1, 2) / math.sqrt(hd), dim=-1)
            out[g, s:e] = (p @ v).transpose(0, 1).reshape(e - s, H)
    return out


@pytest.mark.parametrize("hd,nh,lens", [(64, 12, [1, 17, 64, 65, 200]), (32, 4, [8, 33, 64, 3]),
                                         (32, 8, [200, 1, 65]),
                                         (64, 16, [512, 1, 130]), (64, 8, [100, 1, 128, 37]),
                                         (64, 12, [416, 385, 3])])
def test_attention_varlen_matches_torch(cuda_lib, hd, nh, lens):
    from paper_2408_12526_b200 import _lib

    torch.manual_seed(sum(lens))
    G, H = 2, nh * hd
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(cu[-1])
    cap = T + 5
    qkv = torch.randn(G, cap, 3 * H, device="cuda").half()
    ctx = torch.zeros(2, G, cap, H, device="cuda", dtype=torch.float16)  # (hi, lo) context planes
    cu_d = torch.from_numpy(cu).cuda()
    _lib.check(cuda_lib.sp_op_attention(qkv.data_ptr(), ctx[0].data_ptr(), ctx[1].data_ptr(), cu_d.data_ptr(),
                                        len(lens), max(lens), G, nh, hd, cap, None))
    torch.cuda.synchronize()
    ref = _attn_ref(qkv, cu, G, nh, hd)
    got = ctx[0, :, :T].float() + ctx[1, :, :T].float()
    # the kernels round P to fp16 for the P V product: ~1e-4 of |ctx|
    torch.testing.assert_close(got, ref[:, :T], rtol=2e-3, atol=2e-3)
    assert torch.all(ctx[:, :, T:] == 0), "attention wrote past the packed tokens"


_FORCED_ATTN = r"""
import math, sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2408_12526_b200 import _lib
from test_gpu_kernels import _attn_ref
lib = _lib.load()
cases = [(64, 12, [1, 17, 64, 65, 200]), (64, 16, [512, 1, 130]), (64, 8, [100, 1, 128, 37]),
         (64, 12, [416, 385, 3]), (64, 4, [256, 255, 129]), (64, 4, [511, 300]),
         (32, 4, [8, 33, 64, 3]), (32, 8, [300, 1, 129])]  # head_dim 32: mma.sync (0) or the tc3 variant
for grow in (False, True):
    for hd, nh, lens in cases:
        torch.manual_seed(sum(lens) + grow)
        G, H = 2, nh * hd
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        T = int(cu[-1]); cap = T + 5
        qkv = torch.randn(G, cap, 3 * H, device='cuda')
        if grow:  # scores that keep rising along the keys: exercises the running-max rescale
            qkv[:, :, H:2 * H] *= torch.linspace(0.2, 3.0, cap, device='cuda')[None, :, None]
        qkv = qkv.half()
        ctx = torch.zeros(2, G, cap, H, device='cuda', dtype=torch.float16)
        cu_d = torch.from_numpy(cu).cuda()
        _lib.check(lib.sp_op_attention(qkv.data_ptr(), ctx[0].data_ptr(), ctx[1].data_ptr(), cu_d.data_ptr(),
                                       len(lens), max(lens), G, nh, hd, cap, None))
        torch.cuda.synchronize()
        ref = _attn_ref(qkv, cu, G, nh, hd)
        torch.testing.assert_close(ctx[0, :, :T].float() + ctx[1, :, :T].float(), ref[:, :T], rtol=2e-3, atol=2e-3)
        assert torch.all(ctx[:, :, T:] == 0)
print('ok')
"""


@pytest.mark.parametrize("kind", ["0", "1", "2", "3"])
def test_attention_kernels_forced(kind):
    """Every attention kernel (mma.sync, two-pass tcgen05, single-pass two-CTA tcgen05) against the
    fp32 reference at every length class, with and without key scores that rise along the sequence
    (forces the single-pass kernel's running-max rescale). Fresh process: SP_ATTN_TC is read once."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    r = subprocess.run([sys.executable, "-c", _FORCED_ATTN], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "SP_ATTN_TC": kind}, cwd=str(Path(__file__).resolve().parents[1]))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
