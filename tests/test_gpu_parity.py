"""Group-level parity on the B200: the CUDA engine (through the C ABI) vs the float64 oracle on
identical (fp16/fp32-rounded) weights and identical inputs.

Bar (BASELINE.json north star): fp32 logits within 1e-3 relative — |dz| <= 1e-3 * max|z_ref| per
request (conftest.rel_err_rows) — and identical argmax wherever the reference's top-2 margin exceeds
twice that tolerance (rows inside the band must be rare).
"""
import numpy as np
import pytest

from conftest import rel_err_rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-3


def _check_logits(got, ref, tol=TOL):
    err = rel_err_rows(got, ref)
    assert err <= tol, f"max row-relative logit error {err:.3e} > {tol}"
    ref2 = np.atleast_2d(ref)
    got2 = np.atleast_2d(got)
    srt = np.sort(ref2, axis=1)
    margin = (srt[:, -1] - srt[:, -2]) / np.maximum(np.abs(ref2).max(axis=1), 1e-30)
    decided = margin > 2 * tol
    assert np.array_equal(np.argmax(got2, 1)[decided], np.argmax(ref2, 1)[decided])
    assert decided.mean() >= 0.9, "too many near-tie rows to judge argmax parity"
    return err


def _seqs(rng, n, lo, hi, vocab=30522):
    out = []
    for _ in range(n):
        L = int(rng.integers(lo, hi + 1))
        ids = rng.integers(1000, vocab, size=L)
        ids[0] = 101  # [CLS]
        out.append(ids.astype(np.int32))
    return out


@pytest.fixture(scope="module")
def tiny():
    from oracle.bert import OracleBertGroup
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group

    cfg, K = PRESETS["tiny"]
    w = random_bert_group(cfg, K, seed=11)
    return StudentGroup(w, max_tokens=2048, max_seqs=64), OracleBertGroup(w)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_tiny_bert_group_all_prefixes(tiny, k):
    grp, orc = tiny
    rng = np.random.default_rng(100 + k)
    seqs = _seqs(rng, 7, 8, 64)
    rep_ref, z_ref = orc.forward(seqs, k)
    z = grp.logits(seqs, k)
    _check_logits(z, z_ref)
    rep = grp.rep(seqs, k)
    assert rel_err_rows(rep, rep_ref) <= TOL


def test_tiny_bert_batch1_single_sequence_squeezes(tiny):
    grp, orc = tiny
    ids = _seqs(np.random.default_rng(5), 1, 8, 64)[0]
    z = grp.logits(ids)
    assert z.shape == (2,)
    _, z_ref = orc.forward([ids])
    _check_logits(z, z_ref[0])


def test_tiny_bert_edge_lengths(tiny):
    """Length-1 sequences (CLS only), exactly one and just over one 64-token attention block."""
    grp, orc = tiny
    rng = np.random.default_rng(9)
    seqs = [s[:L] for s, L in zip(_seqs(rng, 5, 64, 64), [1, 2, 63, 64, 64])] + _seqs(rng, 2, 65, 130)
    _, z_ref = orc.forward(seqs)
    _check_logits(grp.logits(seqs), z_ref)


def test_tiny_bert_at_capacity(tiny):
    """A packed request that fills the group exactly (64 ragged sequences = max_seqs, 2048 tokens =
    max_tokens) matches the oracle for every prefix; one token or one sequence more is rejected."""
    grp, orc = tiny
    rng = np.random.default_rng(17)
    lens = rng.integers(1, 64, size=64)
    lens[-1] += 2048 - int(lens.sum())  # exactly max_tokens
    while lens[-1] < 1 or lens[-1] > 512:  # keep every sequence a legal length
        lens = rng.integers(1, 64, size=64)
        lens[-1] += 2048 - int(lens.sum())
    seqs = [np.concatenate([[101], rng.integers(1000, 30522, size=int(L) - 1)]).astype(np.int32) for L in lens]
    assert sum(len(x) for x in seqs) == 2048 and len(seqs) == 64
    for k in (1, 4):
        _, z_ref = orc.forward(seqs, k)
        _check_logits(grp.logits(seqs, k), z_ref)
    with pytest.raises(ValueError):
        grp.logits(seqs[:-1] + [np.concatenate([seqs[-1], [1000]]).astype(np.int32)])
    with pytest.raises(ValueError):
        grp.logits(seqs + [np.array([101], np.int32)])


def test_tiny_bert_k_out_of_range(tiny):
    grp, _ = tiny
    seqs = _seqs(np.random.default_rng(1), 2, 8, 16)
    for bad in (0, 5, -1):
        with pytest.raises(ValueError):
            grp.logits(seqs, bad)


def test_tiny_bert_rejects_bad_tokens(tiny):
    grp, _ = tiny
    with pytest.raises(ValueError):
        grp.logits([np.array([101, 30522], np.int32)])
    with pytest.raises(ValueError):
        grp.logits([np.array([], np.int32)])
    with pytest.raises(ValueError):
        grp.logits([np.arange(513, dtype=np.int32) + 1000])


def test_tiny_bert_host_api_matches_device_api(tiny):
    from paper_2408_12526_b200.group import pack_sequences

    grp, _ = tiny
    seqs = _seqs(np.random.default_rng(3), 4, 8, 64)
    ids, cu, _ = pack_sequences(seqs)
    z_host = grp.forward_host(ids, cu, 3)
    z_dev = grp.logits(seqs, 3)
    np.testing.assert_array_equal(z_host, z_dev.astype(np.float32))  # same kernels, same order: bit-identical


def test_torch_op_host_path_matches_forward_host(tiny):
    """torch.ops.studentpar.group_forward_host (the C++ extension over the same C entry point) and
    StudentGroup.forward_host (direct C call) return bit-identical logits."""
    from paper_2408_12526_b200.group import pack_sequences, torch_ops

    grp, _ = tiny
    ops = torch_ops()
    assert ops is not None, "the torch extension library was not built"
    for seqs in (_seqs(np.random.default_rng(5), 1, 8, 64), _seqs(np.random.default_rng(6), 3, 8, 64)):
        ids, cu, _ = pack_sequences(seqs)
        z = grp.forward_host(ids, cu, 3)
        out = torch.empty((len(cu) - 1, grp.n_classes), dtype=torch.float32)
        ops.group_forward_host(grp._handle.value, torch.from_numpy(ids), torch.from_numpy(cu), 3, out, True,
                               grp.device.index)
        np.testing.assert_array_equal(out.numpy(), z)


@pytest.mark.parametrize("exact", [True, False])
def test_dense_group_matches_oracle(exact):
    """exact=True: fp16 (hi, lo) weights (3 products per k-slice); exact=False: fp16 weights only."""
    from oracle.dense import group_forward_weights
    from paper_2408_12526_b200 import StudentGroup, random_dense_group

    w = random_dense_group(d_in=8, rep_dim=16, depth=2, n_students=3, n_classes=2, seed=4, exact=exact)
    assert w.exact_weights == exact
    grp = StudentGroup(w, max_tokens=512)
    x = np.random.default_rng(2).normal(size=(300, 8))
    for k in (1, 2, 3):
        rep_ref, z_ref = group_forward_weights(w, x, k)  # the engine carries x as an fp16 (hi, lo) pair
        _check_logits(grp.logits(x, k), z_ref)
        assert rel_err_rows(grp.rep(x, k), rep_ref) <= TOL


def test_dense_exact_weights_with_hi_only_input():
    """C-ABI dense forward with x_lo = NULL on a group that carries weight lo terms: the
    (token hi only, weight hi+lo) kernel instantiations, small-token and persistent paths."""
    from oracle.dense import group_forward_weights
    from paper_2408_12526_b200 import StudentGroup, random_dense_group

    w = random_dense_group(d_in=64, rep_dim=256, depth=2, n_students=3, n_classes=2, seed=12)
    assert w.exact_weights
    grp = StudentGroup(w, max_tokens=512)
    for n in (8, 40, 300):
        x = np.random.default_rng(n).normal(size=(n, 64)).astype(np.float16).astype(np.float64)
        x16 = torch.zeros((n, w.d_in_padded), dtype=torch.float16, device=grp.device)
        x16[:, :64] = torch.from_numpy(x).to(torch.float16).to(grp.device)
        logits = torch.empty((n, 2), dtype=torch.float32, device=grp.device)
        grp.forward_dense_device(x16, n, 3, None, logits, True, x16_lo=None)
        torch.cuda.synchronize()
        _, z_ref = group_forward_weights(w, x, 3)
        _check_logits(logits.cpu().numpy(), z_ref)


def test_dense_group_wide_matches_oracle():
    """Reference-architecture students at the BERT-base width (H=768, K=8)."""
    from oracle.dense import group_forward_weights
    from paper_2408_12526_b200 import StudentGroup, random_dense_group

    w = random_dense_group(d_in=768, rep_dim=768, depth=2, n_students=8, n_classes=2, seed=8)
    grp = StudentGroup(w, max_tokens=256)
    x = np.random.default_rng(3).normal(size=(256, 768))
    rep_ref, z_ref = group_forward_weights(w, x)
    _check_logits(grp.logits(x), z_ref)
    for n in (1, 16, 17, 100):  # small-T kernel (< 17 rows) and the persistent kernel with W lo tiles
        _, z_n = group_forward_weights(w, x[:n])
        _check_logits(grp.logits(x[:n]), z_n)
    x1 = x[0]
    z1 = grp.logits(x1)
    assert z1.shape == (2,)


def test_base_bert_group_batch1_parity():
    """BERT-base-sized group (K=8, H=768, 12 heads) at batch-1 on ragged lengths incl. L=512."""
    from oracle.bert import OracleBertGroup
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group

    cfg, K = PRESETS["base"]
    w = random_bert_group(cfg, K, seed=1)
    grp = StudentGroup(w, max_tokens=1024, max_seqs=8)
    orc = OracleBertGroup(w)
    rng = np.random.default_rng(0)
    for L in (16, 100, 512):
        ids = _seqs(rng, 1, L, L)
        _, z_ref = orc.forward(ids)
        _check_logits(grp.logits(ids), z_ref)
        _, z_ref4 = orc.forward(ids, 4)
        _check_logits(grp.logits(ids, 4), z_ref4)


@pytest.mark.parametrize("name", ["tiny", "pad", "wide"])
def test_dense_engine_matches_reference_golden(name):
    """Reference-built StudentModel groups (tests/golden, made by the unmodified reference) through
    the engine: logits vs the reference's own logits for every prefix k, argmax identical."""
    from goldens import load_dense
    from paper_2408_12526_b200 import StudentGroup, dense_group_from_arrays

    case = load_dense(name)
    w = dense_group_from_arrays(case["students"], case["alphas"], case["classifier"])
    grp = StudentGroup(w, max_tokens=256)
    # tiny holds float64 reference weights: the group carries their fp16 lo terms, so the engine
    # is held to the reference's own logits there too
    assert w.exact_weights == (not case["engine_precision"])
    for k in range(1, case["K"] + 1):
        z = grp.logits(case["x"], k)
        _check_logits(z, case["logits"][k])
        np.testing.assert_allclose(grp.rep(case["x"][0], k)[: w.rep_dim].shape, case["rep1"][k].shape)


def test_trained_reference_checkpoint_real_data_accuracy():
    """ensemble-checkpoint-v1 trained and saved by the reference -> engine: prefix accuracies on the
    reference's gaussian-task validation/test splits equal the reference's prefix_accuracy."""
    from goldens import GOLDEN, load_trained_task
    from oracle.dense import group_forward_weights
    from paper_2408_12526_b200 import StudentGroup

    task = load_trained_task()
    grp = StudentGroup.from_checkpoint(GOLDEN / "ensemble_trained.json", max_tokens=256)
    for k in range(1, len(grp) + 1):
        assert grp.accuracy(task["x_val"], task["y_val"], k) == pytest.approx(task["acc_val"][k - 1], abs=0)
        assert grp.accuracy(task["x_test"], task["y_test"], k) == pytest.approx(task["acc_test"][k - 1], abs=0)
        z = grp.logits(task["x_val"], k)
        # the checkpoint's float64 weights travel as fp16 (hi, lo) pairs: the engine reproduces the
        # reference's OWN logits (saved by the reference at training time) at the 1e-3 bar
        assert grp.weights.exact_weights
        _check_logits(z, task[f"logits_val_k{k}"])
        _, z_oracle = group_forward_weights(grp.weights, task["x_val"], k)
        _check_logits(z, z_oracle)


def test_reference_object_snapshot_if_available(ref):
    """StudentGroup.from_ensemble on a live reference EnsembleState (build container + GPU only)."""
    from paper_2408_12526_b200 import StudentGroup

    rng = np.random.Generator(np.random.PCG64(0))
    students = [ref.nn.StudentModel.build(32, 64, 2, rng) for _ in range(3)]
    state = ref.distill.EnsembleState(students, [1.0, 0.6, 0.3], ref.nn.DenseLayer.init(2, 64, "identity", rng))
    grp = StudentGroup.from_ensemble(state)
    x = rng.normal(size=(16, 32))
    _check_logits(grp.logits(x, 2), state.classifier.forward(state.rep(x, 2)))


def test_host_graph_path_bit_identical_to_device_path():
    """Batch-1 forward_host replays a captured CUDA graph per 16-token bucket (kernels read the live
    length from cu_seqlens); it must reproduce the eager device path bit for bit, across buckets
    and across replays of one bucket with different lengths and k."""
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group

    cfg, K = PRESETS["base"]
    w = random_bert_group(cfg, 3, seed=21)
    grp = StudentGroup(w, max_tokens=512, max_seqs=4)
    grp.prepare_graphs(64, 3)
    rng = np.random.default_rng(4)
    for L in (1, 15, 16, 17, 33, 48, 130, 300, 512):
        ids = _seqs(rng, 1, L, L)[0]
        for k in (3, 2):
            z_host = grp.forward_host(ids, np.array([0, L], np.int32), k)
            z_dev = grp.logits([ids], k).astype(np.float32)
            np.testing.assert_array_equal(z_host, z_dev)


@pytest.mark.parametrize("env", ["SP_ATTN_TC=0", "SP_ATTN_TC=1", "SP_ATTN_TC=2", "SP_ATTN_TC=3", "SP_GRAPHS=0"])
def test_forced_variants_match_oracle(env):
    """The two switches the engine keeps: SP_ATTN_TC forces one of the four attention kernels (the
    default picks by length), SP_GRAPHS=0 disables the batch-1 CUDA graphs. Each runs in a fresh
    process (switches are read once) against the float64 oracle at the 1e-3 bar."""
    import subprocess
    import sys

    code = (
        "import numpy as np, sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')\n"
        "from oracle.bert import OracleBertGroup\n"
        "from conftest import rel_err_rows\n"
        "from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group\n"
        "cfg, K = PRESETS['base']; w = random_bert_group(cfg, 3, seed=5)\n"
        "g = StudentGroup(w, max_tokens=1024, max_seqs=4); o = OracleBertGroup(w)\n"
        "rng = np.random.default_rng(0)\n"
        "cases = [[L] for L in (1, 16, 77, 128, 200, 512)] + [[5, 40, 60]]\n"
        "for lens in cases:\n"
        "    seqs = [np.r_[101, rng.integers(1000, 30522, size=L - 1)].astype(np.int32) for L in lens]\n"
        "    z = g.logits(seqs); _, zr = o.forward(seqs)\n"
        "    err = rel_err_rows(z, zr); assert err <= 1e-3, (lens, err)\n"
        "    if len(lens) == 1:\n"
        "        zh = g.forward_host(seqs[0], np.array([0, lens[0]], np.int32))\n"
        "        assert rel_err_rows(zh, zr) <= 1e-3\n"
        "print('ok')\n")
    key, val = env.split("=")
    import os

    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       env={**os.environ, key: val}, cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_device_graph_path_matches_eager():
    """sp_group_forward_graph (device buffers, bucket-graph replay) equals the eager forward (the bucket's
    tile configuration may change split-K summation order: fp32 rounding level)."""
    import torch
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group

    cfg, K = PRESETS["base"]
    g = StudentGroup(random_bert_group(cfg, 3, seed=11), max_tokens=512, max_seqs=1)
    rng = np.random.default_rng(3)
    out_g = torch.empty(1, cfg.n_classes, device="cuda")
    out_e = torch.empty(1, cfg.n_classes, device="cuda")
    for L in (1, 16, 17, 100, 129, 300, 512):
        ids = torch.from_numpy(np.r_[101, rng.integers(1000, cfg.vocab, size=L - 1)].astype(np.int32)).cuda()
        cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
        for k in (3, 1):
            g.forward_graph_device(ids, cu, L, k, out_g)
            g.forward_packed_device(ids, cu, 1, L, L, k, None, out_e)
            torch.cuda.synchronize()
            torch.testing.assert_close(out_g, out_e, rtol=1e-4, atol=1e-6)


def test_bert_student_checkpoint_loads_into_engine(tmp_path):
    """A BERT-kind group saved as ensemble-checkpoint-v1 (bert-student entries) and loaded through
    StudentGroup.from_checkpoint runs bit-identically to the group it was saved from."""
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
    from paper_2408_12526_b200.checkpoint import save_bert_ensemble

    cfg, K = PRESETS["tiny"]
    w = random_bert_group(cfg, K, seed=12)
    path = tmp_path / "bert_group.json"
    save_bert_ensemble(w, path)
    a = StudentGroup(w, max_tokens=512, max_seqs=8)
    b = StudentGroup.from_checkpoint(path, max_tokens=512, max_seqs=8)
    seqs = _seqs(np.random.default_rng(12), 5, 8, 64)
    for k in range(1, K + 1):
        np.testing.assert_array_equal(a.logits(seqs, k), b.logits(seqs, k))
