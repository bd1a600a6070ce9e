"""Parity at every BASELINE.json configuration at full K, and the serving loop on the real engine.

* BERT-large-sized group (K=12, H=1024, 16 heads): batched ragged requests large enough (>= 1024
  tokens) that the persistent projections run as CTA pairs (tcgen05 cta_group::2), and batch-1 at
  both ends of the length range;
* BERT-base-sized group (K=8): 16 ragged requests in one batch;
* the K=32 group at every prefix the adaptive path can select.
Bar everywhere (BASELINE.json): |dz| <= 1e-3 * max|z_ref| per request (conftest.rel_err_rows) and
identical argmax wherever the reference's top-2 margin exceeds twice that.
"""
import numpy as np
import pytest

from conftest import rel_err_rows

pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-3


def _seqs(rng, lens, vocab=30522):
    out = []
    for L in lens:
        ids = rng.integers(1000, vocab, size=int(L)).astype(np.int32)
        ids[0] = 101
        out.append(ids)
    return out


def _check(z, z_ref):
    z, z_ref = np.atleast_2d(z), np.atleast_2d(z_ref)
    err = rel_err_rows(z, z_ref)
    assert err <= TOL, f"max row-relative logit error {err:.3e}"
    srt = np.sort(z_ref, axis=1)
    decided = (srt[:, -1] - srt[:, -2]) > 2 * TOL * np.abs(z_ref).max(axis=1)
    assert np.array_equal(np.argmax(z, 1)[decided], np.argmax(z_ref, 1)[decided])
    return err


@pytest.fixture(scope="module")
def large():
    from oracle.bert import OracleBertGroup
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group

    cfg, K = PRESETS["large"]
    assert K == 12
    w = random_bert_group(cfg, K, seed=21)
    return StudentGroup(w, max_tokens=2048, max_seqs=16), OracleBertGroup(w)


def test_large_bert_full_group_batched_pair_path(large):
    grp, orc = large
    rng = np.random.default_rng(3)
    seqs = _seqs(rng, rng.integers(100, 220, size=8))
    assert sum(len(s) for s in seqs) >= 1024  # the paired persistent GEMM path
    _, z_ref = orc.forward(seqs)
    _check(grp.logits(seqs), z_ref)


@pytest.mark.parametrize("L", [512, 1])
def test_large_bert_full_group_batch1_extreme_lengths(large, L):
    """Batch-1 at the maximum position count (persistent projections, longest attention) and a lone
    CLS token; the host path (forward_host, bucket graph) and the reference-style logits() agree."""
    grp, orc = large
    ids = _seqs(np.random.default_rng(L), [L])[0]
    _, z_ref = orc.forward([ids])
    z = grp.logits(ids)
    _check(z, z_ref)
    cu = np.array([0, L], np.int32)
    np.testing.assert_allclose(grp.forward_host(ids, cu)[0], z, rtol=0, atol=1e-5)
    with pytest.raises(ValueError):
        grp.logits(np.concatenate([ids, ids]) if L == 512 else np.zeros(0, np.int32))


def test_base_bert_full_group_16_ragged_requests():
    from oracle.bert import OracleBertGroup
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group

    cfg, K = PRESETS["base"]
    w = random_bert_group(cfg, K, seed=41)
    grp = StudentGroup(w, max_tokens=8192, max_seqs=16)
    rng = np.random.default_rng(41)
    seqs = _seqs(rng, rng.integers(16, 513, size=16))
    _, z_ref = OracleBertGroup(w).forward(seqs)
    _check(grp.logits(seqs), z_ref)


def test_k32_group_batch1_every_adaptive_prefix():
    """K=32 students: every prefix k the adaptive path can pick, on the max-|logit| bar."""
    from oracle.bert import OracleBertGroup
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group

    cfg, K = PRESETS["k32"]
    assert K == 32
    w = random_bert_group(cfg, K, seed=5)
    grp = StudentGroup(w, max_tokens=128, max_seqs=1)
    ids = _seqs(np.random.default_rng(8), [48])[0]
    orc = OracleBertGroup(w)
    for k in (1, 8, 16, 17, 32):
        _, z_ref = orc.forward([ids], k)
        _check(grp.logits(ids, k), z_ref)


def test_adaptive_server_on_engine_single_and_batched():
    """The serving loop drives the real engine through forward_host on a bursty trace (B8 group,
    k in [2, 8]): single request in flight (bucket graphs) and continuous batching (queued requests
    packed into one unpadded launch). Every launch's logits equal the same requests run one by one
    at the launch's k."""
    import time

    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
    from paper_2408_12526_b200.serving import AdaptiveServer, generate_phases, synth_tokens

    cfg, K = PRESETS["base"]
    group = StudentGroup(random_bert_group(cfg, K, seed=1), max_tokens=4096, max_seqs=32)
    trace = generate_phases([(2000.0, 20.0), (40000.0, 5.0), (1000.0, 40.0)], seed=0, max_len=512, bin_width=32)
    tokens = {r.id: synth_tokens(r, 0, cfg.vocab) for r in trace}
    checked = []

    def execute(batch, k, active):
        ids = np.concatenate([tokens[r.id] for r in batch])
        cu = np.concatenate([[0], np.cumsum([len(tokens[r.id]) for r in batch])]).astype(np.int32)
        t0 = time.perf_counter()
        z = group.forward_host(ids, cu, k)
        ms = 1e3 * (time.perf_counter() - t0)
        assert z.shape == (len(batch), 2) and np.all(np.isfinite(z))
        if len(batch) > 1 and len(checked) < 3:
            one = np.stack([group.forward_host(tokens[r.id], np.array([0, len(tokens[r.id])], np.int32), k)[0]
                            for r in batch])
            np.testing.assert_allclose(z, one, rtol=0, atol=2e-5)
            checked.append(len(batch))
        return ms

    single = AdaptiveServer(execute, max_students=K, min_students=2, buffer_capacity=16, idle_window_ms=5.0)
    m1 = single.run(trace)
    assert m1.completed == len(trace) and max(single.batches) == 1
    batched = AdaptiveServer(execute, max_students=K, min_students=2, buffer_capacity=256, idle_window_ms=5.0,
                             max_batch_seqs=32, max_batch_tokens=4096)
    m2 = batched.run(trace)
    assert m2.completed == len(trace) and max(batched.batches) > 1 and checked
    assert all(2 <= r.k <= K for r in m1.records + m2.records)


def test_sharded_host_path_matches_group_host_path():
    """ShardedStudentGroup.forward_host (the N-GPU bench's e2e path: pinned staging, forward,
    logit reduce, D2H) at world size 1 equals StudentGroup.forward_host on the same weights."""
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
    from paper_2408_12526_b200.parallel import ShardedStudentGroup

    cfg, K = PRESETS["tiny"]
    sh = ShardedStudentGroup(cfg, K, seed=4, rank=0, world=1, max_tokens=256, max_seqs=4)
    ref = StudentGroup(random_bert_group(cfg, K, seed=4), max_tokens=256, max_seqs=4)
    rng = np.random.default_rng(2)
    for lens in ([17], [5, 60, 33], [128, 1]):
        seqs = _seqs(rng, lens)
        ids = np.concatenate(seqs)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        for k in (1, K):
            z = sh.forward_host(ids, cu, k)
            assert z.shape == (len(lens), 2)
            np.testing.assert_allclose(z, ref.forward_host(ids, cu, k), rtol=0, atol=1e-5)


def test_sharded_partials_sum_to_group_logits():
    """Two shards of one group (world size 2, ranks built in this process, so the logit reduce is
    skipped): their partial logits sum to the whole group's logits. Batch-1 runs each shard's bucket
    graph (the N-GPU bench step, graphs captured ahead by prepare_graphs); a prefix k that leaves a
    shard without students gives that shard zero partials; several sequences take the eager path."""
    import torch
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
    from paper_2408_12526_b200.parallel import ShardedStudentGroup

    cfg, K = PRESETS["tiny"]
    shards = [ShardedStudentGroup(cfg, K, seed=6, rank=r, world=2, max_tokens=256, max_seqs=4) for r in range(2)]
    ref = StudentGroup(random_bert_group(cfg, K, seed=6), max_tokens=256, max_seqs=4)
    for sh in shards:
        sh.prepare_graphs(64, K)
    rng = np.random.default_rng(9)
    for lens in ([7], [16], [33], [64], [5, 60, 33]):
        seqs = _seqs(rng, lens)
        ids = np.concatenate(seqs)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        d_ids = torch.from_numpy(ids).cuda()
        d_cu = torch.from_numpy(cu).cuda()
        for k in (1, 2, 3, K):
            want = ref.forward_host(ids, cu, k)
            parts_host = [sh.forward_host(ids, cu, k) for sh in shards]
            np.testing.assert_allclose(parts_host[0] + parts_host[1], want, rtol=0, atol=1e-5)
            parts_dev = []
            for sh in shards:
                z = torch.full((4, 2), float("nan"), device="cuda")
                sh.forward_packed_device(d_ids, d_cu, len(lens), len(ids), max(lens), k, z)
                parts_dev.append(z[: len(lens)].cpu().numpy())
            np.testing.assert_allclose(parts_dev[0] + parts_dev[1], want, rtol=0, atol=1e-5)
            if k == 1:
                assert not parts_dev[1].any() and not parts_host[1].any()


def test_p2p_mailbox_reduce_two_shards_matches_group():
    """Device-side logit reduce (sp_reduce.cu): two shards of one group in this process share the
    root's mailbox; rank 1 publishes its partial logits, rank 0 publishes and combines in rank order.
    The root's logits equal the whole group's (device path with graphs, eager batched path, and the
    host path through mapped memory without a stream sync), for prefixes that leave rank 1 empty."""
    import torch
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
    from paper_2408_12526_b200.parallel import ShardedStudentGroup

    cfg, K = PRESETS["tiny"]
    root = ShardedStudentGroup(cfg, K, seed=7, rank=0, world=2, max_tokens=256, max_seqs=4, reduce="p2p")
    peer = ShardedStudentGroup(cfg, K, seed=7, rank=1, world=2, max_tokens=256, max_seqs=4, reduce="p2p",
                               mailbox=root.mailbox)
    ref = StudentGroup(random_bert_group(cfg, K, seed=7), max_tokens=256, max_seqs=4)
    rng = np.random.default_rng(5)
    for rep in range(3):  # more requests than mailbox banks
        for lens in ([9], [16], [40], [5, 60, 33]):
            seqs = _seqs(rng, lens)
            ids = np.concatenate(seqs)
            cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
            d_ids, d_cu = torch.from_numpy(ids).cuda(), torch.from_numpy(cu).cuda()
            for k in (1, 3, K):
                want = ref.forward_host(ids, cu, k)
                out = torch.full((4, 2), float("nan"), device="cuda")
                junk = torch.zeros((4, 2), device="cuda")
                peer.forward_packed_device(d_ids, d_cu, len(lens), len(ids), max(lens), k, junk)
                root.forward_packed_device(d_ids, d_cu, len(lens), len(ids), max(lens), k, out)
                np.testing.assert_allclose(out[: len(lens)].cpu().numpy(), want, rtol=0, atol=1e-5)
                assert peer.forward_host(ids, cu, k) is None
                z = root.forward_host(ids, cu, k)
                np.testing.assert_allclose(z, want, rtol=0, atol=1e-5)
    assert root._seq == peer._seq
