"""Host-side logic of the engine on CPU: input packing/validation, weight shards, placement and
prefix-k mapping, checkpoint ingestion, seeding and the serving-side restatements — checked
against golden vectors from the unmodified reference (tests/golden/)."""
import json

import numpy as np
import pytest

from goldens import GOLDEN, load_trained_task
from paper_2408_12526_b200 import serving
from paper_2408_12526_b200.checkpoint import ensemble_arrays_from_dict, load_ensemble_weights
from paper_2408_12526_b200.group import pack_sequences, validate_packed
from paper_2408_12526_b200.parallel import local_prefix, placement
from paper_2408_12526_b200.seeding import fork_seed
from paper_2408_12526_b200.weights import BertConfig, random_bert_group, random_dense_group

SS = np.load(GOLDEN / "servesim_ref.npz")


def test_pack_sequences_and_squeeze():
    ids, cu, sq = pack_sequences([np.array([101, 5, 6]), np.array([101])])
    assert ids.dtype == np.int32 and cu.tolist() == [0, 3, 4] and not sq
    ids, cu, sq = pack_sequences(np.array([101, 7], np.int32))
    assert sq and cu.tolist() == [0, 2]
    ids2, cu2, sq2 = pack_sequences((ids, cu))
    assert np.array_equal(ids2, ids) and not sq2


@pytest.mark.parametrize("ids,cu", [
    ([1, 2], [0, 1, 1]),          # empty sequence
    ([1, 2], [1, 2]),             # cu[0] != 0
    ([1, 2, 3], [0, 2]),          # cu[-1] != len(ids)
    ([1, 99], [0, 2]),            # id outside vocab
    (list(range(9)), [0, 9]),     # longer than max_pos
])
def test_validate_packed_rejects(ids, cu):
    with pytest.raises(ValueError):
        validate_packed(np.asarray(ids), np.asarray(cu), vocab=50, max_pos=8)


def test_bert_shard_is_bitwise_subset_of_group():
    cfg = BertConfig(hidden=16, n_heads=2, vocab=40, max_pos=8)
    full = random_bert_group(cfg, 5, seed=3)
    shard = random_bert_group(cfg, 5, seed=3, students=[1, 3])
    sub = full.subset([1, 3])
    for name in ["word_emb", "w_qkv", "b_ffn2", "w_pool", "alpha", "w_cls", "ln2_gamma"]:
        assert np.array_equal(getattr(shard, name), getattr(sub, name)), name
    assert full.alpha[0] == 1.0


def test_placement_matches_reference_allocate_students():
    # reference (servesim.py:225-234): (group j, student i) -> (i + j*S) % G; one group (j = 0)
    keys, vals = SS["alloc_keys"], SS["alloc_vals"]
    ref = {(int(j), int(i)): int(g) for (j, i), g in zip(keys, vals)}
    for i in range(3):
        assert ref[(0, i)] == i % 4
    pl = placement(3, 4)
    for rank, studs in enumerate(pl):
        for i in studs:
            assert ref[(0, i)] == rank
    assert placement(8, 8) == [[i] for i in range(8)]
    assert placement(32, 8)[3] == [3, 11, 19, 27]
    with pytest.raises(ValueError):
        placement(0, 2)


def test_local_prefix_partitions_global_k():
    for K, world in [(8, 1), (8, 2), (12, 8), (32, 8), (5, 3)]:
        pl = placement(K, world)
        for k in range(1, K + 1):
            counts = [local_prefix(k, pl[r], K) for r in range(world)]
            assert sum(counts) == k
    with pytest.raises(ValueError):
        local_prefix(0, [0], 4)
    with pytest.raises(ValueError):
        local_prefix(5, [0], 4)


def test_checkpoint_loader_reads_reference_ensemble():
    """ensemble-checkpoint-v1 written by the reference's save_ensemble (distill.py:604-607)."""
    d = json.loads((GOLDEN / "ensemble_trained.json").read_text())
    students, multipliers, clf = ensemble_arrays_from_dict(d)
    assert multipliers[0] == 1.0 and len(students) == len(multipliers)
    w = load_ensemble_weights(GOLDEN / "ensemble_trained.json")
    assert w.n_students == len(students) and w.rep_dim == students[0][0][0].shape[0]
    # oracle on the decoded float64 arrays reproduces the reference's prefix accuracies exactly
    from oracle.dense import group_forward

    task = load_trained_task()
    for k in range(1, len(students) + 1):
        _, z = group_forward(students, multipliers, clf, task["x_val"], k)
        np.testing.assert_allclose(z, task[f"logits_val_k{k}"], rtol=1e-12, atol=1e-14)
        acc = float(np.mean(np.argmax(z, 1) == task["y_val"]))
        assert acc == pytest.approx(task["acc_val"][k - 1], abs=0)


def test_checkpoint_rejects_bad_input():
    d = json.loads((GOLDEN / "ensemble_trained.json").read_text())
    bad = dict(d, schema="something-else")
    with pytest.raises(ValueError):
        ensemble_arrays_from_dict(bad)
    bad = json.loads(json.dumps(d))
    bad["mode"] = "json"
    bad["students"][0]["mode"] = "json"
    lay = bad["students"][0]["input_proj"]
    lay["weight"] = [[float("nan")] * lay["in_dim"]] * lay["out_dim"]
    with pytest.raises(ValueError):
        ensemble_arrays_from_dict(bad)


def test_fork_seed_matches_reference():
    got = np.asarray([fork_seed(0, "x"), fork_seed(12345, "bert-student-7")], dtype=np.uint64)
    assert np.array_equal(got, SS["fork_seed_0_x"])


def test_generate_workload_matches_reference():
    reqs = serving.generate_workload(serving.PoissonSpec(rps=2000.0, duration_ms=50.0), seed=7)
    np.testing.assert_array_equal([r.arrival_ms for r in reqs], SS["wl_arrival"])
    np.testing.assert_array_equal([r.length_tokens for r in reqs], SS["wl_len"])
    reqs2 = serving.generate_workload(serving.PoissonSpec(rps=500.0, duration_ms=100.0), seed=1, max_len=512,
                                      bin_width=32)
    np.testing.assert_array_equal([r.arrival_ms for r in reqs2], SS["wl2_arrival"])
    np.testing.assert_array_equal([r.length_tokens for r in reqs2], SS["wl2_len"])


def test_generate_phases_matches_reference_cli_semantics():
    reqs = serving.generate_phases([(2000.0, 40.0), (10000.0, 25.0), (2000.0, 60.0)], seed=11)
    np.testing.assert_array_equal([r.arrival_ms for r in reqs], SS["ph_arrival"])
    np.testing.assert_array_equal([r.length_tokens for r in reqs], SS["ph_len"])
    assert [r.id for r in reqs] == list(range(len(reqs)))


def test_nearest_rank_percentile_matches_reference():
    vals = list(SS["pct_values"])
    for p, exp in zip(SS["pct_p"], SS["pct_out"]):
        assert serving.nearest_rank_percentile(vals, p) == exp
    with pytest.raises(ValueError):
        serving.nearest_rank_percentile([], 50)


def test_controller_rule_matches_reference_table():
    code = {serving.DROP_ONE: 0, serving.ADD_ONE: 1, serving.HOLD: 2}
    for k, full, idle, idle_s, occ_s, exp in SS["ctrl_cases"]:
        got = serving.decide_controller_action(int(k), 1, 8, bool(full), None if idle < 0 else float(idle),
                                               int(idle_s), int(occ_s), 100.0)
        assert code[got] == int(exp)


def test_adaptive_server_drops_under_burst_and_recovers():
    """Bursty trace (cli.py phases shape): the controller sheds students while the backlog is
    full and adds them back after the idle window; k is snapshotted per request."""
    reqs = serving.generate_phases([(2000.0, 100.0), (20000.0, 20.0), (500.0, 400.0)], seed=0)

    def execute(batch, k, active):  # synthetic service time: 0.1 ms per active student per request
        return 0.1 * k * len(batch)

    srv = serving.AdaptiveServer(execute, max_students=8, min_students=2, buffer_capacity=4, idle_window_ms=5.0)
    m = srv.run(reqs)
    assert m.completed == len(reqs)
    ks = [k for _, k in m.k_timeline]
    assert min(ks) < 8, "burst should drop students"
    assert ks[-1] == 8, "idle tail should restore the full group"
    assert all(2 <= r.k <= 8 for r in m.records)
    assert m.p99_ms >= m.p50_ms > 0


def test_adaptive_server_continuous_batching_packs_the_backlog():
    """With max_batch_seqs > 1 every launch takes the whole FIFO backlog (up to the token budget) the
    moment the engine is free: no batching wait (a lone request runs alone), no padding."""
    reqs = serving.generate_phases([(2000.0, 50.0), (50000.0, 10.0), (500.0, 200.0)], seed=1, max_len=128)
    seen = []

    def execute(batch, k, active):
        assert active == 1  # one launch in flight per GPU
        seen.append(batch)
        return 0.05 + 0.002 * sum(r.length_tokens for r in batch)

    srv = serving.AdaptiveServer(execute, max_students=8, min_students=2, buffer_capacity=256,
                                 max_batch_seqs=64, max_batch_tokens=2048)
    m = srv.run(reqs)
    assert m.completed == len(reqs)
    assert max(len(b) for b in seen) > 1 and min(len(b) for b in seen) == 1
    assert all(len(b) <= 64 and (len(b) == 1 or sum(r.length_tokens for r in b) <= 2048) for b in seen)
    order = [r.id for b in seen for r in b]
    assert order == sorted(order)  # FIFO


def test_adaptive_server_reproduces_reference_simulation(ref):
    """The serving loop is the reference's event loop: driven by the reference's own analytic
    service_time (servesim.py:287-307) with one request per element (max_merge=1) and the
    reference's slots / buffer capacity (group_count, :220-222), it reproduces Simulation's
    student-number timeline and every request's completion time exactly, through a burst that
    drops students and an idle tail that adds them back."""
    import studentpar.perfmodel as pm

    sim = ref.servesim
    model = pm.PerfModel()
    model.calibrate(pm.baseline_reference(), 11.6)
    factors = sim.ServiceFactors(model=model, depth=2, width_per_student=256, capacity=pm.DEFAULT_CAPACITY,
                                 pcie_tokens_per_ms=pm.DEFAULT_PCIE_TOKENS_PER_MS, gather_ms=pm.DEFAULT_GATHER_MS)
    table = ref.distill.AccuracyTable([(k, 0.9 + 0.01 * k, 0.9 + 0.01 * k) for k in range(1, 4)])
    ctl = sim.ControllerConfig(max_students=3, accuracy_table=table, min_students=1, idle_window_ms=300.0)
    G, R = 4, 3
    cluster = sim.ClusterConfig(controller=ctl, nodes=1, gpus_per_node=G, group_size=3, replicas_per_gpu=R,
                                max_merge=1)
    reqs = serving.generate_phases([(2000.0, 200.0), (30000.0, 60.0), (300.0, 900.0)], seed=3)
    ref_reqs = [sim.Request(r.id, r.arrival_ms, r.length_tokens) for r in reqs]
    want = sim.run_simulation(cluster, ref_reqs, factors)

    def execute(batch, k, active):
        (r,) = batch
        b = sim.bin_of(r.length_tokens, cluster)
        el = sim.BufferElement(bin=b, padded_len=(b + 1) * cluster.bin_width, requests=[ref_reqs[r.id]])
        return sim.service_time(el, k, cluster, factors, active_groups=active)

    cap = lambda k: sim.group_count(k, G, R)  # noqa: E731
    srv = serving.AdaptiveServer(execute, max_students=3, min_students=1, start_k=3, buffer_capacity=cap,
                                 idle_window_ms=300.0, max_batch_seqs=1, slots=cap)
    got = srv.run(reqs)
    assert [k for _, k in got.k_timeline] == [k for _, k in want.student_number_timeline]
    assert [t for t, _ in got.k_timeline] == pytest.approx([t for t, _ in want.student_number_timeline], abs=1e-9)
    assert min(k for _, k in got.k_timeline) < 3 and got.k_timeline[-1][1] == 3
    assert srv.rejected_pushes == want.rejected_pushes
    assert [(r.request_id, r.completion_ms) for r in got.records] == \
        pytest.approx([(r.request_id, r.completion_ms) for r in want.per_request], abs=1e-9)


@pytest.mark.parametrize("mode", ["binary", "json"])
def test_bert_student_checkpoint_round_trip_bit_exact(tmp_path, mode):
    """bert-student entries in ensemble-checkpoint-v1 (checkpoint.py): save -> load reproduces every
    array bit for bit (float64 base64 / decimal lists of fp16 / fp32 values)."""
    from paper_2408_12526_b200.checkpoint import load_ensemble_weights, save_bert_ensemble

    cfg = BertConfig(hidden=128, n_heads=4, n_layers=2, vocab=300, max_pos=40, n_classes=3)
    w = random_bert_group(cfg, 3, seed=5)
    path = tmp_path / f"bert_{mode}.json"
    save_bert_ensemble(w, path, mode)
    back = load_ensemble_weights(path)
    assert back.cfg == w.cfg and back.kind == "bert"
    for name in ["word_emb", "pos_emb", "type_emb", "emb_ln_gamma", "emb_ln_beta", "w_qkv", "b_qkv", "w_o", "b_o",
                 "ln1_gamma", "ln1_beta", "w_ffn1", "b_ffn1", "w_ffn2", "b_ffn2", "ln2_gamma", "ln2_beta", "w_pool",
                 "b_pool", "alpha", "w_cls", "b_cls"]:
        a, b = getattr(w, name), getattr(back, name)
        assert a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes(), name


def test_bert_student_checkpoint_rejects_malformed(tmp_path):
    import copy

    from paper_2408_12526_b200.checkpoint import bert_group_from_dict, bert_group_to_dict

    cfg = BertConfig(hidden=128, n_heads=4, n_layers=1, vocab=64, max_pos=16)
    d = bert_group_to_dict(random_bert_group(cfg, 2, seed=1), "json")
    bert_group_from_dict(d)
    bad = copy.deepcopy(d)
    bad["students"][1]["layers"][0]["ffn1"]["activation"] = "tanh"
    with pytest.raises(ValueError):
        bert_group_from_dict(bad)
    bad = copy.deepcopy(d)
    bad["multipliers"][0] = 0.5  # alpha_0 must be 1 (distill.py:152-153)
    with pytest.raises(ValueError):
        bert_group_from_dict(bad)
    bad = copy.deepcopy(d)
    bad["students"][0]["pooler"]["bias"][3] = float("nan")  # nnkernel.py:486-487
    with pytest.raises(ValueError):
        bert_group_from_dict(bad)
    bad = copy.deepcopy(d)
    bad["students"][0]["layers"][0]["o"]["out_dim"] = 64
    with pytest.raises(ValueError):
        bert_group_from_dict(bad)
