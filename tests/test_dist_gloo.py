"""Multi-GPU student sharding, exercised on CPU with world_size 2 over gloo.

Each rank holds the round-robin shard of the group (parallel.placement, servesim.py:231), computes
its partial logits W_c sum_{m in shard, m < k} alpha_m S_m (bias only on rank 0; the per-shard
compute is the float64 oracle here since there is no GPU), and the product's reduce_partials
all-reduces them. The result must equal the full group's logits for every prefix k.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_12526_b200.parallel import local_prefix, placement, reduce_partials
from paper_2408_12526_b200.weights import BertConfig, random_bert_group

CFG = BertConfig(hidden=16, n_layers=1, n_heads=2, vocab=64, max_pos=16, n_classes=3)
K = 5
SEQS = [np.array([1, 5, 9, 33], np.int32), np.array([1, 60], np.int32), np.array([1], np.int32)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q):
    from oracle.bert import OracleBertGroup

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = placement(K, world)[rank]
        shard = random_bert_group(CFG, K, seed=9, students=mine)
        orc = OracleBertGroup(shard)
        results = {}
        for k in range(1, K + 1):
            kl = local_prefix(k, mine, K)
            rep = np.zeros((len(SEQS), CFG.hidden))
            for j in range(kl):
                rep += orc.alpha[j] * orc.pooled(j, SEQS)
            z = rep @ orc.w_cls.T + (orc.b_cls if rank == 0 else 0.0)
            t = torch.from_numpy(z.copy())
            reduce_partials(t)
            results[k] = t.numpy()
        out_q.put((rank, results))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_group_reduce_equals_full_group():
    from oracle.bert import OracleBertGroup

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = OracleBertGroup(random_bert_group(CFG, K, seed=9))
    for k in range(1, K + 1):
        _, z_ref = full.forward(SEQS, k)
        for r in range(world):
            np.testing.assert_allclose(got[r][k], z_ref, rtol=1e-12, atol=1e-14)
        np.testing.assert_array_equal(got[0][k], got[1][k])  # every rank answers identically
