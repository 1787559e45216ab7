"""Multi-rank host logic on CPU: LPT sharding and the world_size-2 gather over
gloo (the N>1 path has no collective inside the step)."""

import os
import socket

import numpy as np
import pytest

from paper_1909_08723_b200.sharding import decode_corpus_sharded, plan_shards


class _F:
    def __init__(self, uid, n):
        self.utt_id, self.data = uid, np.zeros((n, 1), np.float32)


def test_plan_shards_is_a_balanced_partition():
    rng = np.random.default_rng(0)
    lengths = rng.integers(300, 3500, size=257).tolist()
    for world in (1, 2, 4, 8):
        shards = plan_shards(lengths, world)
        flat = sorted(i for s in shards for i in s)
        assert flat == list(range(len(lengths)))
        loads = [sum(lengths[i] for i in s) for s in shards]
        assert max(loads) - min(loads) <= max(lengths)
        for s in shards:
            assert [lengths[i] for i in s] == sorted(lengths[i] for i in s)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    feats = [_F(f"u{i}", 10 + (i * 37) % 50) for i in range(23)]

    def decode(batch):
        return [(f.utt_id, len(f.data), rank) for f in batch]

    out = decode_corpus_sharded(feats, decode, batch_size=4, rank=rank, world=world)
    q.put((rank, out))
    dist.destroy_process_group()


def test_world2_gloo_gather_restores_input_order():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert outs[0] == outs[1]
    res = outs[0]
    assert [r[0] for r in res] == [f"u{i}" for i in range(23)]
    assert {r[2] for r in res} == {0, 1}          # both ranks did work


def _oracle_worker(rank, world, port, q):
    """A real decode_fn: the oracle decoder (restated reference decode_batch +
    PyTorch-CPU adapters) of the c1 workload on this rank's shard."""
    import torch
    import torch.distributed as dist
    from oracle import harness as H
    torch.set_num_threads(1)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = H.workload("c1", n_utts=6)
    model = H.OracleModel(wl)
    utts = H.corpus(wl, 0)
    utts = [(u, x[: 120 + 40 * i]) for i, (u, x) in enumerate(utts)]     # ragged lengths
    feats = [_F(u, 1) for u, _ in utts]
    for f, (_, x) in zip(feats, utts):
        f.data = x
    seen = []

    def decode(shard):
        seen.extend(f.utt_id for f in shard)
        return model.decode([(f.utt_id, f.data) for f in shard])

    out = decode_corpus_sharded(feats, decode, rank=rank, world=world)
    q.put((rank, [(r.utt_id, list(r.tokens), r.score, r.steps) for r in out], seen))
    dist.destroy_process_group()


def test_world2_gloo_sharded_oracle_decode_equals_unsharded():
    """decode_corpus_sharded over two gloo ranks with the oracle decoder as
    decode_fn: every utterance decoded once, results gathered in input order
    and identical to one process decoding the whole corpus (batch
    invariance, reference test_acceptance.py:251-297)."""
    import torch.multiprocessing as mp
    from oracle import harness as H
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_oracle_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = {}
    for _ in procs:
        r, res, seen = q.get(timeout=300)
        outs[r] = (res, seen)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert outs[0][0] == outs[1][0]
    assert sorted(outs[0][1] + outs[1][1]) == sorted(r[0] for r in outs[0][0])
    assert outs[0][1] and outs[1][1]                      # both ranks decoded
    import torch
    nt = torch.get_num_threads()
    torch.set_num_threads(1)            # the ranks' CPU GEMMs ran single-threaded
    try:
        wl = H.workload("c1", n_utts=6)
        model = H.OracleModel(wl)
        utts = [(u, x[: 120 + 40 * i]) for i, (u, x) in enumerate(H.corpus(wl, 0))]
        want = [(r.utt_id, list(r.tokens), r.score, r.steps) for r in model.decode(utts)]
    finally:
        torch.set_num_threads(nt)
    assert outs[0][0] == want
