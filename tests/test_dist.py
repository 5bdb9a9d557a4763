"""world_size-2 gloo tests of the multi-GPU host logic (CPU only).

* shard_units partitions batch x KV heads exactly, sequence-major.
* The C1 exchange: each rank computes Eq. 3's column sums for its own KV heads (oracle
  arithmetic), the ranks all-reduce them, and the moments / rho computed from the
  reduced sums equal the single-process result — i.e. splitting a sequence's KV heads
  over ranks does not change rho (the CUDA path computes the local sums with
  arkv_prefill_begin and the moments with arkv_prefill_finish around the same reduce).
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2603_08727_b200.parallel import sequence_group_ranks, shard_units
from synth import Shape, prefill_inputs

pytestmark = pytest.mark.dist


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("batch,heads,world", [(1, 8, 1), (1, 8, 2), (1, 8, 8), (4, 8, 8), (8, 8, 4), (4, 8, 2)])
def test_shard_units_partition(batch, heads, world):
    seen = set()
    for r in range(world):
        s = shard_units(batch, heads, world, r)
        for b in range(s["seq_lo"], s["seq_hi"]):
            for h in range(s["kvh_lo"], s["kvh_hi"]):
                assert (b, h) not in seen
                seen.add((b, h))
        grp = sequence_group_ranks(batch, world, r)
        assert r in grp
    assert seen == {(b, h) for b in range(batch) for h in range(heads)}


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = Shape(batch=1, n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=16, prompt_len=80, window=8)
        cfg = O.Cfg(n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=16, window=8, budget_tokens=40)
        qw, k, v = prefill_inputs(sh, seed=13)
        s = shard_units(1, 4, world, rank)
        G = 2
        res = []
        for l in range(2):
            qwl = qw[0, l, s["kvh_lo"] * G:s["kvh_hi"] * G].double().numpy()
            kl = k[0, l, s["kvh_lo"]:s["kvh_hi"]].double().numpy()
            a = O.windowed_attention(qwl, kl, cfg)               # local heads only
            col = torch.tensor(a.sum(axis=(0, 1)))              # local Eq. 3 column sums
            dist.all_reduce(col, op=dist.ReduceOp.SUM)          # collective C1
            c = col.numpy()
            st = O.compute_stats(c / c.sum())
            res.append((st, O.oq_score(*st, cfg.tau)))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_c1_colsum_allreduce_matches_single_process():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sh = Shape(batch=1, n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=16, prompt_len=80, window=8)
    cfg = O.Cfg(n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=16, window=8, budget_tokens=40)
    qw, k, v = prefill_inputs(sh, seed=13)
    stats, oq, rho, _ = O.prefill_stats(qw.double().numpy(), k.double().numpy(), cfg)
    for r in range(world):
        for l in range(2):
            np.testing.assert_allclose(out[r][l][0], stats[0, l], rtol=1e-12)
            assert out[r][l][1] == pytest.approx(oq[0, l], rel=1e-12)
    # both ranks agree bitwise (NCCL/gloo all-reduce returns identical bytes)
    assert out[0] == out[1]


def _bench_worker(rank, world, port, q):
    """One rank of bench.py's own partition code on CPU: shard_units + shard_inputs +
    sequence_group, then the C1 column-sum all-reduce (oracle arithmetic for the local
    Eq. 3 sums, standing in for arkv_prefill_begin)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2603_08727_b200.parallel import sequence_group
        wl = dict(n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=16, batch=1, prompt_len=80, window=8)
        shard = shard_units(wl["batch"], wl["n_kv_heads"], world, rank)
        group = sequence_group(wl["batch"], world, rank)
        (qw, k, v), pool = bench.shard_inputs(wl, shard, 1234, "cpu", 3)
        cfg = O.Cfg(n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=16, window=8, budget_tokens=40)
        res = []
        for l in range(2):
            a = O.windowed_attention(qw[0, l].double().numpy(), k[0, l].double().numpy(), cfg)
            col = torch.tensor(a.sum(axis=(0, 1)))
            dist.all_reduce(col, op=dist.ReduceOp.SUM, group=group)
            c = col.numpy()
            res.append(O.oq_score(*O.compute_stats(c / c.sum()), cfg.tau))
        q.put((rank, (shard, [t.clone() for t in (qw, k, v)], [t.clone() for t in pool[2]], res)))
    finally:
        dist.destroy_process_group()


def test_bench_partition_world2():
    """bench.py --gpus 2 at a 1-sequence workload: each rank holds half the KV heads (and
    their q heads) of the same sequence, bit-identical to slicing the single-rank inputs;
    the C1 all-reduce over the sequence group gives both ranks the single-process q_l."""
    import bench
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = dict(n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=16, batch=1, prompt_len=80, window=8)
    full = shard_units(1, 4, 1, 0)
    (qw, k, v), pool = bench.shard_inputs(wl, full, 1234, "cpu", 3)
    for r in range(world):
        shard, (qr, kr, vr), step2, _ = out[r]
        h0, h1 = shard["kvh_lo"], shard["kvh_hi"]
        assert torch.equal(kr, k[:, :, h0:h1]) and torch.equal(vr, v[:, :, h0:h1])
        assert torch.equal(qr, qw[:, :, 2 * h0:2 * h1])
        assert torch.equal(step2[0], pool[2][0][:, :, 2 * h0:2 * h1]) and torch.equal(step2[1], pool[2][1][:, :, h0:h1])
    cfg = O.Cfg(n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=16, window=8, budget_tokens=40)
    _, oq, _, _ = O.prefill_stats(qw.double().numpy(), k.double().numpy(), cfg)
    for l in range(2):
        assert out[0][3][l] == pytest.approx(oq[0, l], rel=1e-12)
    assert out[0][3] == out[1][3]
