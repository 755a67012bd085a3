"""Multi-rank round-end exchange on CPU (gloo, world_size 2 and 3): clients sharded
k -> rank k mod G, all-to-all of client slices, shard-local aggregation (the oracle
stands in for the GPU kernel), all-gather of w'. The result must be bit-identical to
the single-process deterministic aggregation for every world size."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fedopt_ref


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_kernel(srcs, nks, deterministic, w_slice, m_slice, w_out, m_out, eta, mu, nesterov, agg):
    w = w_slice.numpy()
    deltas = [w.astype(np.float64) - s.numpy().astype(np.float64) for s in srcs]
    pg = fedopt_ref.finalize_deltas(deltas, nks, list(range(len(srcs))), deterministic)
    wn, mn = fedopt_ref.server_step(w, m_slice.numpy(), pg, eta, mu, nesterov)
    w_out.copy_(torch.from_numpy(wn))
    m_out.copy_(torch.from_numpy(mn))


def _worker(rank, world, port, n, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_10853_b200.dist import ShardedAggregator, clients_of
    rng = np.random.default_rng(5)
    w = rng.normal(0, 0.02, n).astype(np.float32)
    m = rng.normal(0, 1e-3, n).astype(np.float32)
    wks = [(w + rng.normal(0, 2e-3, n)).astype(np.float32) for _ in range(K)]
    nk = {k: 1000 + 7 * k for k in range(K)}
    agg = ShardedAggregator(n, K, device="cpu", kernel=_oracle_kernel)
    local = {k: torch.from_numpy(wks[k]) for k in clients_of(rank, world, K)}
    agg.exchange(local)
    w_new, m_shard = agg.step(torch.from_numpy(w), torch.from_numpy(m[agg.lo:agg.hi].copy()), nk, 0.7, 0.9, True)
    q.put((rank, w_new.numpy(), agg.lo, agg.hi, m_shard.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,K", [(2, 1001, 8), (3, 4099, 5), (2, 64, 3)])
def test_sharded_exchange_bit_identical(world, n, K):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, K, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    w = rng.normal(0, 0.02, n).astype(np.float32)
    m = rng.normal(0, 1e-3, n).astype(np.float32)
    wks = [(w + rng.normal(0, 2e-3, n)).astype(np.float32) for _ in range(K)]
    ref_w, ref_m = fedopt_ref.fed_round(w, m, wks, [1000 + 7 * k for k in range(K)], 0.7, 0.9, True)
    m_full = np.zeros(n, np.float32)
    for rank, wn, lo, hi, ms in res:
        assert np.array_equal(wn.view(np.uint32), ref_w.view(np.uint32)), rank
        m_full[lo:hi] = ms
    assert np.array_equal(m_full.view(np.uint32), ref_m.view(np.uint32))


def test_shard_bounds_cover():
    from paper_2405_10853_b200.dist import clients_of, shard_bounds
    for n in (1, 7, 1000, 1339232256):
        for G in (1, 2, 4, 8):
            spans = [shard_bounds(n, G, r)[:2] for r in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all(lo % 4 == 0 for lo, hi in spans if hi > lo)
    assert clients_of(1, 4, 8) == [1, 5]


def _worker_round_end(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_10853_b200.dist import NO_BAD, gather_vector, reduce_round_end, shard_bounds
    full = torch.arange(n, dtype=torch.float32) * 0.5 - 3.0
    lo, hi, _ = shard_bounds(n, world, rank)
    m_full = gather_vector(full[lo:hi].clone(), n)        # the checkpoint's momentum (federation.py)
    stats = torch.full((6 + 3,), float(rank + 1), dtype=torch.float64)
    bad = torch.tensor([NO_BAD if rank != 1 else lo + 5], dtype=torch.int64)
    s, first_bad = reduce_round_end(stats, bad)
    q.put((rank, m_full.numpy(), s, first_bad, lo))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1001), (3, 10)])
def test_round_end_gather_and_reduce(world, n):
    """G > 1 round end (federation.py): the sharded momentum gathers to the full [N] vector
    (so a checkpoint is restorable, server.py:164), the per-shard norm statistics sum, and
    the first non-finite index is the minimum over ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_round_end, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.arange(n, dtype=np.float32) * 0.5 - 3.0
    lo1 = res[1][4]
    for rank, m_full, s, first_bad, _ in res:
        assert m_full.shape == (n,) and np.array_equal(m_full, want)
        assert np.allclose(s, sum(range(1, world + 1)))
        assert first_bad == lo1 + 5
