"""Multi-GPU round-end exchange: clients sharded over ranks, one fused aggregation.

Partitioning: client k trains on rank k mod G; its end weights w_k
stay in that rank's HBM. At round end every rank needs, for its N/G slice of the
parameter vector, every client's slice — an all-to-all of f32 client shards
(grouped NCCL send/recv over NVLink 5). Each rank then runs the single-GPU fused
kernel (fb_fedagg_step_f32) on its slice with the clients in id order, which
makes the result bit-identical to G = 1 (the f64 pairwise tree never crosses a
rank boundary), and an all-gather of f32 w' rebuilds the global model on every
rank. Momentum stays sharded. Bytes per rank per direction:
4 N ceil(K/G) (G-1)/G (all-to-all) + 4 N (G-1)/G (all-gather).
"""
from __future__ import annotations

import ctypes as C

from . import ext


def shard_bounds(n: int, world: int, rank: int, align: int = 4):
    """Contiguous, 16-byte aligned slice [lo, hi) of an n-vector owned by `rank`."""
    per = ((n + world - 1) // world + align - 1) // align * align
    lo = min(n, rank * per)
    hi = min(n, lo + per)
    return lo, hi, per


def clients_of(rank: int, world: int, n_clients: int):
    return [k for k in range(n_clients) if k % world == rank]


NO_BAD = 1 << 62  # "no non-finite index" (any value >= n means none)


def gather_vector(shard, n: int, group=None):
    """All ranks' contiguous shards (shard_bounds layout) -> the full [n] vector on every rank.
    Used for the server momentum before a checkpoint (restore_server, server.py:164, needs
    the full-length vector)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi, per = shard_bounds(n, world, rank)
    mine = torch.zeros(per, dtype=shard.dtype, device=shard.device)
    mine[: hi - lo].copy_(shard[: hi - lo])
    if dist.get_backend(group) == "nccl":
        full = torch.empty(per * world, dtype=shard.dtype, device=shard.device)
        dist.all_gather_into_tensor(full, mine, group=group)
    else:
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        full = torch.cat(parts)
    return full[:n]


def reduce_round_end(stats, bad, group=None):
    """Sum the per-shard telemetry side reductions and take the global first non-finite index
    (min over ranks) in one host round trip: (stats f64 numpy, first_bad int)."""
    import torch
    import torch.distributed as dist
    s = stats.clone()
    b = bad.clone()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(s, group=group)
        dist.all_reduce(b, op=dist.ReduceOp.MIN, group=group)
    return s.cpu().numpy(), int(b.item())


def _global_bad(local_bad, count: int, offset: int):
    """A kernel's first-bad index (relative to its launch of `count` elements, >= count when
    none) -> a global index, or NO_BAD."""
    import torch
    return torch.where(local_bad < count, local_bad + offset, torch.full_like(local_bad, NO_BAD))


class ShardedAggregator:
    """Round-end aggregation + outer step across `world` ranks (torch.distributed / NCCL).

    local: {client_id: f32 device tensor [N]} for the clients this rank trained;
    n_k:   {client_id: n_k} for ALL contributing clients (known from the round plan).
    w: the global model (replicated, f32 [N]); m_shard: this rank's momentum slice."""

    def __init__(self, n: int, n_clients: int, group=None, device=None, kernel=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n = n
        self.K = n_clients
        self.lo, self.hi, self.per = shard_bounds(n, self.world, self.rank)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        # shard-local aggregation + outer step; the GPU kernel unless a test injects the oracle
        self.kernel = kernel or fused_kernel
        # receive buffers: one slice per client (padded to `per`); none needed on one GPU
        self.recv = torch.empty(self.K if self.world > 1 else 0, self.per, dtype=torch.float32, device=dev)
        self.src = {}
        self.w_full = torch.empty(self.per * self.world, dtype=torch.float32, device=dev)
        # round-norm side reductions of this shard (fb_fedagg_round_norms_f32): 6 fixed + K clients
        self.stats = torch.zeros(6 + n_clients, dtype=torch.float64, device=dev)
        self.bad = torch.full((1,), NO_BAD, dtype=torch.int64, device=dev)  # global index after step()
        self.ids = list(range(n_clients))

    def exchange(self, local: dict):
        """all-to-all: every client's slice r lands on rank r (grouped send/recv)."""
        if self.world == 1:
            self.src = dict(local)
            return
        self.src = {k: self.recv[k] for k in range(self.K)}
        dist = self.dist
        ops = []
        for k in range(self.K):
            owner = k % self.world
            if owner == self.rank:
                wk = local[k]
                for r in range(self.world):
                    lo, hi, _ = shard_bounds(self.n, self.world, r)
                    if r == self.rank:
                        self.recv[k, : hi - lo].copy_(wk[lo:hi], non_blocking=True)
                    elif hi > lo:
                        ops.append(dist.P2POp(dist.isend, wk[lo:hi], r, self.group))
            elif self.hi > self.lo:
                ops.append(dist.P2POp(dist.irecv, self.recv[k, : self.hi - self.lo], owner, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def step(self, w, m_shard, n_k: dict, eta, mu, nesterov, deterministic=True, w_out=None):
        """Fused aggregation + outer step on this rank's slice, then all-gather of w'."""
        import torch
        cnt = self.hi - self.lo
        ids = sorted(n_k) if deterministic else list(n_k)
        w_slice = w[self.lo:self.hi]
        m_new = torch.empty_like(m_shard)
        wo = self.w_full[self.rank * self.per: self.rank * self.per + cnt]
        self.ids = ids
        self.stats.zero_()
        self.bad.fill_(NO_BAD)
        if cnt > 0:
            self.kernel([self.src[k][:cnt] for k in ids], [int(n_k[k]) for k in ids], deterministic, w_slice,
                        m_shard, wo, m_new, eta, mu, nesterov, self)
            self.bad.copy_(_global_bad(self.bad, cnt, self.lo))
        if self.world > 1:
            mine = self.w_full[self.rank * self.per:(self.rank + 1) * self.per]
            if self.dist.get_backend(self.group) == "nccl":
                self.dist.all_gather_into_tensor(self.w_full, mine, group=self.group)
            else:
                parts = list(self.w_full.split(self.per))
                self.dist.all_gather(parts, mine.clone(), group=self.group)
        out = w_out if w_out is not None else torch.empty_like(w)
        out.copy_(self.w_full[: self.n])
        return out, m_new


def fused_kernel(srcs, nks, deterministic, w_slice, m_slice, w_out, m_out, eta, mu, nesterov, agg):
    """fb_fedagg_round_norms_f32 on one rank's slice (clients already in reduction order):
    the fused step plus this shard's share of every round norm (agg.stats[6 + K])."""
    ptrs = (C.c_void_p * len(srcs))(*[t.data_ptr() for t in srcs])
    nk = (C.c_int64 * len(srcs))(*nks)
    ext.call("fb_fedagg_round_norms_f32", ptrs, nk, len(srcs), int(deterministic), w_slice.data_ptr(),
             m_slice.data_ptr(), w_out.data_ptr(), m_out.data_ptr(), w_slice.numel(), float(eta), float(mu),
             int(nesterov), agg.stats.data_ptr(), agg.bad.data_ptr(), ext.stream_handle())


class PeerAggregator:
    """The round-end exchange as ONE kernel over NVLink peer memory (G > 1).

    Every rank keeps its clients' end weights in a symmetric-memory buffer (torch
    symmetric memory: the same allocation mapped into every peer GPU) and the global model
    replica in another. For its shard [lo, hi) a rank runs fb_fedagg_step_f32_peers with
    client k's pointer set to the owning rank's buffer (a peer address for remote clients),
    so the kernel pulls the remote slices straight over NVLink, reduces all K in id order,
    and stores w' to its own replica and to every peer's replica. That single pass replaces
    the NCCL all-to-all, the shard-local kernel and the NCCL all-gather of
    ShardedAggregator, with the same arithmetic in the same order: bit-identical to one GPU.
    Two device-side barriers bracket it (all clients final before the reads; all replicas
    written before w' is used). Momentum stays sharded. NVLink bytes per rank:
    in 4 (N/G) (K - K/G), out 4 (N/G) (G - 1).

    pull="ce": the remote slices are pulled by the copy engines (one stream per peer) into
    a double-buffered local stage, chunk by chunk, overlapped with the kernel on the
    previous chunk (one peer alone: copy engines 740 GB/s, SM loads 670 GB/s per rank,
    tools/nvlink_pull.py). pull="sm": the kernel loads peer memory directly (one launch,
    no stage). pull="auto" (default) picks "ce" at G = 2 and "sm" above, as measured."""

    def __init__(self, n: int, n_clients: int, group=None, device=None, pull: str = "auto", chunk: int = 1 << 25,
                 ce_clients: int | None = None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        if pull not in ("auto", "ce", "sm"):
            raise ValueError(f"pull must be 'auto', 'ce' or 'sm', got {pull!r}")
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = n
        self.K = n_clients
        self.lo, self.hi, self.per = shard_bounds(n, self.world, self.rank)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.slots = (n_clients + self.world - 1) // self.world
        width = self.per * self.world
        grp = group if group is not None else dist.group.WORLD
        # allocate on every rank first and agree before the (collective) rendezvous, so a rank
        # that cannot map symmetric memory makes ALL ranks fall back instead of leaving the
        # others waiting in the rendezvous
        ok = torch.ones(1, dtype=torch.int32, device=dev)
        try:
            self.clients = symm.empty(self.slots, width, dtype=torch.float32, device=dev)
            self.wbuf = symm.empty(width, dtype=torch.float32, device=dev)
        except Exception:
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            raise RuntimeError("symmetric memory unavailable on at least one rank")
        self.hc = symm.rendezvous(self.clients, grp)
        self.hw = symm.rendezvous(self.wbuf, grp)
        self.cptr = [int(p) for p in self.hc.buffer_ptrs]
        self.wptr = [int(p) for p in self.hw.buffer_ptrs]
        # round-norm side reductions of this shard (fb_fedagg_round_norms_f32_peers): 6 fixed + K clients
        self.stats = torch.zeros(6 + n_clients, dtype=torch.float64, device=dev)
        self.bad = torch.full((1,), NO_BAD, dtype=torch.int64, device=dev)  # global index after step()
        self.ids = list(range(n_clients))
        self.width = width
        # peer views of every rank's client slots (for the copy-engine pull)
        self.peer_clients = [self.hc.get_buffer(r, (self.slots, width), torch.float32) for r in range(self.world)]
        # measured at C4 (tools/multi_gpu_check.py): the staged copy-engine pull wins at G = 2
        # (21.75 vs 24.6 ms), the direct SM pull at G = 4 (21.4 vs 28.5 ms: with every rank
        # pulling from 3 peers the copy engines fall behind the SMs' loads)
        self.pull = pull if pull != "auto" else ("ce" if self.world == 2 else "sm")
        self.chunk = int(chunk)
        self.ce_clients = ce_clients  # pull="ce": how many remote clients the copy engines stage (None = all;
        # the rest are loaded by the kernel's SMs straight from peer memory, both in flight at once)
        self.stage = None
        # one copy stream per peer: pulls from different GPUs run on different copy engines
        self.side = {r: torch.cuda.Stream(device=dev) for r in range(self.world) if r != self.rank}

    def exchange(self, local: dict):
        """Stage this rank's clients into their symmetric slots (a local copy; no transfer)."""
        for k, t in local.items():
            buf = self.client_buffer(k)
            if buf.data_ptr() != t.data_ptr():
                buf.copy_(t[: self.n], non_blocking=True)

    def client_buffer(self, k: int):
        """The [N] f32 slot where this rank keeps client k's end weights (k % world == rank)."""
        assert k % self.world == self.rank, (k, self.rank)
        return self.clients[k // self.world, : self.n]

    def step(self, w, m_shard, n_k: dict, eta, mu, nesterov, deterministic=True, w_out=None):
        import torch
        cnt = self.hi - self.lo
        ids = sorted(n_k) if deterministic else list(n_k)
        reps = [self.wptr[r] + 4 * self.lo for r in range(self.world) if r != self.rank]
        m_new = torch.empty_like(m_shard)
        self.ids = ids
        self.stats.zero_()
        self.bad.fill_(NO_BAD)
        self.hc.barrier(channel=0)  # every rank's clients are final
        if cnt > 0 and self.pull == "sm":
            srcs = [self.cptr[k % self.world] + 4 * ((k // self.world) * self.width + self.lo) for k in ids]
            self._launch(srcs, ids, n_k, deterministic, w, m_shard, m_new, reps, 0, cnt, eta, mu, nesterov,
                         self.stats, self.bad)
            self.bad.copy_(_global_bad(self.bad, cnt, self.lo))
        elif cnt > 0:
            self._staged(ids, n_k, deterministic, w, m_shard, m_new, reps, cnt, eta, mu, nesterov)
        self.hc.barrier(channel=1)  # every shard of w' has landed in every replica
        out = w_out if w_out is not None else torch.empty_like(w)
        out.copy_(self.wbuf[: self.n])
        return out, m_new

    def _launch(self, srcs, ids, n_k, deterministic, w, m_shard, m_new, reps, a, b, eta, mu, nesterov, stats, bad):
        wo = self.wbuf[self.lo + a:self.lo + b]
        ext.call("fb_fedagg_round_norms_f32_peers", (C.c_void_p * len(ids))(*srcs),
                 (C.c_int64 * len(ids))(*[int(n_k[k]) for k in ids]), len(ids), int(deterministic),
                 w[self.lo + a:self.lo + b].data_ptr(), m_shard[a:b].data_ptr(), wo.data_ptr(), m_new[a:b].data_ptr(),
                 (C.c_void_p * max(1, len(reps)))(*[p + 4 * a for p in reps]), len(reps), b - a, float(eta),
                 float(mu), int(nesterov), stats.data_ptr(), bad.data_ptr(), ext.stream_handle())

    def _staged(self, ids, n_k, deterministic, w, m_shard, m_new, reps, cnt, eta, mu, nesterov):
        """Copy-engine pull, chunked and double-buffered: a side stream copies the remote
        clients' slices of chunk c+1 (cudaMemcpyAsync from the peer view, measured 740 GB/s
        per rank vs ~430 GB/s for SM loads mixed into the reduction) while the fused kernel
        reduces chunk c from local HBM and stores w' into every replica. Same kernel, same
        client order: bit-identical to the direct pull and to one GPU."""
        import torch
        remote = [k for k in ids if k % self.world != self.rank]
        if self.ce_clients is not None:
            remote = remote[: self.ce_clients]
        ch = min(cnt, self.chunk)
        nch = (cnt + ch - 1) // ch
        if self.stage is None or self.stage.shape[1:] != (len(remote), ch):
            self.stage = torch.empty(2, len(remote), ch, dtype=torch.float32, device=m_shard.device)
        stats = torch.empty(nch, 6 + len(ids), dtype=torch.float64, device=m_shard.device)
        bad = torch.empty(nch, dtype=torch.int64, device=m_shard.device)
        main = torch.cuda.current_stream()
        peers = sorted({k % self.world for k in remote})
        ready = [{r: torch.cuda.Event() for r in peers} for _ in range(2)]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        for r in peers:
            self.side[r].wait_stream(main)  # after the barrier: the peers' clients are final
        slot = {k: i for i, k in enumerate(remote)}
        for c in range(nch):
            a, b, s = c * ch, min(cnt, (c + 1) * ch), c & 1
            for r in peers:
                st = self.side[r]
                with torch.cuda.stream(st):
                    if c >= 2:
                        st.wait_event(done[s])  # kernel c-2 has consumed this buffer
                    for k in remote:
                        if k % self.world == r:
                            src = self.peer_clients[r][k // self.world, self.lo + a:self.lo + b]
                            self.stage[s, slot[k], : b - a].copy_(src, non_blocking=True)
                    ready[s][r].record(st)
                main.wait_event(ready[s][r])
            srcs = [int(self.stage[s, slot[k]].data_ptr()) if k in slot
                    else self.cptr[k % self.world] + 4 * ((k // self.world) * self.width + self.lo + a) for k in ids]
            self._launch(srcs, ids, n_k, deterministic, w, m_shard, m_new, reps, a, b, eta, mu, nesterov,
                         stats[c], bad[c:c + 1])
            done[s].record(main)
        torch.sum(stats, 0, out=self.stats)
        # per-chunk first-bad indices are relative to each launch: offset, then the minimum
        starts = torch.arange(nch, dtype=torch.int64, device=bad.device) * ch
        counts = torch.clamp(cnt - starts, max=ch)
        glob = torch.where(bad < counts, bad + starts + self.lo, torch.full_like(bad, NO_BAD))
        self.bad.copy_(glob.min().reshape(1))
