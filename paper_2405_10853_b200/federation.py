"""One federated round on B200s: the hot path of FederatedRuntime._run_round
(fedforge/cluster.py:367-383 task plan, :490-580 round) without its control plane.

Clients are sharded over ranks (client k on rank k mod G, one process per GPU);
every client on a rank trains with train_round (end weights stay in HBM), then the
round ends with the fused aggregation + outer step (+ round-norm telemetry): on one
GPU directly; on G GPUs as one fused kernel over NVLink peer memory
(dist.PeerAggregator), or, where peers cannot be mapped, the NCCL all-to-all of client
slices + shard-local kernel + all-gather (dist.ShardedAggregator). Bit-identical for
every G. Optional validation pass
(evaluate_mean_ce) and FEDP checkpoint of (global, momentum) on rank 0.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import ext
from .checkpoint import write_checkpoint_async
from .config import AdamWConfig, ScheduleConfig, TinyLMConfig, TrainTask
from .data import BatchIterator, DataSplit, TokenizedCorpus
from .dist import PeerAggregator, ShardedAggregator, clients_of, gather_vector, reduce_round_end
from .errors import ParamError
from .fedopt import AggregatorState, DeviceVector, ServerOptState, server_step_with_norms
from .model import LossEvaluator, init_params_host
from .telemetry import RoundNorms, norms_from_stats  # noqa: F401
from .trainer import evaluate_mean_ce, train_round


@dataclass
class RoundResult:
    round: int
    params: DeviceVector
    opt: ServerOptState
    norms: RoundNorms | None
    client_metrics: dict = field(default_factory=dict)
    telemetry: dict = field(default_factory=dict)
    val_loss: float | None = None
    checkpoint: object | None = None  # AsyncCheckpointWrite on rank 0 (wait() before reading the file)


class Federation:
    def __init__(self, model_cfg: TinyLMConfig, adamw: AdamWConfig, sched: ScheduleConfig, corpus: TokenizedCorpus,
                 split: DataSplit, *, batch_size: int, micro_batches: int, local_steps: int, server_eta: float,
                 server_mu: float, nesterov: bool = True, deterministic: bool = True, data_seed: int = 99,
                 local_step_overrides: dict | None = None, eval_batches: int = 0, concurrent_clients: int = 1):
        import torch
        import torch.distributed as dist
        ext.lib()
        self.cfg, self.adamw, self.sched = model_cfg, adamw, sched
        self.corpus, self.split = corpus, split
        self.B, self.micro, self.S = batch_size, micro_batches, local_steps
        self.eta, self.mu, self.nesterov, self.det = server_eta, server_mu, nesterov, deterministic
        self.overrides = dict(local_step_overrides or {})
        self.eval_batches = eval_batches
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.K = len(split.shards)
        self.mine = clients_of(self.rank, self.world, self.K)
        self.ev = LossEvaluator(model_cfg)
        # concurrent_clients > 1: this rank's clients train P at a time, one host thread + one CUDA
        # stream + one evaluator (buffers, workspace) each; small models leave the GPU partly idle
        # between dependent kernels, and a second client fills it (C2 +13%, C3 +10% at P = 2,
        # tools/concurrent_clients.py). Results are the same as sequential training.
        self.P = max(1, min(int(concurrent_clients), len(self.mine) or 1))
        self.evs = [self.ev] + [LossEvaluator(model_cfg) for _ in range(self.P - 1)]
        if self.P > 1:  # P workspaces live at once: each client gets 1/P of the fused-pass budget
            from .trainer import ClientSession
            for e in self.evs:
                e.fuse_budget = ClientSession.fuse_budget // self.P
        self.streams = [torch.cuda.Stream() for _ in range(self.P)] if self.P > 1 else []
        self.iters = {k: BatchIterator(corpus, split.shards[k], batch_size, data_seed) for k in self.mine}
        self.n_k = {k: split.shards[k].n_k for k in range(self.K)}
        self.agg = None
        self._ckpt = None
        if self.world > 1:  # fused peer-memory round end where NVLink peers map; NCCL exchange otherwise
            try:
                if dist.get_backend() != "nccl":
                    raise RuntimeError("peer memory needs the NCCL (GPU) process group")
                self.agg = PeerAggregator(self.ev.n_params, self.K)
            except Exception:
                self.agg = ShardedAggregator(self.ev.n_params, self.K)

    def _train_concurrent(self, w, task_of, updates, tele, metrics):
        """Worker i trains clients mine[i::P] in order on stream i; train_round's finish() waits
        for its own stream, so a returned update is final. The round end runs on the caller's
        stream, which therefore waits on every worker stream, and the end weights are marked as
        used there (the allocator must not recycle them before the aggregation has read them)."""
        import threading

        import torch
        main = torch.cuda.current_stream()
        errors = []

        def worker(i):
            try:
                with torch.cuda.stream(self.streams[i]):
                    self.streams[i].wait_stream(main)  # w is final
                    for k in self.mine[i::self.P]:
                        u, t = train_round(w, self.iters[k], self.evs[i], self.adamw, self.sched, task_of(k))
                        updates[k], tele[k], metrics[k] = u, t, u.local_metrics
            except BaseException as e:  # re-raised on the caller's thread
                errors.append(e)

        ths = [threading.Thread(target=worker, args=(i,)) for i in range(self.P)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if errors:
            raise errors[0]
        for st in self.streams:
            main.wait_stream(st)
        for u in updates.values():
            u.w_end.record_stream(main)

    def init_state(self):
        import torch
        w = DeviceVector(torch.from_numpy(init_params_host(self.cfg)).cuda())
        if self.agg is not None:
            m = torch.zeros(self.agg.hi - self.agg.lo, dtype=torch.float32, device="cuda")
        else:
            m = torch.zeros(len(w), dtype=torch.float32, device="cuda")
        return w, ServerOptState(DeviceVector(m) if m.numel() else DeviceVector(torch.zeros(1, device="cuda")),
                                 self.eta, self.mu, self.nesterov)

    def run_round(self, w: DeviceVector, opt: ServerOptState, round_num: int, checkpoint_path=None) -> RoundResult:
        import torch
        updates, tele, metrics = {}, {}, {}

        def task_of(k):
            return TrainTask(round_num, k, self.overrides.get(k, self.S), (round_num - 1) * self.S, self.B,
                             self.micro, {"data": 0}, f"round-{round_num}")

        if self.P == 1:
            for k in self.mine:
                u, t = train_round(w, self.iters[k], self.ev, self.adamw, self.sched, task_of(k))
                updates[k], tele[k], metrics[k] = u, t, u.local_metrics
        else:
            self._train_concurrent(w, task_of, updates, tele, metrics)
        if self.agg is None:
            agg = AggregatorState(round_num, len(w), deterministic=self.det)
            for k in sorted(updates):
                agg.accumulate(updates[k])
            w_new, opt_new, norms = server_step_with_norms(opt, w, agg, round_num)
        else:
            import torch.distributed as dist
            self.agg.exchange({k: u.w_end for k, u in updates.items()})
            w_out = torch.empty_like(w.tensor)
            w_full, m_new = self.agg.step(w.tensor, opt.momentum.tensor, self.n_k, self.eta, self.mu, self.nesterov,
                                          deterministic=self.det, w_out=w_out)
            w_new, opt_new = DeviceVector(w_full), ServerOptState(DeviceVector(m_new), self.eta, self.mu, self.nesterov)
            # every shard's side reductions summed, the first non-finite index min-reduced: the same
            # telemetry and the same failure check as one GPU (fedopt.server_step_with_norms)
            s, first_bad = reduce_round_end(self.agg.stats, self.agg.bad)
            if first_bad < len(w):
                raise ParamError(f"non-finite global model after server step in round {round_num} "
                                 f"(first bad index {first_bad})")
            norms = norms_from_stats(s, self.agg.ids, math.sqrt(s[2]))
        val = None
        if self.eval_batches and self.rank == 0 and self.split.validation.size:
            val = evaluate_mean_ce(self.ev, w_new, self.corpus, self.split.validation, self.B, self.eval_batches)
        if checkpoint_path is not None:
            momentum = opt_new.momentum
            if self.agg is not None:  # momentum is sharded: the checkpoint holds the full [N] vector
                momentum = DeviceVector(gather_vector(opt_new.momentum.tensor, len(w_new)))
            if self.rank == 0:
                if self._ckpt is not None:  # at most one checkpoint in flight
                    self._ckpt.wait()
                # D2H copies ordered behind this round on a side stream; CRC32 + file write on a host
                # thread: the next round's first steps overlap the checkpoint (server.py:100-132)
                self._ckpt = write_checkpoint_async(
                    {"round": round_num, "global": w_new, "momentum": momentum,
                     "server_opt": {"eta": self.eta, "mu": self.mu, "nesterov": self.nesterov}}, checkpoint_path)
        return RoundResult(round_num, w_new, opt_new, norms, metrics, tele, val,
                           self._ckpt if checkpoint_path is not None else None)
