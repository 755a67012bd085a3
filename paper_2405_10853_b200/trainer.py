"""Client half of the round: `train_round`, the Flower-style `fit`.

Drop-in for fedforge/trainer.py:54-114 (same signature, same TrainTask /
StepTelemetry / ClientUpdate contract, same schedule-offset and cursor
semantics, same errors). Each local step is ONE call into the native runtime
(fb_train_step: device data gather -> micro-batch fwd/bwd on tcgen05 ->
deterministic grad-norm + clip decision -> fused AdamW + bf16 shadow ->
telemetry), so the round runs without host synchronisation; telemetry comes
back in a single device->host copy at the end of the round.
"""
from __future__ import annotations

import collections
import ctypes as C
import math
import os

import numpy as np

from . import ext
from .config import AdamWConfig, ScheduleConfig, StepTelemetry, TrainTask, lr_at
from .data import BatchIterator, DeviceCorpus
from .errors import ParamError, RoundFailedError
from .fedopt import DeviceClientUpdate, DeviceVector
from .model import LossEvaluator, check_gpu_shape
from .params import ParamVector

N_TELE = 8

_corpora: dict = {}


def device_corpus(batches: BatchIterator, device) -> DeviceCorpus:
    key = (id(batches.corpus), str(device))
    dc = _corpora.get(key)
    if dc is None or dc.corpus is not batches.corpus:
        dc = DeviceCorpus(batches.corpus, device)
        _corpora[key] = dc
    return dc


class RoundBuffers:
    """Per-evaluator scratch for the step loop (reused across rounds)."""

    def __init__(self, ev: LossEvaluator):
        import torch
        self.scratch = torch.zeros(3 * ext.FB_RED_BLOCKS + 16, dtype=torch.float64, device=ev.device)
        self.row_loss = None

    def rows(self, n, device):
        import torch
        if self.row_loss is None or self.row_loss.numel() < n:
            self.row_loss = torch.empty(n, dtype=torch.float64, device=device)
        return self.row_loss


# micro-batches per pass, tried largest first (C2 / C3 measured 46.1 / 56.1% of sustained bf16 at 4,
# 47.6 / 57.2% at 8, 48.0 / 57.3% at 16; C4 fits 3)
FUSE_CANDIDATES = tuple(int(x) for x in os.environ.get("FB_FUSE_CANDIDATES", "16,8,4,3,2,1").split(","))


def fused_micro(micro_batches: int, batch_size: int, ws_bytes, budget_bytes: int) -> int:
    """Micro-batches per forward/backward pass (fb_data_desc.fuse): the largest of FUSE_CANDIDATES (at
    most micro_batches) whose activation workspace ws_bytes(rows) fits the budget; when it does not divide
    micro_batches the last pass takes the remainder. Same rows and the same per-token gradient scale,
    hence the same local step; fewer, larger passes (measured at the bench shapes: C4 fuse 2 -3.7%
    step time, fuse 3 a further ~1%; C2 fuse 4 -19%, C3 fuse 4 -11%)."""
    for f in FUSE_CANDIDATES:
        if f <= micro_batches and (f == 1 or ws_bytes(batch_size * f) <= budget_bytes):
            return f
    return 1


class ClientSession:
    """One client's round on the device, step by step (train_round is a thin loop over it).

    begin() places the received global in HBM (no copy if it already is), resets the
    AdamW moments and positions the data cursor; step() enqueues one whole local step.
    Failure detection (trainer.py:89-95, localopt.py:87-88) is asynchronous: each step's
    telemetry row (64 B) is copied to pinned host memory behind the step and checked once
    its event has fired; the host never runs more than `max_lag` steps ahead of the last
    checked one, so a non-finite loss or parameter stops the round within max_lag steps
    and the error names the local step. finish() only waits for the last rows."""

    max_lag = 2
    # activation-workspace budget for fused micro-batches. C4: 62 GB at fuse 2, 93 GB at fuse 3, 123 GB
    # at fuse 4; a 1-GPU 8-client C4 round also holds the model state (24 GB), the 8 client end weights
    # (43 GB) and the round-end buffers (~16 GB) on the 192 GB B200, so fuse 3 leaves ~16 GB. 100 GB
    # also admits C3's whole step (fuse 16: 96.9 GB; +1% vs fuse 8, profiles/r02_c3_fuse_budget.txt)
    fuse_budget = int(float(os.environ.get("FB_FUSE_WS_GB", "100")) * 1e9)

    def __init__(self, evaluator: LossEvaluator, batches: BatchIterator, adamw_cfg: AdamWConfig,
                 sched: ScheduleConfig):
        self.ev, self.batches, self.adamw_cfg, self.sched = evaluator, batches, adamw_cfg, sched
        ext.lib()  # no CPU fallback
        cfg = evaluator.cfg
        self.T = batches.corpus.sequence_len
        if self.T > cfg.context_len:
            raise ParamError(f"sequence length {self.T} exceeds context_len {cfg.context_len}")
        check_gpu_shape(cfg, self.T)
        if batches.corpus.vocab_size > cfg.vocab_size:
            raise ParamError("corpus vocabulary larger than the model's")
        self.dc = device_corpus(batches, evaluator.device)
        self.order = self.dc.order(batches)
        self.opt = ext.AdamWCfg(adamw_cfg.beta1, adamw_cfg.beta2, adamw_cfg.eps, adamw_cfg.weight_decay,
                                adamw_cfg.clip_norm)

    def begin(self, params, task: TrainTask):
        import torch
        if task.local_steps < 1:
            raise ParamError(f"local_steps must be >= 1, got {task.local_steps}")
        if task.batch_size != self.batches.batch_size:
            raise ParamError(f"task batch_size {task.batch_size} != iterator batch_size {self.batches.batch_size}")
        ev = self.ev
        self.task = task
        self.w0 = params.tensor if isinstance(params, DeviceVector) else ev._upload(params)
        self.w = self.w0.clone()
        self.shadow, self.grad, self.m1, self.m2 = ev.buffers()
        self.m1.zero_()
        self.m2.zero_()
        self.st = ext.stream_handle()
        ext.call("fb_cast_bf16", self.w.data_ptr(), self.shadow.data_ptr(), self.w.numel(), self.st)
        B, T = task.batch_size, self.T
        # an evaluator shared out to P concurrent clients carries its share of the budget
        budget = getattr(ev, "fuse_budget", None) or self.fuse_budget
        self.fuse = fused_micro(task.micro_batches, B,
                                lambda rows: int(ext.lib().fb_model_workspace_bytes(C.byref(ev._mcfg), rows, T)),
                                budget)
        self.ws = ev.workspace(B * self.fuse, T, extra=B * self.fuse * T * 4 + 512)
        rb = getattr(ev, "_round_bufs", None)
        if rb is None:
            rb = ev._round_bufs = RoundBuffers(ev)
        self.rb = rb
        self.row_loss = rb.rows(task.micro_batches * B * T, ev.device)
        self.tele = torch.zeros(task.local_steps * N_TELE, dtype=torch.float64, device=ev.device)
        self.tele_host = torch.zeros(task.local_steps, N_TELE, dtype=torch.float64, pin_memory=True)
        self.pending = collections.deque()
        self.lrs = []
        self.batches.seek(task.schedule_offset * task.micro_batches * B)
        return self

    def _check_row(self, s: int) -> None:
        row = self.tele_host[s].numpy()
        if not math.isfinite(float(row[0])):
            raise RoundFailedError(self.task.client_id,
                                   f"non-finite loss in round {self.task.round} at local step {s}")
        if row[5] >= 0:
            raise ParamError(f"non-finite parameters after AdamW step (local step {s}, index {int(row[5])})")

    def poll(self, block_through: int = -1) -> None:
        """Check every finished step's telemetry; wait for the steps <= block_through."""
        while self.pending:
            s, ev = self.pending[0]
            if s <= block_through:
                ev.synchronize()
            elif not ev.query():
                break
            self.pending.popleft()
            self._check_row(s)

    def step(self, s: int) -> None:
        import torch
        self.poll(s - 1 - self.max_lag)
        task, B = self.task, self.task.batch_size
        lr = lr_at(self.sched, task.schedule_offset + s)
        self.lrs.append(lr)
        t = s + 1
        desc = ext.DataDesc(self.dc.tokens.data_ptr(), self.order.data_ptr(), self.order.numel(), self.T, B,
                            task.micro_batches, self.fuse, self.batches.cursor)
        ext.call("fb_train_step", C.byref(self.ev._mcfg), self.w.data_ptr(), self.shadow.data_ptr(),
                 self.grad.data_ptr(), self.m1.data_ptr(), self.m2.data_ptr(), C.byref(desc), self.opt, lr,
                 1.0 - self.adamw_cfg.beta1 ** t, 1.0 - self.adamw_cfg.beta2 ** t,
                 self.tele[(s % self.task.local_steps) * N_TELE:].data_ptr(), self.rb.scratch.data_ptr(),
                 self.row_loss.data_ptr(), self.ws.data_ptr(), self.ws.numel(), self.st)
        self.batches.cursor += task.micro_batches * B
        r = s % self.task.local_steps
        self.tele_host[r].copy_(self.tele[r * N_TELE:(r + 1) * N_TELE], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.pending.append((s, ev))

    def finish(self):
        task = self.task
        S = len(self.lrs)
        self.poll(S)
        tv = self.tele_host.numpy()
        telemetry = []
        for s in range(S):
            loss = float(tv[s, 0])
            telemetry.append(StepTelemetry(task.schedule_offset + s, loss, math.sqrt(tv[s, 1]),
                                           math.sqrt(tv[s, 2]), self.lrs[s], math.sqrt(tv[s, 3])))
        update = DeviceClientUpdate(
            client_id=task.client_id, round=task.round, n_k=self.batches.shard.n_k, w_end=self.w, w_start=self.w0,
            local_metrics={"mean_loss": float(np.mean([x.loss for x in telemetry])),
                           "final_loss": telemetry[-1].loss, "final_param_norm": telemetry[-1].param_norm})
        return update, telemetry


def train_round(params, batches: BatchIterator, evaluator: LossEvaluator, adamw_cfg: AdamWConfig,
                sched: ScheduleConfig, task: TrainTask, *, step_hook=None):
    """Run one client round on the GPU; returns (update, per-step telemetry).

    `params` may be a host ParamVector (uploaded once) or a DeviceVector (fast path:
    no host copy). The returned update keeps the trained weights in HBM
    (DeviceClientUpdate); its f64 `delta` is materialised lazily on access."""
    if task.local_steps < 1:
        raise ParamError(f"local_steps must be >= 1, got {task.local_steps}")
    sess = ClientSession(evaluator, batches, adamw_cfg, sched).begin(params, task)
    for s in range(task.local_steps):
        if step_hook is not None:
            step_hook(s)
        sess.step(s)
    return sess.finish()


def evaluate_mean_ce(evaluator: LossEvaluator, params, corpus, indices: np.ndarray, batch_size: int,
                     max_batches: int) -> float:
    """Server validation (trainer.py:117-135): mean next-token CE over a fixed prefix of the
    validation set, forward-only on the GPU (one upload of params, batches gathered on device)."""
    import torch
    if indices.size == 0:
        raise ParamError("validation set is empty")
    ext.lib()
    w = params.tensor if isinstance(params, DeviceVector) else evaluator._upload(params)
    shadow, _, _, _ = evaluator.buffers()
    st = ext.stream_handle()
    ext.call("fb_cast_bf16", w.data_ptr(), shadow.data_ptr(), w.numel(), st)
    T = corpus.sequence_len
    check_gpu_shape(evaluator.cfg, T)
    dc = DeviceCorpus(corpus, evaluator.device) if not isinstance(corpus, DeviceCorpus) else corpus
    n = min(indices.size, batch_size * max_batches)
    order = torch.from_numpy(np.ascontiguousarray(indices[:n], dtype=np.int64)).to(evaluator.device)
    total, count = 0.0, 0
    sums = []
    for start in range(0, n, batch_size):
        rows = min(batch_size, n - start)
        ws = evaluator.workspace(rows, T, extra=rows * T * 4 + 512)
        need = int(ext.lib().fb_model_workspace_bytes(C.byref(evaluator._mcfg), rows, T))
        off = ((need + 255) // 256) * 256
        tok = ws[off:off + rows * T * 4].view(torch.int32)
        ext.call("fb_gather_batch", dc.tokens.data_ptr(), order[start:].data_ptr(), rows, 0, rows, T,
                 tok.data_ptr(), st)
        rl = torch.empty(rows * T, dtype=torch.float64, device=evaluator.device)
        ext.call("fb_model_fwd_bwd", C.byref(evaluator._mcfg), w.data_ptr(), shadow.data_ptr(), None, tok.data_ptr(),
                 rows, T, 1.0, rl.data_ptr(), 0, ws.data_ptr(), need, st)
        sums.append((rl.sum() / (rows * (T - 1)), rows))
    for mean_t, rows in sums:  # one sync at the end
        total += float(mean_t.item()) * rows
        count += rows
    return total / count
