"""Oracle: one client round and one federated round on the CPU.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates
  * train_round                 /root/reference/pkg/src/fedforge/trainer.py:54-114
  * FederatedRuntime._run_round aggregation core, cluster.py:367-383 (task plan), :511-514
"""
from __future__ import annotations

import numpy as np

from . import data_ref, localopt_ref, model_ref


def train_round(w0, tokens, seq_len, order, n_k, mcfg, opt, sched, *, local_steps,
                schedule_offset, batch_size, micro_batches):
    """Returns (w_end f32, telemetry rows [(step, loss, raw, applied, lr, pnorm)])."""
    V, ctx, L, d, H, alibi = mcfg
    cursor = schedule_offset * micro_batches * batch_size
    w = np.asarray(w0, dtype=np.float32).copy()
    m1 = np.zeros_like(w)
    m2 = np.zeros_like(w)
    tele = []
    for s in range(local_steps):
        gstep = schedule_offset + s
        lr = localopt_ref.lr_at(*sched, gstep)
        grads, losses = [], []
        for _ in range(micro_batches):
            rows = data_ref.batch_rows(order, cursor, batch_size)
            cursor += batch_size
            batch = data_ref.gather(tokens, seq_len, rows)
            loss, g = model_ref.loss_and_grad(w, batch, V, ctx, L, d, H, alibi)
            grads.append(g)
            losses.append(loss)
        g = localopt_ref.micro_mean(grads)
        g, raw = localopt_ref.clip(g, opt["clip_norm"])
        w, m1, m2, applied = localopt_ref.adamw(
            w, g, m1, m2, s + 1, lr, opt["beta1"], opt["beta2"], opt["eps"], opt["weight_decay"])
        tele.append((gstep, float(np.mean(losses)), raw, applied, lr, localopt_ref.l2_norm(w)))
    return w, tele
