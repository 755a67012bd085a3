"""Oracle: client optimizer pieces (numpy f64 math, f32 storage).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates
  * adamw_step   /root/reference/pkg/src/fedforge/localopt.py:61-96
  * lr_at        /root/reference/pkg/src/fedforge/localopt.py:119-129
  * clip_grad    /root/reference/pkg/src/fedforge/localopt.py:132-143
  * l2_norm      /root/reference/pkg/src/fedforge/params.py:126-133
  * MicrobatchAccumulator.average  localopt.py:146-169
"""
from __future__ import annotations

import math

import numpy as np


def l2_norm(x) -> float:
    a = np.asarray(x).astype(np.float64, copy=False)
    return float(math.sqrt(float(np.dot(a, a))))


def lr_at(base_lr, warmup, t_max, alpha_f, s):
    if s < warmup:
        return base_lr * (s + 1) / warmup
    if s >= t_max:
        return base_lr * alpha_f
    prog = (s - warmup) / (t_max - warmup)
    return base_lr * (alpha_f + (1.0 - alpha_f) * (0.5 * (1.0 + math.cos(math.pi * prog))))


def clip(g32: np.ndarray, max_norm: float):
    raw = l2_norm(g32)
    if raw <= max_norm:
        return g32, raw
    return (g32.astype(np.float64) * (max_norm / raw)).astype(np.float32), raw


def micro_mean(grads):
    acc = np.zeros(np.asarray(grads[0]).size, dtype=np.float64)
    for g in grads:
        acc += np.asarray(g).astype(np.float64)
    return (acc / len(grads)).astype(np.float32)


def adamw(p32, g32, m1_32, m2_32, t, lr, beta1=0.9, beta2=0.95, eps=1e-8, wd=1e-5):
    """Returns (p', m1', m2', ||u||) with the reference's materialisation points."""
    g = g32.astype(np.float64)
    p = p32.astype(np.float64)
    m1 = beta1 * m1_32.astype(np.float64) + (1 - beta1) * g
    m2 = beta2 * m2_32.astype(np.float64) + (1 - beta2) * g * g
    m1h = m1 / (1 - beta1 ** t)
    m2h = m2 / (1 - beta2 ** t)
    u = (lr * (m1h / (np.sqrt(m2h) + eps) + wd * p)).astype(np.float32)
    p_new = (p - u.astype(np.float64)).astype(np.float32)
    return p_new, m1.astype(np.float32), m2.astype(np.float32), l2_norm(u)
