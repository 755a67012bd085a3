"""Oracle: pseudo-gradient aggregation and the server outer step (numpy f64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates
  * AggregatorState.accumulate / finalize   /root/reference/pkg/src/fedforge/fedopt.py:84-99, :129-144
  * server_step                             /root/reference/pkg/src/fedforge/fedopt.py:167-201
"""
from __future__ import annotations

import numpy as np


def weighted_terms(w_global: np.ndarray, client_weights, n_ks):
    """n_k * (f64(w) - f64(w_k)) for each client (fedopt.py:95 with trainer.py:352)."""
    g = w_global.astype(np.float64)
    return [int(n) * (g - wk.astype(np.float64)) for wk, n in zip(client_weights, n_ks)]


def finalize_deltas(deltas, n_ks, client_ids=None, deterministic=True):
    """Weighted mean of f64 deltas exactly as fedopt.py:129-144 computes it.

    deterministic: sort by client id, pairwise tree (left+right, odd tail carried),
    divide by the integer total. streaming: running sum in the given order.
    A single contribution is returned unchanged (fedopt.py:133-134).
    """
    if len(deltas) == 0:
        raise ValueError("empty aggregation")
    ids = list(range(len(deltas))) if client_ids is None else list(client_ids)
    total = int(sum(int(n) for n in n_ks))
    if len(deltas) == 1:
        return np.array(deltas[0], dtype=np.float64, copy=True)
    if deterministic:
        order = sorted(range(len(deltas)), key=lambda i: ids[i])
        terms = [int(n_ks[i]) * np.asarray(deltas[i], dtype=np.float64) for i in order]
        while len(terms) > 1:
            nxt = []
            for i in range(0, len(terms) - 1, 2):
                nxt.append(terms[i] + terms[i + 1])
            if len(terms) % 2 == 1:
                nxt.append(terms[-1])
            terms = nxt
        return terms[0] / total
    acc = np.zeros_like(np.asarray(deltas[0], dtype=np.float64))
    for d, n in zip(deltas, n_ks):
        acc += int(n) * np.asarray(d, dtype=np.float64)
    return acc / total


def server_step(w: np.ndarray, m: np.ndarray, delta: np.ndarray, eta: float, mu: float,
                nesterov: bool = True):
    """One outer step (fedopt.py:189-196): f64 math, momentum rounded to f32 first."""
    delta = np.asarray(delta, dtype=np.float64)
    m_new64 = mu * m.astype(np.float64) + delta
    with np.errstate(over="ignore", invalid="ignore"):
        m_new = m_new64.astype(np.float32)
        if nesterov:
            upd = eta * (mu * m_new.astype(np.float64) + delta)
        else:
            upd = eta * m_new.astype(np.float64)
        w_new = (w.astype(np.float64) - upd).astype(np.float32)
    return w_new, m_new


def fed_round(w, m, client_weights, n_ks, eta, mu, nesterov=True, client_ids=None,
              deterministic=True):
    """finalize(deterministic) o server_step on client end-weights (cluster.py:511-514)."""
    g = w.astype(np.float64)
    deltas = [g - wk.astype(np.float64) for wk in client_weights]
    pg = finalize_deltas(deltas, n_ks, client_ids, deterministic)
    return server_step(w, m, pg, eta, mu, nesterov)
