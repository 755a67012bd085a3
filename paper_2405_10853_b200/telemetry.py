"""Round telemetry: drop-in for fedforge.metrics.compute_round_norms (metrics.py:167-215).

Every quantity is a side reduction of the fused aggregation pass
(fb_fedagg_round_norms_f32), so on the fast path the norms cost no extra HBM
traffic; for host-format inputs the vectors are uploaded once and the same
kernel runs in norms-only mode.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import ext
from .errors import ParamError


class MetricsError(ValueError):
    pass


@dataclass(frozen=True)
class RoundNorms:
    global_norm: float
    per_client_norms: dict
    avg_client_norm: float
    momentum_norm: float
    pseudograd_norm: float


def norms_from_stats(stats: np.ndarray, client_ids, momentum_norm: float) -> RoundNorms:
    """stats = [|pg|^2, |w'|^2, |m'|^2, |w|^2, |avg|^2, |w-avg|^2, |w_k|^2 ...] (f64)."""
    return RoundNorms(global_norm=math.sqrt(stats[3]),
                      per_client_norms={cid: math.sqrt(stats[6 + i]) for i, cid in enumerate(client_ids)},
                      avg_client_norm=math.sqrt(stats[4]), momentum_norm=momentum_norm,
                      pseudograd_norm=math.sqrt(stats[5]))


def compute_round_norms(w_global, client_vectors: Sequence, weights: Sequence[float], momentum,
                        client_ids: Optional[Sequence[int]] = None, *, vectors_are_deltas: bool = True) -> RoundNorms:
    """Same contract as the reference: client models are w_global - delta_k (or the
    vectors themselves); avg_client_norm is |sum p_k w_k|; pseudograd = w - sum p_k w_k."""
    import torch
    from .fedopt import _dev
    if len(client_vectors) != len(weights) or not client_vectors:
        raise MetricsError("need one weight per client vector")
    if abs(sum(weights) - 1.0) > 1e-9:
        raise MetricsError(f"client weights must sum to 1, got {sum(weights)}")
    if len(client_vectors) > ext.FB_MAX_CLIENTS:
        raise MetricsError(f"at most {ext.FB_MAX_CLIENTS} clients per call")
    ext.lib()
    ids = list(client_ids) if client_ids is not None else list(range(len(client_vectors)))
    w = _dev(w_global)
    n = w.numel()
    models = []
    for v in client_vectors:
        if isinstance(v, torch.Tensor) and v.dtype == torch.float32:
            t = v.contiguous()
        else:
            arr = v.as_f64() if hasattr(v, "as_f64") else np.asarray(v, dtype=np.float64)
            if arr.size != n:
                raise ParamError(f"client vector length {arr.size} != model length {n}")
            mdl = (w.cpu().numpy().astype(np.float64) - arr) if vectors_are_deltas else arr
            t = torch.from_numpy(mdl.astype(np.float32)).to(w.device)
        models.append(t)
    # weights -> integer-like n_k preserving the ratios (the kernel takes n_k; p_k = n_k / sum)
    scale = 1 << 40
    nks = [max(1, int(round(p * scale))) for p in weights]
    stats = torch.zeros(6 + len(models), dtype=torch.float64, device=w.device)
    m = _dev(momentum)
    ptrs = (C.c_void_p * len(models))(*[t.data_ptr() for t in models])
    ext.call("fb_fedagg_round_norms_f32", ptrs, (C.c_int64 * len(nks))(*nks), len(models), 1, w.data_ptr(),
             w.data_ptr(), None, None, n, 1.0, 0.0, 1, stats.data_ptr(), None, ext.stream_handle())
    mn = float(torch.linalg.vector_norm(m.double()).item())
    return norms_from_stats(stats.cpu().numpy(), ids, mn)
