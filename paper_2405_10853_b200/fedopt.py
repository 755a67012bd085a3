"""Server half of the round: pseudo-gradient aggregation and the outer optimizer.

Drop-in for fedforge/fedopt.py: ClientUpdate (:26-46), client_weight (:49-55),
AggregatorState (:58-144) and ServerOptState / server_step (:147-201) with the
same signatures, validation and error types. The arithmetic runs in one fused
sm_100a kernel (fb_fedagg_step_*): every client vector and w, m are streamed
once, the f64 pairwise tree / running sum and the f64 outer step happen in
registers, and m' is rounded to f32 before it feeds w' — bit-identical to the
reference's numpy for the same inputs.

Fast path: clients that trained on the GPU hand over DeviceClientUpdate objects
(end weights resident in HBM); finalize() then returns a lazy PseudoGradient and
server_step() fuses delta + weighted mean + outer step in a single HBM pass.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

from . import ext
from .errors import AggregationError, ParamError
from .params import ParamVector, require_finite


def _torch():
    import torch
    return torch


class DeviceVector:
    """A flat f32 vector resident in HBM with the read-side ParamVector API."""

    __slots__ = ("tensor",)

    def __init__(self, tensor):
        t = _torch()
        if tensor.dtype != t.float32 or tensor.dim() != 1 or not tensor.is_cuda:
            raise ParamError("DeviceVector needs a 1-D float32 CUDA tensor")
        self.tensor = tensor.contiguous()

    @property
    def data(self) -> np.ndarray:
        a = self.tensor.cpu().numpy()
        a.setflags(write=False)
        return a

    def as_f64(self) -> np.ndarray:
        return self.tensor.cpu().numpy().astype(np.float64)

    def to_param_vector(self) -> ParamVector:
        return ParamVector(self.tensor.cpu().numpy(), check=False)

    def bitwise_equal(self, other) -> bool:
        return np.array_equal(self.data.view(np.uint32), np.asarray(other.data).view(np.uint32))

    def __len__(self) -> int:
        return int(self.tensor.numel())


def _dev(v, device="cuda"):
    """f32 device tensor for a ParamVector / DeviceVector / numpy / tensor."""
    t = _torch()
    if isinstance(v, DeviceVector):
        return v.tensor
    if isinstance(v, t.Tensor):
        return v.to(device=device, dtype=t.float32).contiguous()
    data = v.data if isinstance(v, ParamVector) else np.asarray(v, dtype=np.float32)
    a = np.ascontiguousarray(data, dtype=np.float32)
    if not a.flags.writeable:  # ParamVector storage is read-only; torch wants a writable host buffer
        a = a.copy()
    return t.from_numpy(a).to(device)


@dataclass
class ClientUpdate:
    """Host-format contribution: delta = received - trained weights, float64."""

    client_id: int
    round: int
    n_k: int
    delta: np.ndarray
    local_metrics: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.n_k < 1:
            raise ParamError(f"client {self.client_id}: n_k must be >= 1, got {self.n_k}")
        self.delta = np.ascontiguousarray(self.delta, dtype=np.float64)
        if self.delta.ndim != 1 or self.delta.size == 0:
            raise ParamError(f"client {self.client_id}: delta must be a non-empty 1-D vector")
        require_finite(self.delta, f"delta of client {self.client_id}")

    @property
    def length(self) -> int:
        return int(self.delta.size)


class DeviceClientUpdate:
    """GPU-resident contribution: the client's end weights w_k in HBM plus the global
    it started from. `delta` (f64 host array) is materialised only on access."""

    def __init__(self, client_id: int, round: int, n_k: int, w_end, w_start, local_metrics=None):
        if n_k < 1:
            raise ParamError(f"client {client_id}: n_k must be >= 1, got {n_k}")
        self.client_id = client_id
        self.round = round
        self.n_k = int(n_k)
        self.w_end = w_end      # torch f32 [N] on the device
        self.w_start = w_start  # torch f32 [N] on the device (the received global)
        self.local_metrics = dict(local_metrics or {})
        self._delta = None

    @property
    def length(self) -> int:
        return int(self.w_end.numel())

    @property
    def delta(self) -> np.ndarray:
        if self._delta is None:
            d = self.w_start.cpu().numpy().astype(np.float64) - self.w_end.cpu().numpy().astype(np.float64)
            require_finite(d, f"delta of client {self.client_id}")
            self._delta = d
        return self._delta


def client_weight(n_k: int, n_total: int) -> float:
    if n_total == 0:
        raise ParamError("total sample count is zero")
    if not 1 <= n_k <= n_total:
        raise ParamError(f"n_k={n_k} outside [1, {n_total}]")
    return n_k / n_total


class PseudoGradient:
    """Lazy result of AggregatorState.finalize(): numpy-compatible (np.asarray
    materialises the f64 vector on the GPU and copies it back), but server_step
    consumes it without ever leaving the device."""

    def __init__(self, agg: "AggregatorState"):
        self._agg = agg
        self._host = None

    @property
    def size(self) -> int:
        return self._agg.model_len

    @property
    def shape(self):
        return (self._agg.model_len,)

    dtype = np.dtype(np.float64)
    ndim = 1

    def __len__(self):
        return self._agg.model_len

    def __array__(self, dtype=None, copy=None):
        if self._host is None:
            self._host = self._agg._materialize()
        return self._host if dtype is None else self._host.astype(dtype)

    def __getitem__(self, i):
        return np.asarray(self)[i]


class AggregatorState:
    """Weighted aggregation of one round's contributions (streaming or deterministic).

    Streaming mode sums in arrival order; deterministic mode reduces with a pairwise
    tree in client-id order at finalize (bit-identical for any arrival order). Both
    are evaluated by the fused GPU kernel at finalize/server_step time."""

    def __init__(self, round_num: int, model_len: int, *, deterministic: bool = False):
        if model_len <= 0:
            raise ParamError(f"model_len must be positive, got {model_len}")
        self.round = round_num
        self.model_len = model_len
        self.deterministic = deterministic
        self.total_weight = 0
        self.contributors: set = set()
        self._updates: list = []

    def accumulate(self, update) -> "AggregatorState":
        if update.round != self.round:
            raise AggregationError(f"round mismatch: aggregator at {self.round}, update from {update.round}")
        if update.client_id in self.contributors:
            raise AggregationError(f"duplicate contribution from client {update.client_id}")
        if update.length != self.model_len:
            raise ParamError(f"delta length {update.length} != model length {self.model_len}")
        self.total_weight += update.n_k
        self.contributors.add(update.client_id)
        self._updates.append(update)
        return self

    def merge(self, other: "AggregatorState") -> "AggregatorState":
        if other.round != self.round:
            raise AggregationError(f"round mismatch in merge: {self.round} vs {other.round}")
        if other.model_len != self.model_len:
            raise ParamError("model length mismatch in merge")
        overlap = self.contributors & other.contributors
        if overlap:
            raise AggregationError(f"overlapping contributors in merge: {sorted(overlap)}")
        out = AggregatorState(self.round, self.model_len, deterministic=self.deterministic)
        out.total_weight = self.total_weight + other.total_weight
        out.contributors = self.contributors | other.contributors
        out._updates = self._updates + other._updates
        return out

    @property
    def updates(self) -> list:
        return list(self._updates)

    @property
    def weighted_sum(self) -> np.ndarray:
        """sum_k n_k * delta_k (f64) in arrival order: bitwise the reference's running sum
        (fedopt.py:95), evaluated on the device (fb_fedagg_weighted_sum)."""
        if not self._updates:
            return np.zeros(self.model_len)
        t = _torch()
        ext.lib()
        ups = list(self._updates)  # arrival order, whatever the finalize mode
        dev = [u for u in ups if isinstance(u, DeviceClientUpdate)]
        if len(dev) == len(ups) and len({u.w_start.data_ptr() for u in ups}) == 1:
            srcs, f64, w = [u.w_end for u in ups], 0, ups[0].w_start
        else:
            srcs, f64, w = [t.from_numpy(u.delta).cuda() for u in ups], 1, None
        out = t.empty(self.model_len, dtype=t.float64, device="cuda")
        ext.call("fb_fedagg_weighted_sum", (C.c_void_p * len(srcs))(*[x.data_ptr() for x in srcs]), f64,
                 (C.c_int64 * len(ups))(*[u.n_k for u in ups]), len(ups), ext.ptr(w), self.model_len,
                 out.data_ptr(), ext.stream_handle())
        return out.cpu().numpy()

    def weights(self) -> dict:
        if not self.contributors:
            return {}
        return {u.client_id: u.n_k / self.total_weight for u in self._updates}

    def finalize(self) -> PseudoGradient:
        if not self.contributors:
            raise AggregationError(f"finalize on empty aggregator for round {self.round}")
        return PseudoGradient(self)

    # -- device plumbing --------------------------------------------------------------
    def _ordered(self):
        if self.deterministic:
            return sorted(self._updates, key=lambda u: u.client_id)
        return list(self._updates)

    def _sources(self, device="cuda"):
        """(kind, [device tensors], w_ref) — f32 end weights sharing one global, or f64 deltas."""
        t = _torch()
        ups = self._ordered()
        if len(ups) > ext.FB_MAX_CLIENTS:
            raise AggregationError(f"at most {ext.FB_MAX_CLIENTS} contributions per fused launch")
        dev = [u for u in ups if isinstance(u, DeviceClientUpdate)]
        if len(dev) == len(ups):
            starts = {u.w_start.data_ptr() for u in ups}
            if len(starts) == 1:
                return "f32", [u.w_end for u in ups], ups[0].w_start
        return "f64", [t.from_numpy(u.delta).to(device) for u in ups], None

    def _launch(self, w, m, w_out, m_out, eta, mu, nesterov, pg_out=None, stats=None, bad=None):
        kind, srcs, w_ref = self._sources(w.device if w is not None else "cuda")
        t = _torch()
        if w is None:  # pseudo-gradient only: any w works for the f64-delta form
            w = w_ref if w_ref is not None else t.zeros(self.model_len, dtype=t.float32, device="cuda")
            m = w
        elif kind == "f32" and w_ref.data_ptr() != w.data_ptr() and not t.equal(w_ref, w):
            kind, srcs = "f64", [t.from_numpy(u.delta).to(w.device) for u in self._ordered()]
        ptrs = (C.c_void_p * len(srcs))(*[s.data_ptr() for s in srcs])
        nks = (C.c_int64 * len(srcs))(*[u.n_k for u in self._ordered()])
        fn = "fb_fedagg_step_f32" if kind == "f32" else "fb_fedagg_step_f64delta"
        ext.call(fn, ptrs, nks, len(srcs), int(self.deterministic), w.data_ptr(), m.data_ptr(),
                 ext.ptr(w_out), ext.ptr(m_out), self.model_len, float(eta), float(mu), int(nesterov),
                 ext.ptr(stats), ext.ptr(bad), ext.ptr(pg_out), ext.stream_handle())
        return srcs  # keep alive until the stream has consumed them

    def _pg_device(self):
        t = _torch()
        ext.lib()
        pg = t.empty(self.model_len, dtype=t.float64, device="cuda")
        srcs = self._launch(None, None, None, None, 1.0, 0.0, False, pg_out=pg)
        t.cuda.current_stream().synchronize()
        del srcs
        return pg

    def _materialize(self) -> np.ndarray:
        return self._pg_device().cpu().numpy()


@dataclass
class ServerOptState:
    """Server-side (Nesterov) momentum over the pseudo-gradient stream."""

    momentum: object  # ParamVector (host) or DeviceVector (HBM)
    eta: float
    mu: float
    nesterov: bool = True

    def __post_init__(self):
        if self.eta <= 0:
            raise ParamError(f"server eta must be > 0, got {self.eta}")
        if not 0 <= self.mu < 1:
            raise ParamError(f"server mu must be in [0, 1), got {self.mu}")

    @classmethod
    def fresh(cls, model_len: int, eta: float, mu: float, nesterov: bool = True) -> "ServerOptState":
        return cls(ParamVector.zeros(model_len), eta, mu, nesterov)


def server_step(opt: ServerOptState, w_prev, delta, round_num: Optional[int] = None):
    """m' = mu m + delta ; Nesterov w' = w - eta (mu m' + delta), plain w' = w - eta m'.

    Same contract as the reference (f64 math, m' materialised to f32 first). If
    `delta` is the PseudoGradient of a GPU aggregator the whole aggregation is fused
    into this one kernel. Host ParamVector inputs give host outputs; DeviceVector
    inputs stay in HBM."""
    t = _torch()
    n = len(w_prev)
    ext.lib()  # no CPU fallback
    if len(opt.momentum) != n or len(delta) != n:
        raise ParamError(f"server_step length mismatch: w={n}, delta={len(delta)}, momentum={len(opt.momentum)}")
    on_device = isinstance(w_prev, DeviceVector)
    w = _dev(w_prev)
    m = _dev(opt.momentum)
    w_out = t.empty_like(w)
    m_out = t.empty_like(m)
    bad = t.empty(1, dtype=t.int64, device=w.device)
    stats = t.empty(3, dtype=t.float64, device=w.device)
    if isinstance(delta, PseudoGradient):
        keep = delta._agg._launch(w, m, w_out, m_out, opt.eta, opt.mu, opt.nesterov, stats=stats, bad=bad)
    else:
        d = np.ascontiguousarray(delta, dtype=np.float64)
        dd = t.from_numpy(d).to(w.device)
        keep = [dd]
        ptrs = (C.c_void_p * 1)(dd.data_ptr())
        ext.call("fb_fedagg_step_f64delta", ptrs, (C.c_int64 * 1)(1), 1, 1, w.data_ptr(), m.data_ptr(),
                 w_out.data_ptr(), m_out.data_ptr(), n, float(opt.eta), float(opt.mu), int(opt.nesterov),
                 stats.data_ptr(), bad.data_ptr(), None, ext.stream_handle())
    first_bad = int(bad.item())  # one 8-byte D2H per round
    del keep
    if first_bad < n:
        if not np.isfinite(w_out[first_bad].item()):
            where = f" in round {round_num}" if round_num is not None else ""
            raise ParamError(f"non-finite global model after server step{where}")
        raise ParamError(f"non-finite value {m_out[first_bad].item()!r} in server momentum at index {first_bad}")
    if on_device:
        return DeviceVector(w_out), replace(opt, momentum=DeviceVector(m_out))
    return (ParamVector(w_out.cpu().numpy(), check=False),
            replace(opt, momentum=ParamVector(m_out.cpu().numpy(), check=False)))


def server_step_with_norms(opt: ServerOptState, w_prev, agg: AggregatorState, round_num: Optional[int] = None):
    """Fast path of FederatedRuntime._run_round (cluster.py:511-520): finalize + server_step +
    compute_round_norms in ONE pass over HBM. Returns (w', opt', RoundNorms)."""
    from .telemetry import norms_from_stats
    t = _torch()
    ext.lib()
    n = len(w_prev)
    kind, srcs, w_ref = agg._sources()
    if kind != "f32":
        raise ParamError("server_step_with_norms needs device-resident client updates sharing one global")
    w = _dev(w_prev)
    m = _dev(opt.momentum)
    w_out, m_out = t.empty_like(w), t.empty_like(m)
    ups = agg._ordered()
    stats = t.zeros(6 + len(ups), dtype=t.float64, device=w.device)
    bad = t.empty(1, dtype=t.int64, device=w.device)
    ptrs = (C.c_void_p * len(srcs))(*[s_.data_ptr() for s_ in srcs])
    nks = (C.c_int64 * len(ups))(*[u.n_k for u in ups])
    ext.call("fb_fedagg_round_norms_f32", ptrs, nks, len(ups), int(agg.deterministic), w.data_ptr(), m.data_ptr(),
             w_out.data_ptr(), m_out.data_ptr(), n, float(opt.eta), float(opt.mu), int(opt.nesterov),
             stats.data_ptr(), bad.data_ptr(), ext.stream_handle())
    st = stats.cpu().numpy()
    if int(bad.item()) < n:
        where = f" in round {round_num}" if round_num is not None else ""
        raise ParamError(f"non-finite global model after server step{where}")
    norms = norms_from_stats(st, [u.client_id for u in ups], float(np.sqrt(st[2])))
    return DeviceVector(w_out), replace(opt, momentum=DeviceVector(m_out)), norms
