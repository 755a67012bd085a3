"""Host-side boundary type: the reference's flat parameter vector.

Behaviour contract (fedforge/params.py:59-133): a `ParamVector` is a non-empty, 1-D,
read-only float32 vector, finite unless built with check=False; `require_finite` names the
first offending index; `l2_norm` accumulates in float64. Only callers that cross the
boundary with host arrays see this type; the GPU fast path keeps vectors in HBM
(fedopt.DeviceVector) and computes norms as kernel side reductions.
"""
from __future__ import annotations

import math

import numpy as np

from .errors import ParamError


def require_finite(arr: np.ndarray, what: str = "vector") -> None:
    bad = np.flatnonzero(~np.isfinite(arr))
    if bad.size:
        i = int(bad[0])
        raise ParamError(f"non-finite value {arr[i]!r} in {what} at index {i}")


def _frozen_f32(data) -> np.ndarray:
    a = np.ascontiguousarray(data, dtype=np.float32)
    if a.flags.writeable and a.base is not None:
        a = a.copy()  # never alias a caller's writable buffer
    a.flags.writeable = False
    return a


class ParamVector:
    """Immutable flat float32 vector; share freely across threads."""

    __slots__ = ("_data",)

    def __init__(self, data, *, check: bool = True):
        a = np.ascontiguousarray(data, dtype=np.float32)
        if a.ndim != 1:
            raise ParamError(f"expected a 1-D vector, got shape {a.shape}")
        if not a.size:
            raise ParamError("parameter vector must be non-empty")
        if check:
            require_finite(a, "parameter vector")
        self._data = _frozen_f32(a)

    @classmethod
    def zeros(cls, n: int) -> "ParamVector":
        if n < 1:
            raise ParamError(f"vector length must be positive, got {n}")
        return cls(np.zeros(n, np.float32), check=False)

    @classmethod
    def from_bytes(cls, raw) -> "ParamVector":
        return cls(np.frombuffer(raw, dtype="<f4"))

    data = property(lambda self: self._data, doc="read-only float32 storage")

    def to_bytes(self) -> bytes:
        return self._data.astype("<f4", copy=False).tobytes()

    def as_f64(self) -> np.ndarray:
        return self._data.astype(np.float64)

    def bitwise_equal(self, other: "ParamVector") -> bool:
        a, b = self._data, other._data
        return a.size == b.size and bool((a.view(np.uint32) == b.view(np.uint32)).all())

    def __len__(self) -> int:
        return self._data.size

    def __repr__(self) -> str:
        return f"ParamVector(len={self._data.size})"


def l2_norm(v) -> float:
    """sqrt of the float64 dot product (params.py:126-133)."""
    a = v.data if isinstance(v, ParamVector) else np.asarray(v)
    if not a.size:
        raise ParamError("l2_norm of an empty vector")
    require_finite(a, "l2_norm input")
    x = a.astype(np.float64, copy=False)
    return math.sqrt(float(x @ x))
