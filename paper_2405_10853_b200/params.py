"""Host-boundary currency: immutable flat f32 vectors with f64-accumulated norms.

Mirrors fedforge/params.py:59-133 (require_finite, ParamVector, l2_norm, axpy) so
callers can hand reference-style vectors to the GPU path and get the same
types back. On the fast path vectors never leave the device; these types only
appear where a reference caller crosses the boundary.
"""
from __future__ import annotations

import math
from typing import Iterable

import numpy as np

from .errors import ParamError


def require_finite(arr: np.ndarray, what: str = "vector") -> None:
    if not np.isfinite(arr).all():
        idx = int(np.argmin(np.isfinite(arr)))
        raise ParamError(f"non-finite value {arr[idx]!r} in {what} at index {idx}")


class ParamVector:
    """Immutable flat float32 parameter vector (read-only numpy storage)."""

    __slots__ = ("_data",)

    def __init__(self, data: Iterable[float] | np.ndarray, *, check: bool = True):
        arr = np.ascontiguousarray(data, dtype=np.float32)
        if arr.ndim != 1:
            raise ParamError(f"expected a 1-D vector, got shape {arr.shape}")
        if arr.size == 0:
            raise ParamError("parameter vector must be non-empty")
        if check:
            require_finite(arr, "parameter vector")
        if arr.flags.writeable:
            arr = arr.copy() if arr.base is not None else arr
            arr.setflags(write=False)
        self._data = arr

    @classmethod
    def zeros(cls, n: int) -> "ParamVector":
        if n <= 0:
            raise ParamError(f"vector length must be positive, got {n}")
        return cls(np.zeros(n, dtype=np.float32), check=False)

    @classmethod
    def from_bytes(cls, raw: bytes) -> "ParamVector":
        return cls(np.frombuffer(raw, dtype="<f4"))

    @property
    def data(self) -> np.ndarray:
        return self._data

    def to_bytes(self) -> bytes:
        return self._data.astype("<f4", copy=False).tobytes()

    def as_f64(self) -> np.ndarray:
        return self._data.astype(np.float64)

    def bitwise_equal(self, other: "ParamVector") -> bool:
        return len(self) == len(other) and bool(np.array_equal(self._data.view(np.uint32), other._data.view(np.uint32)))

    def __len__(self) -> int:
        return int(self._data.size)

    def __repr__(self) -> str:
        return f"ParamVector(len={len(self)})"


def l2_norm(v) -> float:
    arr = v.data if isinstance(v, ParamVector) else np.asarray(v)
    if arr.size == 0:
        raise ParamError("l2_norm of an empty vector")
    require_finite(arr, "l2_norm input")
    a = arr.astype(np.float64, copy=False)
    return float(math.sqrt(float(np.dot(a, a))))
