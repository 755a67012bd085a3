"""FEDP checkpoint container with an asynchronous device path.

Byte format (the reference's round-boundary container, fedforge/params.py:203-316 and
server.py:100-132; restated here as a format, little endian throughout):

    file    = "FEDP" | version:u32 (= 1) | count:u32 | section * count
    section = name_len:u16 | name (utf-8) | kind:u8 | size:u64 | payload[size] | crc32(payload):u32
    kinds   : 0 f32 vector, 1 u64 scalar, 2 f64 scalar, 3 JSON (sort_keys, utf-8), 4 f64 vector

A section is described once by a `_Section` (its fixed head bytes, its payload as a
buffer, its CRC); the encoder, the file writer and the async path all consume that list.

Device vectors (DeviceVector / CUDA f32 tensors) take the async path: `snapshot()` orders
one D2H copy per vector on a side stream behind the producing stream's work into pinned
host memory and returns at once, so the caller enqueues the next round immediately; the
CRC32 and the file write happen when the copies have landed (`PendingCheckpoint.write`,
or in a background thread with `write_checkpoint_async`). The payload buffers are written
straight to the file; the blob is never concatenated in memory.
"""
from __future__ import annotations

import json
import os
import struct
import tempfile
import threading
import zlib
from dataclasses import dataclass
from typing import Any, Callable, Mapping

import numpy as np

from .errors import ParamError
from .params import ParamVector, require_finite

MAGIC = b"FEDP"
FORMAT_VERSION = 1
KIND_F32_VECTOR, KIND_U64_SCALAR, KIND_F64_SCALAR, KIND_JSON, KIND_F64_VECTOR = 0, 1, 2, 3, 4

_FILE_HEAD = struct.Struct("<4sII")   # magic, version, count
_NAME_LEN = struct.Struct("<H")
_KIND_SIZE = struct.Struct("<BQ")
_CRC32 = struct.Struct("<I")


class CheckpointError(Exception):
    pass


class CheckpointFormatError(CheckpointError):
    pass


class CheckpointVersionError(CheckpointError):
    pass


class CheckpointChecksumError(CheckpointError):
    pass


@dataclass
class _Section:
    name: str
    kind: int
    payload: Any          # bytes, or a host numpy array (read through its buffer)
    ready: Callable[[], None] | None = None  # waits for an in-flight D2H copy

    def head(self) -> bytes:
        nb = self.name.encode("utf-8")
        return _NAME_LEN.pack(len(nb)) + nb + _KIND_SIZE.pack(self.kind, self.nbytes)

    @property
    def nbytes(self) -> int:
        return self.payload.nbytes if isinstance(self.payload, np.ndarray) else len(self.payload)

    def buffer(self) -> memoryview:
        if self.ready is not None:
            self.ready()
            self.ready = None
        p = self.payload
        return memoryview(p).cast("B") if isinstance(p, np.ndarray) else memoryview(p)

    def crc(self) -> bytes:
        return _CRC32.pack(zlib.crc32(self.buffer()) & 0xFFFFFFFF)


def _is_device_f32(value) -> bool:
    t = getattr(value, "tensor", value)
    return type(t).__module__.startswith("torch") and getattr(t, "is_cuda", False) and str(t.dtype) == "torch.float32"


def _scalar_or_json(name: str, value) -> _Section:
    if isinstance(value, bool):  # bool is an int subclass; the format has no boolean kind
        raise ParamError(f"section {name!r}: encode booleans inside a JSON section")
    if isinstance(value, int):
        if value < 0 or value >= 1 << 64:
            raise ParamError(f"section {name!r}: integer {value} out of u64 range")
        return _Section(name, KIND_U64_SCALAR, struct.pack("<Q", value))
    if isinstance(value, float):
        return _Section(name, KIND_F64_SCALAR, struct.pack("<d", value))
    if isinstance(value, (str, dict, list)):
        return _Section(name, KIND_JSON, json.dumps(value, sort_keys=True).encode("utf-8"))
    raise ParamError(f"section {name!r}: unsupported value type {type(value).__name__}")


def _plan(sections: Mapping[str, Any], copy_stream=None) -> list:
    """Describe every section; start the D2H copy of every device vector (async)."""
    out = []
    for name, value in sections.items():
        if len(name.encode("utf-8")) > 0xFFFF:
            raise ParamError(f"section name too long: {name!r}")
        if isinstance(value, ParamVector):
            out.append(_Section(name, KIND_F32_VECTOR, value.data.astype("<f4", copy=False)))
        elif _is_device_f32(value):
            out.append(_device_section(name, getattr(value, "tensor", value), copy_stream))
        elif isinstance(value, np.ndarray):
            if value.dtype != np.float64 or value.ndim != 1:
                raise ParamError(f"array section {name!r} must be a 1-D float64 array")
            require_finite(value, f"section {name!r}")
            out.append(_Section(name, KIND_F64_VECTOR, value.astype("<f8", copy=False)))
        else:
            out.append(_scalar_or_json(name, value))
    return out


def _device_section(name: str, t, copy_stream) -> _Section:
    import torch
    src = t.reshape(-1)
    host = torch.empty(src.numel(), dtype=torch.float32, pin_memory=True)
    producer = torch.cuda.current_stream(src.device)
    stream = copy_stream or torch.cuda.Stream(device=src.device)
    stream.wait_stream(producer)           # the copy sees the round's final values
    with torch.cuda.stream(stream):
        host.copy_(src, non_blocking=True)
        done = torch.cuda.Event()
        done.record(stream)
    src.record_stream(stream)              # keep the device storage alive until the copy ran
    arr = host.numpy()
    return _Section(name, KIND_F32_VECTOR, arr, ready=done.synchronize)


class PendingCheckpoint:
    """A snapshot of sections at the round boundary; device vectors are in flight to
    pinned host memory. `write(path)` / `encode()` wait only for those copies."""

    def __init__(self, sections: Mapping[str, Any], copy_stream=None):
        self._parts = _plan(sections, copy_stream)

    def _chunks(self):
        yield _FILE_HEAD.pack(MAGIC, FORMAT_VERSION, len(self._parts))
        for s in self._parts:
            yield s.head()
            yield s.buffer()
            yield s.crc()

    def encode(self) -> bytes:
        return b"".join(bytes(c) for c in self._chunks())

    def write(self, path) -> int:
        """Atomic: a temp file in the target directory, fsync, rename over `path`."""
        directory = os.path.dirname(os.fspath(path)) or "."
        fd, tmp = tempfile.mkstemp(prefix=".fedp-", dir=directory)
        size = 0
        try:
            with os.fdopen(fd, "wb") as fh:
                for c in self._chunks():
                    size += fh.write(c)
                fh.flush()
                os.fsync(fh.fileno())
            os.replace(tmp, path)
        except BaseException:
            if os.path.exists(tmp):
                os.unlink(tmp)
            raise
        return size


class AsyncCheckpointWrite:
    """Handle of a background checkpoint write (write_checkpoint_async)."""

    def __init__(self, pending: PendingCheckpoint, path):
        self.path = path
        self.nbytes = None
        self.error = None
        self._t = threading.Thread(target=self._run, args=(pending,), daemon=True)
        self._t.start()

    def _run(self, pending):
        try:
            self.nbytes = pending.write(self.path)
        except BaseException as e:  # surfaced by wait()
            self.error = e

    def done(self) -> bool:
        return not self._t.is_alive()

    def wait(self) -> int:
        self._t.join()
        if self.error is not None:
            raise self.error
        return self.nbytes


def snapshot(sections: Mapping[str, Any], copy_stream=None) -> PendingCheckpoint:
    return PendingCheckpoint(sections, copy_stream)


def encode_sections(sections: Mapping[str, Any]) -> bytes:
    return PendingCheckpoint(sections).encode()


def write_checkpoint(sections: Mapping[str, Any], path) -> int:
    """Write now (waits for any device copies); returns the byte length."""
    return PendingCheckpoint(sections).write(path)


def write_checkpoint_async(sections: Mapping[str, Any], path, copy_stream=None) -> AsyncCheckpointWrite:
    """Snapshot now (D2H copies enqueued behind the current stream), write in the background:
    the device can start the next round while the CRC32 and the file write run on the host."""
    return AsyncCheckpointWrite(PendingCheckpoint(sections, copy_stream), path)


# ---------------------------------------------------------------------------------- decode
def _f32_vector(b: memoryview):
    return ParamVector.from_bytes(b)


_DECODE = {
    KIND_F32_VECTOR: _f32_vector,
    KIND_U64_SCALAR: lambda b: struct.unpack("<Q", b)[0],
    KIND_F64_SCALAR: lambda b: struct.unpack("<d", b)[0],
    KIND_JSON: lambda b: json.loads(bytes(b).decode("utf-8")),
    KIND_F64_VECTOR: lambda b: np.frombuffer(b, dtype="<f8").copy(),
}


def _field(view: memoryview, off: int, n: int, what: str) -> memoryview:
    if off + n > len(view):
        raise CheckpointFormatError(f"truncated blob: {what} needs {n} bytes at offset {off}, "
                                    f"only {len(view) - off} left")
    return view[off:off + n]


def decode_sections(raw) -> dict:
    """Parse a container; checks magic, version, every CRC32 and that nothing trails."""
    view = memoryview(raw).cast("B")
    magic, version, count = _FILE_HEAD.unpack(_field(view, 0, _FILE_HEAD.size, "header"))
    if magic != MAGIC:
        raise CheckpointFormatError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if version != FORMAT_VERSION:
        raise CheckpointVersionError(f"unsupported format version {version}")
    off = _FILE_HEAD.size
    out = {}
    for i in range(count):
        (nl,) = _NAME_LEN.unpack(_field(view, off, _NAME_LEN.size, f"section {i} name length"))
        off += _NAME_LEN.size
        name = bytes(_field(view, off, nl, f"section {i} name")).decode("utf-8")
        off += nl
        kind, size = _KIND_SIZE.unpack(_field(view, off, _KIND_SIZE.size, f"kind/size of {name!r}"))
        off += _KIND_SIZE.size
        payload = _field(view, off, size, f"payload of {name!r}")
        off += size
        (crc,) = _CRC32.unpack(_field(view, off, _CRC32.size, f"crc of {name!r}"))
        off += _CRC32.size
        if zlib.crc32(payload) & 0xFFFFFFFF != crc:
            raise CheckpointChecksumError(f"checksum mismatch in section {name!r}")
        dec = _DECODE.get(kind)
        if dec is None:
            raise CheckpointFormatError(f"unknown section kind {kind} in {name!r}")
        out[name] = dec(payload)
    if off != len(view):
        raise CheckpointFormatError(f"{len(view) - off} trailing bytes after the last section")
    return out


def read_checkpoint(path) -> dict:
    with open(path, "rb") as fh:
        return decode_sections(fh.read())
