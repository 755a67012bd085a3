"""FEDP checkpoint container (byte-compatible with fedforge/params.py:203-316).

`magic "FEDP" | u32 version 1 | u32 count`, then per section
`u16 name_len | name | u8 kind | u64 payload_len | payload | u32 crc32(payload)`,
kinds 0 f32 vector, 1 u64, 2 f64, 3 JSON (sorted keys), 4 f64 vector.
Device vectors (DeviceVector / CUDA tensors) are copied to pinned host memory
with one async D2H each at the round boundary; the CRC32 runs on the host.
"""
from __future__ import annotations

import json
import os
import struct
import tempfile
import zlib
from typing import Any, Mapping

import numpy as np

from .errors import ParamError
from .params import ParamVector, require_finite

MAGIC = b"FEDP"
FORMAT_VERSION = 1
KIND_F32_VECTOR, KIND_U64_SCALAR, KIND_F64_SCALAR, KIND_JSON, KIND_F64_VECTOR = 0, 1, 2, 3, 4
_HEADER = struct.Struct("<4sII")
_NAME = struct.Struct("<H")
_META = struct.Struct("<BQ")
_CRC = struct.Struct("<I")


class CheckpointError(Exception):
    pass


class CheckpointFormatError(CheckpointError):
    pass


class CheckpointVersionError(CheckpointError):
    pass


class CheckpointChecksumError(CheckpointError):
    pass


def _host_f32(value) -> np.ndarray | None:
    """f32 host array for ParamVector / DeviceVector / f32 CUDA tensor, else None."""
    if isinstance(value, ParamVector):
        return value.data
    if hasattr(value, "tensor"):  # DeviceVector
        value = value.tensor
    try:
        import torch
        if isinstance(value, torch.Tensor) and value.dtype == torch.float32:
            host = torch.empty(value.numel(), dtype=torch.float32, pin_memory=value.is_cuda)
            host.copy_(value.reshape(-1), non_blocking=True)
            if value.is_cuda:
                torch.cuda.current_stream().synchronize()
            return host.numpy()
    except ImportError:
        pass
    return None


def _section(name: str, value) -> bytes:
    nb = name.encode("utf-8")
    if len(nb) > 0xFFFF:
        raise ParamError(f"section name too long: {name!r}")
    f32 = _host_f32(value)
    if f32 is not None:
        kind, payload = KIND_F32_VECTOR, f32.astype("<f4", copy=False).tobytes()
    elif isinstance(value, np.ndarray):
        if value.dtype != np.float64 or value.ndim != 1:
            raise ParamError(f"array section {name!r} must be a 1-D float64 array")
        require_finite(value, f"section {name!r}")
        kind, payload = KIND_F64_VECTOR, value.astype("<f8", copy=False).tobytes()
    elif isinstance(value, bool):
        raise ParamError(f"section {name!r}: encode booleans inside a JSON section")
    elif isinstance(value, int):
        if not 0 <= value < 2 ** 64:
            raise ParamError(f"section {name!r}: integer {value} out of u64 range")
        kind, payload = KIND_U64_SCALAR, struct.pack("<Q", value)
    elif isinstance(value, float):
        kind, payload = KIND_F64_SCALAR, struct.pack("<d", value)
    elif isinstance(value, (str, dict, list)):
        kind, payload = KIND_JSON, json.dumps(value, sort_keys=True).encode("utf-8")
    else:
        raise ParamError(f"section {name!r}: unsupported value type {type(value).__name__}")
    return b"".join([_NAME.pack(len(nb)), nb, _META.pack(kind, len(payload)), payload,
                     _CRC.pack(zlib.crc32(payload) & 0xFFFFFFFF)])


def encode_sections(sections: Mapping[str, Any]) -> bytes:
    return _HEADER.pack(MAGIC, FORMAT_VERSION, len(sections)) + b"".join(_section(k, v) for k, v in sections.items())


def decode_sections(raw: bytes) -> dict:
    pos = 0

    def take(n, what):
        nonlocal pos
        if pos + n > len(raw):
            raise CheckpointFormatError(f"truncated blob: needed {n} bytes for {what} at offset {pos}")
        out = raw[pos:pos + n]
        pos += n
        return out

    magic, version, count = _HEADER.unpack(take(_HEADER.size, "header"))
    if magic != MAGIC:
        raise CheckpointFormatError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if version != FORMAT_VERSION:
        raise CheckpointVersionError(f"unsupported format version {version}")
    out = {}
    for _ in range(count):
        (nl,) = _NAME.unpack(take(_NAME.size, "name length"))
        name = take(nl, "name").decode("utf-8")
        kind, plen = _META.unpack(take(_META.size, "section meta"))
        payload = take(plen, f"payload of {name!r}")
        (crc,) = _CRC.unpack(take(_CRC.size, f"crc of {name!r}"))
        if zlib.crc32(payload) & 0xFFFFFFFF != crc:
            raise CheckpointChecksumError(f"checksum mismatch in section {name!r}")
        if kind == KIND_F32_VECTOR:
            out[name] = ParamVector.from_bytes(payload)
        elif kind == KIND_U64_SCALAR:
            out[name] = struct.unpack("<Q", payload)[0]
        elif kind == KIND_F64_SCALAR:
            out[name] = struct.unpack("<d", payload)[0]
        elif kind == KIND_JSON:
            out[name] = json.loads(payload.decode("utf-8"))
        elif kind == KIND_F64_VECTOR:
            out[name] = np.frombuffer(payload, dtype="<f8").copy()
        else:
            raise CheckpointFormatError(f"unknown section kind {kind} in {name!r}")
    if pos != len(raw):
        raise CheckpointFormatError(f"{len(raw) - pos} trailing bytes after last section")
    return out


def write_checkpoint(sections: Mapping[str, Any], path) -> int:
    """Atomic write: temp file, fsync, os.replace (params.py:292-311)."""
    blob = encode_sections(sections)
    directory = os.path.dirname(os.fspath(path)) or "."
    fd, tmp = tempfile.mkstemp(prefix=".ckpt-", dir=directory)
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(blob)
            fh.flush()
            os.fsync(fh.fileno())
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise
    return len(blob)


def read_checkpoint(path) -> dict:
    with open(path, "rb") as fh:
        return decode_sections(fh.read())
