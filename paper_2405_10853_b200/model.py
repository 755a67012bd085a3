"""TinyLM on the B200: flat device buffers + the native runtime (libfedb200).

Drop-in for fedforge.model.LossEvaluator (model.py:172-250): same manifest
(named_parameters order, model.py:184-190), same seeded init (model.py:123-141,
done on the host with a CPU torch.Generator so it is bit-identical), same
loss / loss_and_grad contract — but forward/backward run as tcgen05 GEMMs,
fused attention, LN and CE kernels on the GPU. There is no CPU path: shapes the
kernels do not implement raise UnsupportedShapeError.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import ext
from .config import TinyLMConfig
from .errors import ParamError, TokenRangeError, UnsupportedShapeError
from .params import ParamVector


@dataclass(frozen=True)
class LayoutEntry:
    tensor_name: str
    shape: tuple
    offset: int

    @property
    def size(self) -> int:
        return int(np.prod(self.shape))


def manifest_entries(cfg: TinyLMConfig) -> tuple:
    V, d = cfg.vocab_size, cfg.d_model
    names = [("embed.weight", (V, d))]
    if not cfg.use_alibi:
        names.append(("pos_embed.weight", (cfg.context_len, d)))
    for i in range(cfg.n_layers):
        b = f"blocks.{i}."
        names += [(b + "ln1.weight", (d,)), (b + "ln1.bias", (d,)), (b + "qkv.weight", (3 * d, d)),
                  (b + "attn_proj.weight", (d, d)), (b + "ln2.weight", (d,)), (b + "ln2.bias", (d,)),
                  (b + "mlp_fc.weight", (4 * d, d)), (b + "mlp_proj.weight", (d, 4 * d))]
    names += [("ln_f.weight", (d,)), ("ln_f.bias", (d,)), ("head.weight", (V, d))]
    out, off = [], 0
    for n, sh in names:
        out.append(LayoutEntry(n, sh, off))
        off += int(np.prod(sh))
    return tuple(out)


def init_params_host(cfg: TinyLMConfig) -> np.ndarray:
    """Seeded init walked in manifest order with one CPU torch.Generator:
    head = 0, residual projections ~ N(0, 0.02/sqrt(2L)), LN w=1 b=0, rest ~ N(0, 0.02)."""
    import torch
    gen = torch.Generator().manual_seed(cfg.seed)
    resid = 0.02 / math.sqrt(2 * cfg.n_layers)
    chunks = []
    for e in manifest_entries(cfg):
        t = torch.empty(e.shape, dtype=torch.float32)
        if e.tensor_name == "head.weight":
            t.zero_()
        elif e.tensor_name.endswith(("attn_proj.weight", "mlp_proj.weight")):
            t.normal_(0.0, resid, generator=gen)
        elif "ln" in e.tensor_name:
            t.fill_(1.0) if e.tensor_name.endswith("weight") else t.zero_()
        else:
            t.normal_(0.0, 0.02, generator=gen)
        chunks.append(t.reshape(-1))
    return torch.cat(chunks).numpy()


def check_gpu_shape(cfg: TinyLMConfig, T: int | None = None) -> None:
    """The kernels' only shape limits: TMA row pitches (d_model, vocab multiples of 8) and a
    head dim <= 256. Attention runs on tcgen05 for dh in {64, 128} with T % 128 == 0 and on
    the fixed-order CUDA-core kernels for every other shape (the reference's desk configs)."""
    dh = cfg.d_model // cfg.n_heads
    why = []
    if cfg.d_model % 8:
        why.append(f"d_model={cfg.d_model} not a multiple of 8")
    if dh > 256:
        why.append(f"head dim {dh} above 256")
    if cfg.vocab_size % 8:
        why.append(f"vocab_size={cfg.vocab_size} not a multiple of 8")
    if why:
        raise UnsupportedShapeError("sm_100a kernels do not implement this shape: " + "; ".join(why))


def set_deterministic(enable: bool = True) -> None:
    """Bitwise-reproducible training (reference tests/test_trainer.py:56-63; the package default,
    FB_DETERMINISTIC=0 opts out at load): the
    tcgen05 attention backward sums its per-key-block dQ slabs in key-block order. False trades
    that for ~1.4% of C4 step time (dQ partials reduce-added in arrival order).
    fb_set_deterministic; process-wide."""
    ext.call("fb_set_deterministic", int(bool(enable)))


def model_cfg_struct(cfg: TinyLMConfig) -> ext.ModelCfg:
    return ext.ModelCfg(cfg.vocab_size, cfg.context_len, cfg.n_layers, cfg.d_model, cfg.n_heads, int(cfg.use_alibi))


def validate_batch(batch: np.ndarray, cfg: TinyLMConfig) -> np.ndarray:
    """model.py:153-169 contract: 2-D, 2 <= T <= ctx, ids in [0, V)."""
    arr = np.ascontiguousarray(batch)
    if arr.ndim != 2:
        raise ParamError(f"batch must be 2-D (B, T), got shape {arr.shape}")
    if arr.shape[1] > cfg.context_len:
        raise ParamError(f"sequence length {arr.shape[1]} exceeds context_len {cfg.context_len}")
    if arr.shape[1] < 2:
        raise ParamError("need at least 2 tokens per row for a next-token target")
    bad = (arr < 0) | (arr >= cfg.vocab_size)
    if bad.any():
        i, t = np.argwhere(bad)[0]
        raise TokenRangeError(f"token id {arr[i, t]} out of range [0, {cfg.vocab_size}) at row {i}, position {t}")
    return arr.astype(np.int32)


class LossEvaluator:
    """Device-resident TinyLM. Not thread-safe (one per worker / stream), like the reference."""

    def __init__(self, cfg: TinyLMConfig, device="cuda"):
        import torch
        self.cfg = cfg
        self.device = torch.device(device)
        self.manifest_entries = manifest_entries(cfg)
        self.n_params = self.manifest_entries[-1].offset + self.manifest_entries[-1].size
        self._mcfg = model_cfg_struct(cfg)
        self._ws = {}
        self._bufs = None

    @property
    def manifest(self):
        return self.manifest_entries

    def init_params(self) -> ParamVector:
        return ParamVector(init_params_host(self.cfg))

    # -- device buffers -------------------------------------------------------------
    def workspace(self, batch: int, T: int, extra: int = 0):
        import torch
        L = ext.lib()
        need = int(L.fb_model_workspace_bytes(C.byref(self._mcfg), batch, T)) + extra
        key = (batch, T)
        ws = self._ws.get(key)
        if ws is None or ws.numel() < need:
            self._ws.clear()
            ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def buffers(self):
        """(shadow bf16, grad f32, m1, m2) sized for this model, reused across calls."""
        import torch
        if self._bufs is None:
            n = self.n_params
            self._bufs = (torch.empty(n, dtype=torch.bfloat16, device=self.device),
                          torch.empty(n, dtype=torch.float32, device=self.device),
                          torch.empty(n, dtype=torch.float32, device=self.device),
                          torch.empty(n, dtype=torch.float32, device=self.device))
        return self._bufs

    def _upload(self, params):
        import torch
        if isinstance(params, torch.Tensor):
            w = params.to(self.device, torch.float32).contiguous()
        else:
            data = params.data if isinstance(params, ParamVector) else np.asarray(params, dtype=np.float32)
            if data.size != self.n_params:
                raise ParamError(f"parameter vector length {data.size} != model size {self.n_params}")
            a = np.ascontiguousarray(data, dtype=np.float32)
            if not a.flags.writeable:  # ParamVector storage is read-only
                a = a.copy()
            w = torch.from_numpy(a).to(self.device)
        if w.numel() != self.n_params:
            raise ParamError(f"parameter vector length {w.numel()} != model size {self.n_params}")
        return w

    def _run(self, params, batch, want_grad):
        import torch
        arr = validate_batch(batch, self.cfg)
        ext.lib()  # raises FedB200Error without the library or a B200: no CPU fallback
        B, T = arr.shape
        check_gpu_shape(self.cfg, T)
        w = self._upload(params)
        shadow, grad, _, _ = self.buffers()
        st = ext.stream_handle()
        ext.call("fb_cast_bf16", w.data_ptr(), shadow.data_ptr(), w.numel(), st)
        tok = torch.from_numpy(arr).to(self.device)
        ws = self.workspace(B, T)
        row_loss = torch.empty(B * T, dtype=torch.float64, device=self.device)
        if want_grad:
            grad.zero_()
        ext.call("fb_model_fwd_bwd", C.byref(self._mcfg), w.data_ptr(), shadow.data_ptr(),
                 grad.data_ptr() if want_grad else None, tok.data_ptr(), B, T, 1.0 / (B * (T - 1)),
                 row_loss.data_ptr(), int(want_grad), ws.data_ptr(), ws.numel(), st)
        loss = float(row_loss.sum().item() / (B * (T - 1)))
        if not math.isfinite(loss):
            raise ParamError(f"non-finite loss {loss}")
        return loss, (grad.cpu().numpy().copy() if want_grad else None)

    def loss(self, params, batch: np.ndarray) -> float:
        return self._run(params, batch, False)[0]

    def loss_and_grad(self, params, batch: np.ndarray):
        return self._run(params, batch, True)
