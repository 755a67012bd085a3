"""ctypes binding of libfedb200.so (the C ABI in include/fedb200.h).

There is no CPU fallback: if the library is missing or the device is not a
B200 (sm_100), every product entry point raises. ctypes.CDLL releases the GIL
during each call, so client threads can drive separate streams concurrently.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FB_LIB_PATH") or os.path.join(_HERE, "libfedb200.so")  # override: A/B experiments only

FB_OK, FB_BAD_ARG, FB_CUDA_ERROR, FB_NONFINITE, FB_UNSUPPORTED = 0, 1, 2, 3, 4
FB_RED_BLOCKS = 1184
FB_MAX_CLIENTS = 64

EPI = {"bf16": 0, "f32": 1, "acc_f32": 2, "resid_f32": 3, "gelu": 4, "dgelu": 5, "resid_f32_bf16": 6, "bf16_rowdot": 7,
       "ce_exp": 8}

_vp, _i, _i64, _d = C.c_void_p, C.c_int, C.c_int64, C.c_double


class AdamWCfg(C.Structure):
    _fields_ = [("beta1", _d), ("beta2", _d), ("eps", _d), ("weight_decay", _d), ("clip_norm", _d)]


class StepCtl(C.Structure):
    _fields_ = [("lr", _d), ("bc1", _d), ("bc2", _d), ("grad_sumsq", _d), ("clip_scale", _d),
                ("clip_active", C.c_int32), ("pad", C.c_int32)]


# name -> argtypes (every entry returns int)
SIGNATURES = {
    "fb_abi_version": [],
    "fb_device_check": [],
    "fb_fedagg_step_f32": [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _i64, _d, _d, _i, _vp, _vp, _vp, _vp],
    "fb_fedagg_step_f32_peers": [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _i64, _d, _d, _i, _vp, _vp, _vp],
    "fb_fedagg_round_norms_f32_peers": [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _i64, _d, _d, _i, _vp, _vp,
                                        _vp],
    "fb_fedagg_round_norms_f32": [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _i64, _d, _d, _i, _vp, _vp, _vp],
    "fb_fedagg_weighted_sum": [_vp, _i, _vp, _i, _vp, _i64, _vp, _vp],
    "fb_fedagg_step_f64delta": [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _i64, _d, _d, _i, _vp, _vp, _vp, _vp],
    "fb_sumsq_partials": [_vp, _i64, _vp, _vp],
    "fb_sum_partials": [_vp, _i, _vp, _vp],
    "fb_step_prepare": [_vp, _d, _d, _d, _d, _vp, _vp],
    "fb_adamw_step": [_vp, _vp, _vp, _vp, _vp, _i64, AdamWCfg, _vp, _vp, _vp, _vp, _vp],
    "fb_cast_bf16": [_vp, _vp, _i64, _vp],
    "fb_gemm_bf16": [_i, _i, _i, _vp, _i64, _i, _vp, _i64, _i, _vp, _i64, _i, _vp, _vp, _i64, _vp],
    "fb_gemm_bf16_splitk": [_i, _i, _i, _vp, _i64, _i, _vp, _i64, _i, _vp, _i64, _i, _i, _vp, _i64, _vp],
    "fb_embed_fwd": [_vp, _vp, _vp, _vp, _i, _i, _i, _vp],
    "fb_embed_bwd": [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp],
    "fb_embed_bwd_sorted": [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _i64, _vp],
    "fb_set_deterministic": [_i],
    "fb_ln_fwd": [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp],
    "fb_ln_bwd": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp],
    "fb_attn_fwd": [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _vp],
    "fb_attn_bwd": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _vp],
    "fb_attn_bwd_ex": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp],
    "fb_gemm_bf16_rowdot": [_i, _i, _i, _vp, _i64, _i, _vp, _i64, _i, _vp, _i64, _vp, _i64, _vp, _i, _i, _vp],
    "fb_lmhead_ce": [_vp, _vp, _vp, _i, _i, _i, _i, _i, C.c_float, _i, _vp, _vp, _i64, _vp, _vp],
    "fb_gather_batch": [_vp, _vp, _i64, _i64, _i, _i, _vp, _vp],
    "fb_profile_begin": [_i],
    "fb_gemm_set_2sm": [_i],
    "fb_gemm_set_group_m": [_i],
    "fb_profile_end": [_vp],
    "fb_model_fwd_bwd": [_vp, _vp, _vp, _vp, _vp, _i, _i, C.c_float, _vp, _i, _vp, _i64, _vp],
    "fb_train_step": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, AdamWCfg, _d, _d, _d, _vp, _vp, _vp, _vp, _i64, _vp],
}

class ModelCfg(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("ctx", C.c_int32), ("n_layers", C.c_int32), ("d_model", C.c_int32),
                ("n_heads", C.c_int32), ("use_alibi", C.c_int32)]


class DataDesc(C.Structure):
    _fields_ = [("d_corpus", _vp), ("d_order", _vp), ("n_order", _i64), ("seq_len", C.c_int32),
                ("batch", C.c_int32), ("micro", C.c_int32), ("fuse", C.c_int32), ("cursor", _i64)]


_lib = None
_lock = threading.Lock()


class FedB200Error(RuntimeError):
    pass


def lib(require_device: bool = True):
    """Load the library (once). Raises if it is missing: there is no fallback."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise FedB200Error(f"{LIB_PATH} not built; run `python -m paper_2405_10853_b200.build`")
            L = C.CDLL(LIB_PATH)
            for name, args in SIGNATURES.items():
                fn = getattr(L, name, None)
                if fn is None:
                    continue
                fn.argtypes = args
                fn.restype = C.c_int
            for name in ("fb_model_n_params",):
                getattr(L, name).argtypes = [C.POINTER(ModelCfg)]
                getattr(L, name).restype = C.c_int64
            L.fb_model_workspace_bytes.argtypes = [C.POINTER(ModelCfg), _i, _i]
            L.fb_model_workspace_bytes.restype = C.c_int64
            L.fb_embed_bwd_work_bytes.argtypes = [_i, _i]
            L.fb_embed_bwd_work_bytes.restype = C.c_int64
            L.fb_attn_bwd_work_floats.argtypes = [_i, _i, _i, _i]
            L.fb_attn_bwd_work_floats.restype = C.c_int64
            L.fb_lmhead_ce_work_floats.argtypes = [_i, _i]
            L.fb_lmhead_ce_work_floats.restype = C.c_int64
            L.fb_last_error.argtypes = []
            L.fb_last_error.restype = C.c_char_p
            # the reference's bitwise replay semantics (tests/test_trainer.py:56-63) by default:
            # fixed-order dQ in the tensor-core attention backward (1.4% of C4 step time)
            L.fb_set_deterministic(0 if os.environ.get("FB_DETERMINISTIC", "1") == "0" else 1)
            _lib = L
    if require_device:
        _device_ok()
    return _lib


_dev_checked = False


def _device_ok():
    global _dev_checked
    if _dev_checked:
        return
    import torch
    if not torch.cuda.is_available():
        raise FedB200Error("paper_2405_10853_b200 needs a CUDA B200 (sm_100); no CUDA device visible")
    torch.cuda.init()
    rc = _lib.fb_device_check()
    if rc != FB_OK:
        raise FedB200Error(_lib.fb_last_error().decode())
    _dev_checked = True


def check(rc: int, what: str = "") -> None:
    if rc != FB_OK:
        msg = _lib.fb_last_error().decode() if _lib is not None else ""
        raise FedB200Error(f"{what}: status {rc}: {msg}")


def call(name: str, *args) -> None:
    L = lib()
    check(getattr(L, name)(*args), name)


def ptr(t) -> int:
    """Device pointer of a torch tensor (or None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
