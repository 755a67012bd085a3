"""Run whole C4 (or --config) micro-batches fwd+bwd through fb_model_fwd_bwd, for ncu
launch lists / full captures. `--iters` micro-batches after one warm-up."""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from paper_2405_10853_b200 import ext  # noqa: E402
from paper_2405_10853_b200.config import TinyLMConfig  # noqa: E402
from paper_2405_10853_b200.model import LossEvaluator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--iters", type=int, default=1)
a = ap.parse_args()
c = CONFIGS[a.config]
cfg = TinyLMConfig(vocab_size=c["V"], context_len=c["T"], n_layers=c["L"], d_model=c["d"], n_heads=c["H"])
ev = LossEvaluator(cfg)
if os.environ.get("PM_DET"):
    ext.call("fb_set_deterministic", 1)
N = ev.n_params
w = torch.empty(N, device="cuda").normal_(0, 0.02)
shadow, grad, _, _ = ev.buffers()
ext.call("fb_cast_bf16", w.data_ptr(), shadow.data_ptr(), N, ext.stream_handle())
B, T = int(os.environ.get("PM_B", c["B"])), c["T"]
tok = torch.randint(33, 97, (B * T,), dtype=torch.int32, device="cuda")
ws = ev.workspace(B, T)
rl = torch.empty(B * T, dtype=torch.float64, device="cuda")
grad.zero_()
for i in range(1 + a.iters):
    ext.call("fb_model_fwd_bwd", C.byref(ev._mcfg), w.data_ptr(), shadow.data_ptr(), grad.data_ptr(), tok.data_ptr(),
             B, T, 1.0 / (B * (T - 1)), rl.data_ptr(), 1, ws.data_ptr(), ws.numel(), ext.stream_handle())
    torch.cuda.synchronize()
    print("iter", i, "loss", rl.sum().item() / (B * (T - 1)), flush=True)

if os.environ.get("PM_TIME"):
    # back-to-back micro-batches (no host sync in between), device-timed
    n = int(os.environ["PM_TIME"])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        e0.record()
        for i in range(n):
            ext.call("fb_model_fwd_bwd", C.byref(ev._mcfg), w.data_ptr(), shadow.data_ptr(), grad.data_ptr(),
                     tok.data_ptr(), B, T, 1.0 / (B * (T - 1)), rl.data_ptr(), 1, ws.data_ptr(), ws.numel(),
                     ext.stream_handle())
        e1.record()
        torch.cuda.synchronize()
        print(f"rep {rep}: {e0.elapsed_time(e1) / n:.2f} ms per micro-batch over {n}", flush=True)
