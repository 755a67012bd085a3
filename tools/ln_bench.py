"""fb_ln_bwd / fb_ln_fwd timing at the C2 / C3 / C4 fused-pass shapes (CUDA events, HBM GB/s of the
algorithmic bytes: bwd reads x, dy, dres and writes dx f32 + bf16 = 18 B per element; fwd 6 B)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
st = ext.stream_handle()
for rows, d in [(65536, 512), (65536, 768), (32768, 2048)]:
    x = torch.randn(rows, d, device="cuda")
    g = torch.randn(d, device="cuda")
    b = torch.randn(d, device="cuda")
    y = torch.empty(rows, d, dtype=torch.bfloat16, device="cuda")
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    dy = torch.randn_like(x)
    dres = torch.randn_like(x)
    dx = torch.empty_like(x)
    dxb = torch.empty(rows, d, dtype=torch.bfloat16, device="cuda")
    dg = torch.zeros(d, device="cuda")
    db = torch.zeros(d, device="cuda")
    work = torch.empty(2 * 592 * d, device="cuda")
    fwd = lambda: ext.call("fb_ln_fwd", x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(), mean.data_ptr(),
                           rstd.data_ptr(), rows, d, st)
    bwd = lambda: ext.call("fb_ln_bwd", x.data_ptr(), g.data_ptr(), mean.data_ptr(), rstd.data_ptr(), dy.data_ptr(),
                           dres.data_ptr(), dx.data_ptr(), dxb.data_ptr(), dg.data_ptr(), db.data_ptr(), work.data_ptr(),
                           rows, d, st)
    res = {"rows": rows, "d": d}
    for name, fn, nb in [("fwd", fwd, 6), ("bwd", bwd, 18)]:
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res[name + "_us"] = round(ms * 1e3, 1)
        res[name + "_gbs"] = round(nb * rows * d / ms / 1e6, 0)
    print(json.dumps(res), flush=True)
