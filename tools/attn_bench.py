"""Attention kernel timing at the C2/C3/C4 shapes (CUDA events, algorithmic causal FLOPs)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
for B, T, H, dh in [(8, 2048, 16, 128), (8, 2048, 12, 64), (16, 1024, 8, 64)]:
    d = H * dh
    qkv = torch.randn(B * T, 3 * d, device="cuda").to(torch.bfloat16)
    o = torch.empty(B * T, d, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * T, device="cuda")
    live = torch.empty(B * H * (T // 128) * (T // 64), dtype=torch.uint8, device="cuda")
    do = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    work = torch.empty(int(ext.lib().fb_attn_bwd_work_floats(B, T, H, dh)), device="cuda")
    st = ext.stream_handle()
    fwd = lambda: ext.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), live.data_ptr(), B, T, H, dh, 1, st)
    bwd = lambda: ext.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), live.data_ptr(), dqkv.data_ptr(),
                           work.data_ptr(), B, T, H, dh, 1, st)
    res = {"B": B, "T": T, "H": H, "dh": dh}
    fl = 2.0 * B * H * dh * T * (T + 1)  # causal fwd (QK^T + PV, lower triangle)
    for name, fn, f in [("fwd", fwd, fl), ("bwd", bwd, 2 * fl)]:
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res[name + "_ms"] = round(ms, 3)
        res[name + "_tflops"] = round(f / ms / 1e9, 1)
    print(json.dumps(res), flush=True)
