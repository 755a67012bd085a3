"""A/B of attention-backward library variants at the C4 / C3 shapes: `python tools/attn_bwd_ab.py
lib1.so lib2.so ...` (each via FB_LIB_PATH in a subprocess), interleaved repetitions, CUDA events."""
import json
import os
import subprocess
import sys

CHILD = r"""
import json, os, sys, torch
sys.path.insert(0, os.environ["ROOT"])
from paper_2405_10853_b200 import ext
ext.lib()
out = {}
for B, T, H, dh in [(16, 2048, 16, 128), (16, 2048, 12, 64)]:
    d = H * dh
    torch.manual_seed(0)
    qkv = torch.randn(B * T, 3 * d, device="cuda").to(torch.bfloat16)
    o = torch.empty(B * T, d, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * T, device="cuda")
    live = torch.empty(B * H * (T // 128) * (T // 64), dtype=torch.uint8, device="cuda")
    do = torch.randn_like(o)
    dq = torch.empty_like(qkv)
    work = torch.empty(int(ext.lib().fb_attn_bwd_work_floats(B, T, H, dh)), device="cuda")
    st = ext.stream_handle()
    ext.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), live.data_ptr(), B, T, H, dh, 1, st)
    f = lambda: ext.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), live.data_ptr(),
                         dq.data_ptr(), work.data_ptr(), B, T, H, dh, 1, st)
    for _ in range(3):
        f()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 10)
    fl = 2.0 * 2.0 * B * H * dh * T * (T + 1)
    out[f"dh{dh}"] = {"ms": round(min(ts), 4), "tflops": round(fl / min(ts) / 1e9, 1), "dq_sum": float(dq.float().abs().sum())}
print(json.dumps(out))
"""
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for rep in range(2):
    for lib in sys.argv[1:]:
        env = dict(os.environ, ROOT=root, FB_LIB_PATH=lib if lib != "prod" else "")
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        print(lib, rep, r.stdout.strip() or r.stderr[-500:], flush=True)
