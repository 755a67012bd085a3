"""Per-CTA schedule of the attention backward (FB_ATTN_PROF build: tools/libfedb200_prof.so):
dispatch order, CTA durations, time the dQ warps spend waiting on the ordered-dQ box counters, the
compute warps' stall on the dQ staging box and the last-contributor combine time of the kb = 0 CTAs."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

os.environ["FB_LIB_PATH"] = os.environ.get("FB_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libfedb200_prof.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

L = ext.lib()
L.fb_attn_prof_read.argtypes = [C.c_void_p, C.c_int]
for B, T, H, dh in [(8, 2048, 16, 128), (8, 2048, 12, 64)]:
    d = H * dh
    torch.manual_seed(0)
    qkv = torch.randn(B * T, 3 * d, device="cuda").to(torch.bfloat16)
    o = torch.empty(B * T, d, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * T, device="cuda")
    live = torch.empty(B * H * (T // 128) * (T // 64), dtype=torch.uint8, device="cuda")
    do = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    work = torch.empty(int(L.fb_attn_bwd_work_floats(B, T, H, dh)), device="cuda")
    st = ext.stream_handle()
    ext.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), live.data_ptr(), B, T, H, dh, 1, st)
    for _ in range(3):
        L.fb_attn_prof_clear()
        ext.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), live.data_ptr(),
                 dqkv.data_ptr(), work.data_ptr(), B, T, H, dh, 1, st)
        torch.cuda.synchronize()
    n = (T // 128) * B * H
    buf = (C.c_ulonglong * (8192 * 8))()
    assert L.fb_attn_prof_read(buf, 8192 * 8) == 0
    a = np.array(buf[: n * 8], dtype=np.int64).reshape(n, 8).astype(np.float64)
    t0 = a[:, 0].min()
    start, end, wait = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2] / 1e3
    kb = np.arange(n) % (T // 128)
    dur = end - start
    order = np.argsort(start, kind="stable")
    inversions = int((np.diff(order) < 0).sum())
    per_kb = {int(k): {"dur_us": round(float(dur[kb == k].mean()), 2), "wait_us": round(float(wait[kb == k].mean()), 2)}
              for k in range(T // 128)}
    ntile = np.array([(T // 128 - k) * (2 if dh == 128 else 1) for k in kb], dtype=np.float64)
    print(json.dumps({"compute_sfree_stall_us_per_cta": round(float(a[:, 6].mean() / 1e3), 2),
                      "last_path_us_per_kb0_cta": round(float(a[kb == 0, 7].mean() / 1e3), 2)}))
    print(json.dumps({"shape": [B, T, H, dh], "total_us": round(float(end.max()), 1),
                      "sum_dur_us_per_sm": round(float(dur.sum()) / 148, 1), "sum_wait_us_per_sm": round(float(wait.sum()) / 148, 1),
                      "dispatch_inversions": inversions, "per_kb": per_kb}), flush=True)
    # dispatch spread of one mid-grid (b, h): start of kb 0..15
    bh = (B * H) // 2
    print("bh", bh, "start us:", np.round(start[bh * (T // 128):(bh + 1) * (T // 128)] - start[bh * (T // 128)], 2).tolist())
    print("      wait us:", np.round(wait[bh * (T // 128):(bh + 1) * (T // 128)], 2).tolist())

