"""Phase timeline of one attention-bwd CTA (FB_ATTN_TRACE build: tools/libfedb200_trace.so)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

os.environ["FB_LIB_PATH"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfedb200_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

L = ext.lib()
B, T, H, dh = 8, 2048, 16, 128
d = H * dh
qkv = torch.randn(B * T, 3 * d, device="cuda").to(torch.bfloat16)
o = torch.empty(B * T, d, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(B * H * T, device="cuda")
live = torch.empty(B * H * (T // 128) * (T // 64), dtype=torch.uint8, device="cuda")
do = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
work = torch.empty(int(ext.lib().fb_attn_bwd_work_floats(B, T, H, dh)), device="cuda")
st = ext.stream_handle()
ext.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), live.data_ptr(), B, T, H, dh, 1, st)
for _ in range(2):
    ext.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), live.data_ptr(), dqkv.data_ptr(),
             work.data_ptr(), B, T, H, dh, 1, st)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 4096)()
L.fb_attn_trace_read.argtypes = [C.c_void_p, C.c_int]
assert L.fb_attn_trace_read(buf, 4096) == 0
a = np.array(buf[:16 * 24], dtype=np.int64).reshape(24, 16)
t0 = a[0, 0] if a[0, 0] else a[0, 4]
names = {0: "mma:pds_full", 1: "mma:S/dP(t+1) issued", 2: "mma:dV,dK issued", 3: "mma:dq_empty",
         4: "sm:wait_S", 5: "sm:S_ready", 6: "sm:P/dS_stored", 7: "sm:drain(t-1)_done"}
for t in range(24):
    if a[t, 4] == 0:
        break
    print(f"tile {t:2d}: " + " ".join(f"{n}={(a[t, i] - t0) / 1000:7.2f}" for i, n in names.items()))
d = np.diff(a[:, 5][a[:, 5] > 0]) / 1000
print("per-tile period (us):", np.round(d, 2))
ew = (a[:, 6] - a[:, 5])[a[:, 5] > 0] / 1000
dr = (a[:, 7] - a[:, 6])[a[:, 5] > 0] / 1000
ws = (a[:, 5] - a[:, 4])[a[:, 5] > 0] / 1000
print("elementwise (us):", np.round(ew, 2))
print("drain (us):", np.round(dr, 2))
print("wait for S (us):", np.round(ws, 2))
