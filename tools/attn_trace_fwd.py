"""Step timeline of one attention-forward CTA (pair 0 = heaviest, (b,h) = 5) from the
FB_ATTN_TRACE build (tools/libfedb200_trace.so): per KV step, when the MMA thread issued
S(t+1) / PV0(t) / PV1(t) and when each softmax warpgroup got S and released P (us)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

os.environ["FB_LIB_PATH"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfedb200_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

L = ext.lib()
B, T, H, dh = 8, 2048, int(os.environ.get("TH", 16)), int(os.environ.get("TDH", 128))
d = H * dh
qkv = torch.randn(B * T, 3 * d, device="cuda").to(torch.bfloat16)
o = torch.empty(B * T, d, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(B * H * T, device="cuda")
live = torch.empty(B * H * (T // 128) * (T // 64), dtype=torch.uint8, device="cuda")
st = ext.stream_handle()
for _ in range(2):
    ext.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), live.data_ptr(), B, T, H, dh, 1, st)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 2048)()
L.fb_attn_trace_read_fwd.argtypes = [C.c_void_p, C.c_int]
assert L.fb_attn_trace_read_fwd(buf, 2048) == 0
a = np.array(buf[:], dtype=np.int64).reshape(128, 16)
t0 = a[a > 0].min()
names = ["g0:S", "g1:S", "g0:max", "g1:max", "g0:exp", "g1:exp", "g0:P", "g1:P", "m:pf0", "m:pf1", "m:pv0", "m:pv1",
         "m:s0", "m:s1"]
for t in range(128):
    if a[t].max() == 0:
        break
    print(f"t{t:02d} " + " ".join(f"{n}={(a[t, i] - t0) / 1000:6.2f}" if a[t, i] else f"{n}=  -   "
                                 for i, n in enumerate(names)))
