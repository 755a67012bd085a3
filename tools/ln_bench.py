"""Time LN fwd / bwd at the C4 shape (16384 x 2048) for the loaded library (FB_LIB_PATH)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
rows, d = 16384, 2048
x = torch.randn(rows, d, device="cuda")
g, b = torch.randn(d, device="cuda"), torch.randn(d, device="cuda")
y = torch.empty(rows, d, dtype=torch.bfloat16, device="cuda")
mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
dy, dres = torch.randn(rows, d, device="cuda"), torch.randn(rows, d, device="cuda")
dx, dxb = torch.empty(rows, d, device="cuda"), torch.empty(rows, d, dtype=torch.bfloat16, device="cuda")
dg, db, work = torch.zeros(d, device="cuda"), torch.zeros(d, device="cuda"), torch.empty(2 * 592 * d, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = ext.stream_handle()
fwd = lambda: ext.call("fb_ln_fwd", x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(), mean.data_ptr(),
                       rstd.data_ptr(), rows, d, st)
bwd = lambda: ext.call("fb_ln_bwd", x.data_ptr(), g.data_ptr(), mean.data_ptr(), rstd.data_ptr(), dy.data_ptr(),
                       dres.data_ptr(), dx.data_ptr(), dxb.data_ptr(), dg.data_ptr(), db.data_ptr(), work.data_ptr(),
                       rows, d, st)
for name, fn, nbytes in [("ln_fwd", fwd, rows * d * 6), ("ln_bwd", bwd, rows * d * 18)]:
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    t = ts[len(ts) // 2]
    print(f"{os.path.basename(os.environ.get('FB_LIB_PATH', 'prod'))} {name}: {t * 1e3:.1f} us, {nbytes / t / 1e6:.0f} GB/s")
