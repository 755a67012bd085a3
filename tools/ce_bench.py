"""Time the fused CE kernel on one C4 LM-head chunk (8192 x 32000 f32 logits)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
rows, V, T = 8192, 32000, 2048
logits = torch.randn(rows, V, device="cuda") * 3
tok = torch.randint(33, 97, (rows + 1,), dtype=torch.int32, device="cuda")
dl = torch.empty(rows, V, dtype=torch.bfloat16, device="cuda")
rl = torch.empty(rows + 1, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ext.call("fb_ce_fwd_bwd", logits.data_ptr(), tok.data_ptr(), dl.data_ptr(), 0, rows, T, V, 1.0, rl.data_ptr(),
             ext.stream_handle())
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = sorted(ts)[len(ts) // 2]
print(f"{os.path.basename(os.environ.get('FB_LIB_PATH', 'prod'))} ce: {t * 1e3:.1f} us, {rows * V * 6 / t / 1e6:.0f} GB/s alg")
