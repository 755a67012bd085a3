"""One attention fwd + bwd at the C4 shape (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
B, T, H, dh = 8, 2048, int(os.environ.get("AO_H", 16)), int(os.environ.get("AO_DH", 128))
d = H * dh
qkv = torch.randn(B * T, 3 * d, device="cuda").to(torch.bfloat16)
o = torch.empty(B * T, d, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(B * H * T, device="cuda")
live = torch.empty(B * H * (T // 128) * (T // 64), dtype=torch.uint8, device="cuda")
do = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
work = torch.empty(int(ext.lib().fb_attn_bwd_work_floats(B, T, H, dh)), device="cuda")
st = ext.stream_handle()
for _ in range(2):
    ext.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), live.data_ptr(), B, T, H, dh, 1, st)
    ext.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), live.data_ptr(), dqkv.data_ptr(),
             work.data_ptr(), B, T, H, dh, 1, st)
torch.cuda.synchronize()
print("ok")
