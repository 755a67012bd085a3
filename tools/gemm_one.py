"""One C4 qkv-fwd GEMM (16384 x 6144 x 2048, bf16 out) a few times, for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
M, N, K = 16384, int(os.environ.get("GN", "6144")), 2048
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(4):
    ext.call("fb_gemm_bf16", M, N, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, C.data_ptr(), N, 0, None, None, 0,
             ext.stream_handle())
torch.cuda.synchronize()
print("ok")
