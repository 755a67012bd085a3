"""One C4-shaped GEMM a few times, for ncu. GN (N, default 6144 = qkv), GK (K, default 2048),
GE (epilogue name, default bf16)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
M, N, K = 16384, int(os.environ.get("GN", "6144")), int(os.environ.get("GK", "2048"))
epi = os.environ.get("GE", "bf16")
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
cdt = torch.bfloat16 if epi in ("bf16", "gelu", "dgelu") else torch.float32
C = torch.empty(M, N, dtype=cdt, device="cuda")
aux = torch.randn(M, N, device="cuda").to(torch.bfloat16 if epi in ("gelu", "dgelu") else torch.float32)
for _ in range(4):
    ext.call("fb_gemm_bf16", M, N, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, C.data_ptr(), N, ext.EPI[epi],
             aux.data_ptr(), aux.data_ptr(), N, ext.stream_handle())
torch.cuda.synchronize()
print("ok")
