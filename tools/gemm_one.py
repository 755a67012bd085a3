"""One C4-shaped GEMM a few times, for ncu. GM (M, default 16384), GN (N, default 6144 = qkv),
GK (K, default 2048), GAM / GBM (A / B MN-major, default 0), GE (epilogue name, default bf16)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
M, N, K = int(os.environ.get("GM", "16384")), int(os.environ.get("GN", "6144")), int(os.environ.get("GK", "2048"))
am, bm = int(os.environ.get("GAM", "0")), int(os.environ.get("GBM", "0"))
epi = os.environ.get("GE", "bf16")
A = torch.randn((K, M) if am else (M, K), device="cuda").to(torch.bfloat16)
B = torch.randn((K, N) if bm else (N, K), device="cuda").to(torch.bfloat16)
cdt = torch.bfloat16 if epi in ("bf16", "gelu", "dgelu", "ce_exp") else torch.float32
C = torch.zeros(M, N, dtype=cdt, device="cuda")
aux = torch.randn(M, N, device="cuda").to(torch.bfloat16 if epi in ("gelu", "dgelu") else torch.float32)
for _ in range(4):
    ext.call("fb_gemm_bf16", M, N, K, A.data_ptr(), M if am else K, am, B.data_ptr(), N if bm else K, bm,
             C.data_ptr(), N, ext.EPI[epi], aux.data_ptr(), aux.data_ptr(), N, ext.stream_handle())
torch.cuda.synchronize()
print("ok")
