"""Interleaved, sustained comparison of the tcgen05 GEMM with cuBLAS (torch.matmul, bf16 out)
at the C4 shapes. Each round times both on every shape; medians over ROUNDS."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
Mt = 16384
shapes = [("qkv_fwd", Mt, 6144, 2048), ("fc_fwd", Mt, 8192, 2048), ("proj2_fwd", Mt, 2048, 8192),
          ("fc_dgrad", Mt, 2048, 8192), ("head_fwd", 8192, 32000, 2048), ("sq8192", 8192, 8192, 8192)]
ROUNDS = int(os.environ.get("ROUNDS", "6"))
st = ext.stream_handle()
bufs = {}
for name, M, N, K in shapes:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    bufs[name] = (A, B, C)


def timeit(fn, reps=8):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {(n, w): [] for n, *_ in shapes for w in ("ours", "cublas")}
for r in range(ROUNDS):
    for name, M, N, K in shapes:
        A, B, C = bufs[name]
        ours = lambda: ext.call("fb_gemm_bf16", M, N, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, C.data_ptr(), N, 0,
                                None, None, 0, st)
        cub = lambda: torch.matmul(A, B.t(), out=C)
        order = [("ours", ours), ("cublas", cub)] if r % 2 == 0 else [("cublas", cub), ("ours", ours)]
        for w, fn in order:
            res[(name, w)].append(2.0 * M * N * K / (timeit(fn) / 1e3) / 1e12)
for name, M, N, K in shapes:
    print(json.dumps({"gemm": name, "M": M, "N": N, "K": K,
                      "ours_tflops": round(statistics.median(res[(name, "ours")]), 1),
                      "cublas_tflops": round(statistics.median(res[(name, "cublas")]), 1)}), flush=True)
