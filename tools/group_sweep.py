"""Interleaved A/B of the 2-SM raster group height (fb_gemm_set_group_m) on the C4 GEMM shapes.
Each round times every (shape, G) once, in rotating order; prints the median TFLOP/s per cell."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

lib = ext.lib()
Mt = 16384
shapes = [("qkv_fwd", Mt, 6144, 2048, 0, 0, "bf16"), ("fc_fwd_gelu", Mt, 8192, 2048, 0, 0, "gelu"),
          ("proj2_fwd_resid", Mt, 2048, 8192, 0, 0, "resid_f32"), ("proj2_dgrad_dgelu", Mt, 8192, 2048, 0, 1, "dgelu"),
          ("fc_dgrad", Mt, 2048, 8192, 0, 1, "f32"), ("qkv_dgrad", Mt, 2048, 6144, 0, 1, "f32"),
          ("qkv_wgrad", 6144, 2048, Mt, 1, 1, "acc_f32"), ("fc_wgrad", 8192, 2048, Mt, 1, 1, "acc_f32"),
          ("head_fwd", 8192, 32000, 2048, 0, 0, "f32"), ("head_dgrad", 8192, 2048, 32000, 0, 1, "f32")]
GS = [int(x) for x in os.environ.get("GS", "0,2,3,4,8").split(",")]
ROUNDS = int(os.environ.get("ROUNDS", "5"))
ws = torch.empty(16 << 20, dtype=torch.float32, device="cuda")
bufs = {}
for name, M, N, K, am, bm, epi in shapes:
    A = torch.randn((K, M) if am else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((K, N) if bm else (N, K), device="cuda").to(torch.bfloat16)
    cdt = torch.bfloat16 if epi in ("bf16", "gelu", "dgelu") else torch.float32
    C = torch.zeros(M, N, dtype=cdt, device="cuda")
    aux = torch.zeros(M, N, dtype=torch.bfloat16 if epi in ("gelu", "dgelu") else torch.float32, device="cuda")
    bufs[name] = (A, B, C, aux)


def run(name, M, N, K, am, bm, epi, reps=6):
    A, B, C, aux = bufs[name]
    st = ext.stream_handle()
    def one():
        if epi in ("f32", "acc_f32"):
            ext.call("fb_gemm_bf16_splitk", M, N, K, A.data_ptr(), M if am else K, am, B.data_ptr(), N if bm else K, bm,
                     C.data_ptr(), N, ext.EPI[epi], 0, ws.data_ptr(), ws.numel() * 4, st)
        else:
            ext.call("fb_gemm_bf16", M, N, K, A.data_ptr(), M if am else K, am, B.data_ptr(), N if bm else K, bm,
                     C.data_ptr(), N, ext.EPI[epi], aux.data_ptr(), aux.data_ptr(), N, st)
    one()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        one()
    e1.record()
    torch.cuda.synchronize()
    return 2.0 * M * N * K * reps / (e0.elapsed_time(e1) / 1e3) / 1e12


res = {(s[0], g): [] for s in shapes for g in GS}
for r in range(ROUNDS):
    order = GS[r % len(GS):] + GS[:r % len(GS)]
    for s in shapes:
        for g in order:
            ext.check(lib.fb_gemm_set_group_m(g), "group")
            res[(s[0], g)].append(run(*s))
for s in shapes:
    print(json.dumps({"gemm": s[0], **{f"G{g}": round(statistics.median(res[(s[0], g)]), 1) for g in GS}}), flush=True)
