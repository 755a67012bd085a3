"""Time the tcgen05 GEMM at the C4 shapes (fwd, dgrad, wgrad), 2-SM vs 1-SM."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
Mt = 16384
shapes = [  # name, M, N, K, a_major, b_major, epi
    ("qkv_fwd", Mt, 6144, 2048, 0, 0, "bf16"), ("fc_fwd_gelu", Mt, 8192, 2048, 0, 0, "gelu"),
    ("proj2_fwd_resid", Mt, 2048, 8192, 0, 0, "resid_f32"), ("proj2_dgrad_dgelu", Mt, 8192, 2048, 0, 1, "dgelu"),
    ("fc_dgrad", Mt, 2048, 8192, 0, 1, "f32"), ("qkv_wgrad", 6144, 2048, Mt, 1, 1, "acc_f32"),
    ("proj_wgrad", 2048, 2048, Mt, 1, 1, "acc_f32"), ("head_fwd", 8192, 32000, 2048, 0, 0, "f32"),
    ("c2_qkv_wgrad", 1536, 512, Mt, 1, 1, "acc_f32"), ("c2_proj_wgrad", 512, 512, Mt, 1, 1, "acc_f32"),
    ("c2_fc2_dgrad_dgelu", 262144, 2048, 512, 0, 1, "dgelu"), ("c2_fc_fwd_gelu", 262144, 2048, 512, 0, 0, "gelu"),
    ("c2_proj2_fwd_resid", 262144, 512, 2048, 0, 0, "resid_f32"), ("c2_proj_fwd_resid", 262144, 512, 512, 0, 0, "resid_f32"),
]
ONLY = [x for x in os.environ.get("GB_ONLY", "").split(",") if x]
for name, M, N, K, am, bm, epi in shapes:
    if ONLY and name not in ONLY:
        continue
    epi = os.environ.get("GB_EPI", epi)
    A = torch.randn((K, M) if am else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((K, N) if bm else (N, K), device="cuda").to(torch.bfloat16)
    cdt = torch.bfloat16 if epi in ("bf16", "gelu", "dgelu") else torch.float32
    C = torch.zeros(M, N, dtype=cdt, device="cuda")
    aux = torch.zeros(M, N, dtype=torch.bfloat16 if epi in ("gelu", "dgelu") else torch.float32, device="cuda")
    res = {"gemm": name, "M": M, "N": N, "K": K}
    for en in (1, 0):
        ext.call("fb_gemm_set_2sm", en)
        f = lambda: ext.call("fb_gemm_bf16", M, N, K, A.data_ptr(), A.stride(0), am, B.data_ptr(), B.stride(0), bm,
                             C.data_ptr(), N, ext.EPI[epi], aux.data_ptr(), aux.data_ptr(), N, ext.stream_handle())
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res["tflops_2sm" if en else "tflops_1sm"] = round(2.0 * M * N * K / ms / 1e9, 1)
    ext.call("fb_gemm_set_2sm", 1)
    if epi == "acc_f32":
        ws = torch.empty(16 << 20, dtype=torch.float32, device="cuda")
        f = lambda: ext.call("fb_gemm_bf16_splitk", M, N, K, A.data_ptr(), A.stride(0), am, B.data_ptr(), B.stride(0),
                             bm, C.data_ptr(), N, ext.EPI[epi], 0, ws.data_ptr(), ws.numel() * 4, ext.stream_handle())
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        res["tflops_splitk_auto"] = round(2.0 * M * N * K / (e0.elapsed_time(e1) / 10) / 1e9, 1)
    print(json.dumps(res), flush=True)
