"""C5 aggregation-only sweep: fused delta + weighted mean + Nesterov step
for K in {8,16,32,64} clients x N in {70.5M, 134.1M, 1.339B}, deterministic tree.

Client vectors are resident in HBM; when K x N does not fit (e.g. 64 x 1.339B = 343 GB)
the parameter vector is processed in slices that do (the kernel is slice-local, so the
result is identical), and the time is summed over slices. GB/s counts (4K + 16) N bytes.
Timing: CUDA events over `reps` launches after 2 warm-ups; every launch streams far more
than the 126 MB L2.
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402

ext.lib()
HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
Ns = [int(x) for x in os.environ.get("AGG_NS", "70542336,134125056,1339232256").split(",")]
Ks = [int(x) for x in os.environ.get("AGG_KS", "8,16,32,64").split(",")]
BUDGET = int(float(os.environ.get("AGG_BUDGET_GB", "120")) * 1e9)
reps = 5
for N in Ns:
    for K in Ks:
        sl = min(N, BUDGET // ((K + 4) * 4) // 1024 * 1024)
        gen = torch.Generator(device="cuda").manual_seed(0)
        w = torch.empty(sl, device="cuda").normal_(0, 0.02, generator=gen)
        m = torch.empty(sl, device="cuda").normal_(0, 1e-3, generator=gen)
        cl = [w + torch.empty(sl, device="cuda").normal_(0, 2e-3, generator=gen) for _ in range(K)]
        wo, mo = torch.empty_like(w), torch.empty_like(m)
        ptrs = (C.c_void_p * K)(*[t.data_ptr() for t in cl])
        nks = (C.c_int64 * K)(*[1000 + 7 * k for k in range(K)])
        total_ms = 0.0
        done = 0
        while done < N:
            cnt = min(sl, N - done)

            def launch():
                ext.call("fb_fedagg_step_f32", ptrs, nks, K, 1, w.data_ptr(), m.data_ptr(), wo.data_ptr(),
                         mo.data_ptr(), cnt, 0.7, 0.9, 1, None, None, None, ext.stream_handle())
            for _ in range(2):
                launch()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                launch()
            e1.record()
            torch.cuda.synchronize()
            total_ms += e0.elapsed_time(e1) / reps
            done += cnt
        byts = (4 * K + 16) * N
        gbs = byts / (total_ms / 1e3) / 1e9
        print(json.dumps({"N": N, "K": K, "slices": -(-N // sl), "ms": round(total_ms, 3), "GB": round(byts / 1e9, 2),
                          "GBps": round(gbs, 1), "frac_hbm": round(gbs / HBM, 3)}), flush=True)
        del cl, w, m, wo, mo
        torch.cuda.empty_cache()
