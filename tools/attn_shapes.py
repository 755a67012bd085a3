import os, sys, json, torch
sys.path.insert(0, '/root/repo')
from paper_2405_10853_b200 import ext
ext.lib()
for B, T, H, dh in [(8, 2048, 16, 128), (2, 4096, 16, 128), (32, 1024, 16, 128), (64, 512, 16, 128)]:
    d = H * dh
    qkv = torch.randn(B * T, 3 * d, device="cuda").to(torch.bfloat16)
    o = torch.empty(B * T, d, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * T, device="cuda")
    live = torch.empty(B * H * (T // 128) * (T // 64), dtype=torch.uint8, device="cuda")
    do = torch.randn_like(o); dqkv = torch.empty_like(qkv)
    work = torch.empty(int(ext.lib().fb_attn_bwd_work_floats(B, T, H, dh)), device="cuda")
    st = ext.stream_handle()
    fwd = lambda: ext.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), live.data_ptr(), B, T, H, dh, 0, st)  # no alibi: all live
    fwd()
    for _ in range(3): fwd()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(10): fwd()
    f1.record(); torch.cuda.synchronize()
    fwd_ms = f0.elapsed_time(f1) / 10
    bwd = lambda: ext.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), live.data_ptr(), dqkv.data_ptr(), work.data_ptr(), B, T, H, dh, 0, st)
    for _ in range(3): bwd()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): bwd()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    tiles = B * H * sum(T // 64 - 2 * kb for kb in range(T // 128))
    ctas = B * H * (T // 128)
    ftiles = B * H * sum(2 * (2 * pb + 2) - 1 for pb in range(T // 256))  # (Q tile, KV tile) steps of 128 x 128
    print(json.dumps({"B": B, "T": T, "bwd_ctas": ctas, "bwd_tiles": tiles, "bwd_us": round(ms * 1e3, 1),
                      "bwd_ns_per_tile_per_sm": round(ms * 1e6 * 148 / tiles, 1), "fwd_ctas": B * H * (T // 256),
                      "fwd_steps": ftiles, "fwd_us": round(fwd_ms * 1e3, 1),
                      "fwd_ns_per_step_per_sm": round(fwd_ms * 1e6 * 148 / ftiles, 1)}))
