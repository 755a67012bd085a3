"""GPU parity of the individual sm_100a kernels through the C ABI.

Integer/byte/f64-register paths are compared bit-exactly with the oracle /
reference golden vectors; bf16 tensor-core GEMMs against a torch fp32 reference
of the same op on the same bf16 inputs (tolerance stated per test)."""
import ctypes as C

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fb():
    from paper_2405_10853_b200 import ext
    ext.lib()
    return ext


def _ptr_array(ts):
    arr = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
    return arr


@pytest.mark.parametrize("tag", ["k8", "k5", "k1", "k13"])
@pytest.mark.parametrize("mode", ["det", "stream"])
def test_fedagg_bitwise_vs_reference(fb, tag, mode):
    g = golden("agg.npz")
    w, m, wk, nk, arr = g[f"{tag}_w"], g[f"{tag}_m"], g[f"{tag}_wk"], g[f"{tag}_nk"], g[f"{tag}_arrival"]
    order = sorted(arr) if mode == "det" else list(arr)
    dev = torch.device("cuda")
    W = torch.from_numpy(w).to(dev)
    M = torch.from_numpy(m).to(dev)
    ks = [torch.from_numpy(wk[k]).to(dev) for k in order]
    nks = (C.c_int64 * len(order))(*[int(nk[k]) for k in order])
    for eta, mu, nes in [(0.7, 0.9, True), (0.1, 0.9, False), (1.0, 0.0, True)]:
        Wo, Mo = torch.empty_like(W), torch.empty_like(M)
        stats = torch.zeros(3, dtype=torch.float64, device=dev)
        bad = torch.zeros(1, dtype=torch.int64, device=dev)
        fb.call("fb_fedagg_step_f32", _ptr_array(ks), nks, len(order), int(mode == "det"), W.data_ptr(),
                M.data_ptr(), Wo.data_ptr(), Mo.data_ptr(), W.numel(), eta, mu, int(nes), stats.data_ptr(),
                bad.data_ptr(), None, fb.stream_handle())
        torch.cuda.synchronize()
        key = f"{tag}_{mode}_{eta}_{mu}_{int(nes)}"
        assert np.array_equal(Wo.cpu().numpy().view(np.uint32), g[key + "_w"].view(np.uint32))
        assert np.array_equal(Mo.cpu().numpy().view(np.uint32), g[key + "_m"].view(np.uint32))
        assert int(bad.item()) >= W.numel()
        pg = g[f"{tag}_pg_{mode}"]
        assert stats[0].item() == pytest.approx(float(np.dot(pg, pg)), rel=1e-12)


def test_fedagg_f64delta_and_nonfinite(fb):
    dev = torch.device("cuda")
    W = torch.tensor([3.0e38, 1.0, 2.0], dtype=torch.float32, device=dev)
    M = torch.zeros(3, dtype=torch.float32, device=dev)
    d = torch.tensor([-3.0e38, 0.5, 0.25], dtype=torch.float64, device=dev)
    Wo, Mo = torch.empty_like(W), torch.empty_like(M)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    fb.call("fb_fedagg_step_f64delta", _ptr_array([d]), (C.c_int64 * 1)(5), 1, 1, W.data_ptr(), M.data_ptr(),
            Wo.data_ptr(), Mo.data_ptr(), 3, 1.0, 0.0, 1, None, bad.data_ptr(), None, fb.stream_handle())
    torch.cuda.synchronize()
    assert bad.item() == 0
    assert Wo[1].item() == 0.5 and Wo[2].item() == 1.75


def test_adamw_bitwise_vs_reference(fb):
    g = golden("adamw.npz")
    dev = torch.device("cuda")
    p = torch.from_numpy(g["p0"].copy()).to(dev)
    m1, m2 = torch.zeros_like(p), torch.zeros_like(p)
    shadow = torch.empty(p.numel(), dtype=torch.bfloat16, device=dev)
    ctl = torch.zeros(6, dtype=torch.float64, device=dev)  # sizeof(fb_step_ctl) = 48
    part = torch.zeros(fb.FB_RED_BLOCKS, dtype=torch.float64, device=dev)
    pu = torch.zeros_like(part)
    cfg = fb.AdamWCfg(float(g["beta1"]), float(g["beta2"]), float(g["eps"]), float(g["wd"]), 1e30)
    for t in range(g["grads"].shape[0]):
        gr = torch.from_numpy(g["grads"][t]).to(dev)
        lr = float(g["lrs"][t])
        fb.call("fb_sumsq_partials", gr.data_ptr(), gr.numel(), part.data_ptr(), fb.stream_handle())
        fb.call("fb_step_prepare", part.data_ptr(), lr, 1 - float(g["beta1"]) ** (t + 1),
                1 - float(g["beta2"]) ** (t + 1), 1e30, ctl.data_ptr(), fb.stream_handle())
        fb.call("fb_adamw_step", p.data_ptr(), gr.data_ptr(), m1.data_ptr(), m2.data_ptr(), shadow.data_ptr(),
                p.numel(), cfg, ctl.data_ptr(), pu.data_ptr(), None, None, fb.stream_handle())
        torch.cuda.synchronize()
        assert np.array_equal(p.cpu().numpy(), g["p"][t])
        assert np.array_equal(m1.cpu().numpy(), g["m1"][t])
        assert np.array_equal(m2.cpu().numpy(), g["m2"][t])
        assert np.sqrt(pu.sum().item()) == pytest.approx(float(g["applied"][t]), rel=1e-12)
    assert torch.equal(shadow, p.to(torch.bfloat16))


def test_clip_decision(fb):
    g = golden("adamw.npz")
    dev = torch.device("cuda")
    x = torch.from_numpy(g["clip_in"]).to(dev)
    part = torch.zeros(fb.FB_RED_BLOCKS, dtype=torch.float64, device=dev)
    ctl = torch.zeros(6, dtype=torch.float64, device=dev)
    fb.call("fb_sumsq_partials", x.data_ptr(), x.numel(), part.data_ptr(), fb.stream_handle())
    fb.call("fb_step_prepare", part.data_ptr(), 1e-3, 0.1, 0.05, 1.0, ctl.data_ptr(), fb.stream_handle())
    torch.cuda.synchronize()
    c = ctl.cpu().numpy()
    assert np.sqrt(c[3]) == pytest.approx(float(g["clip_raw"]), rel=1e-13)
    assert c[4] == pytest.approx(1.0 / float(g["clip_raw"]), rel=1e-13)
    assert ctl.view(torch.int32)[10].item() == 1


def _gemm(fb, A, B, a_major, b_major, M, N, K, epi="f32", C_=None, aux=None, aux_out=None, ld_aux=0):
    if C_ is None:
        C_ = torch.empty(M, N, dtype=torch.bfloat16 if epi in ("bf16", "gelu", "dgelu") else torch.float32,
                         device=A.device)
    fb.call("fb_gemm_bf16", M, N, K, A.data_ptr(), A.stride(0), a_major, B.data_ptr(), B.stride(0), b_major,
            C_.data_ptr(), C_.stride(0), fb.EPI[epi], fb.ptr(aux), fb.ptr(aux_out), ld_aux, fb.stream_handle())
    return C_


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 512, 256), (304, 200, 104), (1024, 1536, 512),
                                   (4096, 6144, 2048), (2048, 32000, 512),
                                   # the reference's desk shapes: d = 8 / 16 / 24, ragged MN-major (2-D TMA chunks)
                                   (8, 32, 48), (16, 16, 8), (24, 72, 64), (200, 96, 40), (64, 24, 16), (72, 1000, 24)])
@pytest.mark.parametrize("a_major,b_major", [(0, 0), (0, 1), (1, 1), (1, 0)])
def test_gemm_layouts(fb, M, N, K, a_major, b_major):
    torch.manual_seed(0)
    dev = torch.device("cuda")
    A = torch.randn(M, K, device=dev).to(torch.bfloat16)
    B = torch.randn(N, K, device=dev).to(torch.bfloat16)
    Ast = A.t().contiguous() if a_major else A
    Bst = B.t().contiguous() if b_major else B
    out = _gemm(fb, Ast, Bst, a_major, b_major, M, N, K)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    err = (out - ref).abs().max().item()
    assert err <= 1e-3 * K ** 0.5 + 1e-2, err


@pytest.mark.parametrize("M,N,K", [(512, 768, 384), (2048, 4096, 512)])
def test_gemm_epilogues(fb, M, N, K):
    torch.manual_seed(1)
    dev = torch.device("cuda")
    A = torch.randn(M, K, device=dev).to(torch.bfloat16)
    B = (0.05 * torch.randn(N, K, device=dev)).to(torch.bfloat16)
    ref = A.float() @ B.float().t()
    # bf16
    o = _gemm(fb, A, B, 0, 0, M, N, K, "bf16")
    torch.testing.assert_close(o.float(), ref, atol=3e-2, rtol=1e-2)
    # acc_f32
    base = torch.randn(M, N, device=dev)
    o = _gemm(fb, A, B, 0, 0, M, N, K, "acc_f32", C_=base.clone())
    torch.testing.assert_close(o, base + ref, atol=1e-3, rtol=1e-4)
    # residual (in place)
    r = base.clone()
    o = _gemm(fb, A, B, 0, 0, M, N, K, "resid_f32", C_=r, aux=r, ld_aux=N)
    torch.testing.assert_close(o, base + ref, atol=1e-3, rtol=1e-4)
    # gelu + pre-activation
    pre = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    o = _gemm(fb, A, B, 0, 0, M, N, K, "gelu", aux_out=pre, ld_aux=N)
    torch.testing.assert_close(pre.float(), ref, atol=3e-2, rtol=1e-2)
    torch.testing.assert_close(o.float(), torch.nn.functional.gelu(pre.float()), atol=2e-2, rtol=1e-2)
    # dgelu
    o = _gemm(fb, A, B, 0, 0, M, N, K, "dgelu", aux=pre, ld_aux=N)
    x = pre.float().requires_grad_()
    torch.nn.functional.gelu(x).backward(ref)
    torch.testing.assert_close(o.float(), x.grad, atol=3e-2, rtol=2e-2)
    torch.cuda.synchronize()


@pytest.mark.parametrize("a_major,b_major", [(0, 0), (0, 1), (1, 1)])
def test_gemm_2sm_matches_1sm(fb, a_major, b_major):
    """The cta_group::2 kernel and the 1-SM kernel give the same fp32 results."""
    torch.manual_seed(5)
    dev = torch.device("cuda")
    M, N, K = 4096, 2048, 1024
    A = torch.randn(M, K, device=dev).to(torch.bfloat16)
    B = torch.randn(N, K, device=dev).to(torch.bfloat16)
    Ast = A.t().contiguous() if a_major else A
    Bst = B.t().contiguous() if b_major else B
    outs = []
    for en in (1, 0):
        fb.call("fb_gemm_set_2sm", en)
        outs.append(_gemm(fb, Ast, Bst, a_major, b_major, M, N, K))
    fb.call("fb_gemm_set_2sm", 1)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("M,N,K,ks", [(1536, 512, 16384, 0), (2048, 2048, 16384, 2), (512, 512, 4096, 5), (384, 1024, 3000, 0)])
def test_gemm_splitk_wgrad(fb, M, N, K, ks):
    """Split-K weight gradient (MN-major A and B, f32 accumulate) == one-pass GEMM within fp32 reassociation."""
    torch.manual_seed(6)
    dev = torch.device("cuda")
    dY = torch.randn(K, M, device=dev).to(torch.bfloat16)   # [tokens][M] -> A MN-major
    X = torch.randn(K, N, device=dev).to(torch.bfloat16)    # [tokens][N] -> B MN-major
    base = torch.randn(M, N, device=dev)
    C1 = base.clone()
    ws = torch.empty(32 << 20, dtype=torch.float32, device=dev)
    fb.call("fb_gemm_bf16_splitk", M, N, K, dY.data_ptr(), M, 1, X.data_ptr(), N, 1, C1.data_ptr(), N,
            fb.EPI["acc_f32"], ks, ws.data_ptr(), ws.numel() * 4, fb.stream_handle())
    ref = base + dY.float().t() @ X.float()
    torch.cuda.synchronize()
    torch.testing.assert_close(C1, ref, atol=2e-3 * K ** 0.5, rtol=1e-4)
    C2 = base.clone()  # deterministic: same result twice
    fb.call("fb_gemm_bf16_splitk", M, N, K, dY.data_ptr(), M, 1, X.data_ptr(), N, 1, C2.data_ptr(), N,
            fb.EPI["acc_f32"], ks, ws.data_ptr(), ws.numel() * 4, fb.stream_handle())
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)


@pytest.mark.parametrize("M,N,K,am,epi", [(6144, 2048, 16384, 1, "acc_f32"), (2048, 8192, 16384, 1, "acc_f32"),
                                         (4160, 2560, 4096, 1, "acc_f32"), (8192, 2048, 32000, 0, "f32")])
def test_gemm_last_wave_split(fb, M, N, K, am, epi):
    """Last-wave split (2-SM raster, ragged final wave cut into K ranges, fixed-order tile-local
    reduction): == torch fp32 within reassociation, deterministic, and the same answer whether
    or not the split is taken (ksplit = 1 runs the plain kernel)."""
    torch.manual_seed(7)
    dev = torch.device("cuda")
    A = torch.randn((K, M) if am else (M, K), device=dev).to(torch.bfloat16)
    B = torch.randn(K, N, device=dev).to(torch.bfloat16)  # MN-major B
    base = torch.randn(M, N, device=dev) if epi == "acc_f32" else torch.zeros(M, N, device=dev)
    ws = torch.empty(16 << 20, dtype=torch.float32, device=dev)
    outs = []
    for ks in (0, 0, 1):
        C = base.clone()
        fb.call("fb_gemm_bf16_splitk", M, N, K, A.data_ptr(), M if am else K, am, B.data_ptr(), N, 1, C.data_ptr(), N,
                fb.EPI[epi], ks, ws.data_ptr(), ws.numel() * 4, fb.stream_handle())
        outs.append(C)
    torch.cuda.synchronize()
    ref = (A.float().t() if am else A.float()) @ B.float() + (base if epi == "acc_f32" else 0)
    torch.testing.assert_close(outs[0], ref, atol=2e-3 * K ** 0.5, rtol=1e-4)
    assert torch.equal(outs[0], outs[1])
    torch.testing.assert_close(outs[0], outs[2], atol=1e-3 * K ** 0.5, rtol=1e-5)


@pytest.mark.parametrize("M,N,K", [(256, 512, 32000), (512, 768, 32000), (8192, 512, 32000), (128, 2048, 32000)])
def test_gemm_splitk_head_dgrad(fb, M, N, K):
    """LM-head dgrad through the split-K entry (K-major dlogits A, MN-major W_head B, f32 out)."""
    torch.manual_seed(8)
    dev = torch.device("cuda")
    A = torch.randn(M, K, device=dev).to(torch.bfloat16)
    B = torch.randn(K, N, device=dev).to(torch.bfloat16)
    C = torch.full((M, N), 7.0, device=dev)
    ws = torch.empty(16 << 20, dtype=torch.float32, device=dev)
    fb.call("fb_gemm_bf16_splitk", M, N, K, A.data_ptr(), K, 0, B.data_ptr(), N, 1, C.data_ptr(), N, fb.EPI["f32"], 0,
            ws.data_ptr(), ws.numel() * 4, fb.stream_handle())
    torch.cuda.synchronize()
    torch.testing.assert_close(C, A.float() @ B.float(), atol=2e-3 * K ** 0.5, rtol=1e-4)


@pytest.mark.parametrize("N", [1024 * 37 + 4, 3_000_004, 1024 * 1000])
@pytest.mark.parametrize("K", [1, 3, 8])
def test_fedagg_bulk_staged_path_is_bitwise_the_register_path(fb, N, K):
    """K <= 8 and n % 4 == 0 take the cp.async.bulk-staged aggregation (whole and partial chunks
    of 1024 parameters); FB_AGG_NO_BULK=1 forces the per-thread-load kernel. w', m', the pseudo-
    gradient and the first-bad index must be bitwise the same; the f64 norm side reductions
    (atomically summed across CTAs) to 1e-12."""
    import os
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(N + K)
    w = torch.empty(N, device=dev).normal_(0, 0.02, generator=gen)
    m = torch.empty(N, device=dev).normal_(0, 1e-3, generator=gen)
    cl = [w + torch.empty(N, device=dev).normal_(0, 2e-3, generator=gen) for _ in range(K)]
    cl[-1][N - 3] = float("nan")  # a non-finite client entry: w' there is NaN, first_bad = N - 3
    nk = (C.c_int64 * K)(*[1000 + 7 * k for k in range(K)])
    ptrs = (C.c_void_p * K)(*[t.data_ptr() for t in cl])
    outs = []
    for no_bulk in ("0", "1"):
        os.environ["FB_AGG_NO_BULK"] = no_bulk
        try:
            wo, mo = torch.empty_like(w), torch.empty_like(m)
            pg = torch.empty(N, dtype=torch.float64, device=dev)
            st = torch.zeros(6 + K, dtype=torch.float64, device=dev)
            bad = torch.zeros(1, dtype=torch.int64, device=dev)
            fb.call("fb_fedagg_step_f32", ptrs, nk, K, 1, w.data_ptr(), m.data_ptr(), wo.data_ptr(), mo.data_ptr(), N,
                    0.7, 0.9, 1, st.data_ptr(), bad.data_ptr(), pg.data_ptr(), fb.stream_handle())
            wr, mr = torch.empty_like(w), torch.empty_like(m)
            fb.call("fb_fedagg_round_norms_f32", ptrs, nk, K, 1, w.data_ptr(), m.data_ptr(), wr.data_ptr(),
                    mr.data_ptr(), N, 0.7, 0.9, 1, st[:6 + K].data_ptr(), None, fb.stream_handle())
            torch.cuda.synchronize()
            outs.append((wo, mo, pg, bad.clone(), st.clone(), wr, mr))
        finally:
            os.environ.pop("FB_AGG_NO_BULK", None)
    (a, b) = outs
    for x, y in zip(a[:3] + a[5:], b[:3] + b[5:]):
        assert torch.equal(x.view(torch.int32) if x.dtype == torch.float32 else x.view(torch.int64),
                           y.view(torch.int32) if y.dtype == torch.float32 else y.view(torch.int64))
    assert int(a[3].item()) == int(b[3].item()) == N - 3
    torch.testing.assert_close(a[4], b[4], rtol=1e-12, atol=0, equal_nan=True)
