"""GPU parity of attention / LayerNorm / embedding / cross-entropy kernels
against a torch fp32 reference of the same op on the same (bf16) inputs."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fb():
    from paper_2405_10853_b200 import ext
    ext.lib()
    return ext


def alibi_ref(H, T, use_alibi, dev):
    slopes = torch.tensor([2.0 ** (-8.0 * (h + 1) / H) for h in range(H)], dtype=torch.float64)
    i = torch.arange(T)[:, None]
    j = torch.arange(T)[None, :]
    b = -slopes[:, None, None] * (i - j)[None].double() if use_alibi else torch.zeros(H, T, T, dtype=torch.float64)
    b = b.float()
    b[:, j.expand(T, T) > i.expand(T, T)] = -math.inf
    return b.to(dev)


def attn_ref(qkv, B, T, H, dh, use_alibi):
    d = H * dh
    x = qkv.float().view(B, T, 3, H, dh)
    q, k, v = x[:, :, 0].transpose(1, 2), x[:, :, 1].transpose(1, 2), x[:, :, 2].transpose(1, 2)
    s = (q @ k.transpose(-1, -2)) / math.sqrt(dh) + alibi_ref(H, T, use_alibi, qkv.device)
    lse = torch.logsumexp(s, dim=-1)
    o = (torch.softmax(s, -1) @ v).transpose(1, 2).reshape(B * T, d)
    return o, lse


@pytest.mark.parametrize("B,T,H,dh,alibi", [(2, 128, 2, 64, 1), (1, 256, 3, 64, 1), (2, 128, 2, 128, 1),
                                             (1, 512, 4, 128, 1), (2, 128, 2, 64, 0), (1, 1024, 12, 64, 1),
                                             (1, 384, 2, 128, 1), (2, 640, 3, 64, 0),
                                             # the C3 / C4 context length (T = 2048), dead-block map on
                                             (1, 2048, 16, 128, 1), (1, 2048, 12, 64, 1),
                                             # CUDA-core path: the reference's desk shapes and ragged T
                                             (3, 64, 4, 16, 1), (2, 16, 2, 8, 1), (2, 8, 2, 4, 0), (1, 16, 3, 8, 1),
                                             (2, 200, 2, 64, 1), (1, 130, 2, 128, 0), (2, 96, 3, 32, 1)])
def test_attention_fwd_bwd(fb, B, T, H, dh, alibi):
    torch.manual_seed(0)
    dev = torch.device("cuda")
    d = H * dh
    qkv = torch.randn(B * T, 3 * d, device=dev).to(torch.bfloat16)
    o = torch.empty(B * T, d, dtype=torch.bfloat16, device=dev)
    lse2 = torch.empty(B * H * T, dtype=torch.float32, device=dev)
    live = torch.empty(B * H * ((T + 127) // 128) * ((T + 63) // 64), dtype=torch.uint8, device=dev)
    fb.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse2.data_ptr(), live.data_ptr(), B, T, H, dh, alibi,
            fb.stream_handle())
    q32 = qkv.float().requires_grad_()
    o_ref, lse_ref = attn_ref(q32, B, T, H, dh, alibi)
    torch.cuda.synchronize()
    torch.testing.assert_close(o.float(), o_ref, atol=2e-2, rtol=2e-2)
    torch.testing.assert_close(lse2.view(B, H, T) * math.log(2.0), lse_ref, atol=1e-3, rtol=1e-3)
    do = torch.randn(B * T, d, device=dev).to(torch.bfloat16)
    o_ref.backward(do.float())
    dqkv = torch.empty_like(qkv)
    work = torch.empty(int(fb.lib().fb_attn_bwd_work_floats(B, T, H, dh)), dtype=torch.float32, device=dev)
    fb.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse2.data_ptr(), live.data_ptr(),
            dqkv.data_ptr(), work.data_ptr(), B, T, H, dh, alibi, fb.stream_handle())
    torch.cuda.synchronize()
    g = q32.grad
    for sl, name in [(slice(0, d), "dq"), (slice(d, 2 * d), "dk"), (slice(2 * d, 3 * d), "dv")]:
        ref = g[:, sl]
        got = dqkv[:, sl].float()
        err = (got - ref).abs().max().item()
        scale = ref.abs().max().item()
        assert err <= 3e-2 * scale + 1e-2, (name, err, scale)


def _attn_run(fb, qkv, do, B, T, H, dh, live):
    d = H * dh
    dev = qkv.device
    o = torch.empty(B * T, d, dtype=torch.bfloat16, device=dev)
    lse2 = torch.empty(B * H * T, dtype=torch.float32, device=dev)
    dqkv = torch.empty_like(qkv)
    work = torch.empty(int(fb.lib().fb_attn_bwd_work_floats(B, T, H, dh)), dtype=torch.float32, device=dev)
    lp = live.data_ptr() if live is not None else None
    fb.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse2.data_ptr(), lp, B, T, H, dh, 1, fb.stream_handle())
    fb.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse2.data_ptr(), lp, dqkv.data_ptr(),
            work.data_ptr(), B, T, H, dh, 1, fb.stream_handle())
    torch.cuda.synchronize()
    return o, lse2, dqkv


@pytest.mark.parametrize("B,T,H,dh", [(2, 2048, 16, 128), (1, 1024, 12, 64), (1, 1408, 16, 128)])
def test_attention_dead_block_skip_is_exact(fb, B, T, H, dh):
    """ALiBi drives far-from-diagonal softmax weights to exactly 0 (ex2 flush); the forward
    marks those blocks dead and skips their PV, the backward skips their MMAs. The outputs
    must be bit-identical to the run without the map, and the map must hold dead blocks."""
    torch.manual_seed(5)
    dev = torch.device("cuda")
    d = H * dh
    qkv = torch.randn(B * T, 3 * d, device=dev).to(torch.bfloat16)
    do = torch.randn(B * T, d, device=dev).to(torch.bfloat16)
    live = torch.full((B * H * (T // 128) * (T // 64),), 7, dtype=torch.uint8, device=dev)
    o1, l1, g1 = _attn_run(fb, qkv, do, B, T, H, dh, live)
    o0, l0, g0 = _attn_run(fb, qkv, do, B, T, H, dh, None)
    assert torch.equal(o1, o0) and torch.equal(l1, l0)
    # dK / dV come from one CTA each; dQ adds the key blocks' partials in descending key-block
    # order, and a skipped (dead) partial is an exact 0 in the unmapped run: all bit-identical
    assert torch.equal(g1, g0)
    m = live.view(B, H, T // 128, T // 64).cpu().numpy()
    causal = np.array([[kt <= 2 * qt + 1 for kt in range(T // 64)] for qt in range(T // 128)])
    vals = m[:, :, causal]
    assert set(np.unique(vals)) <= {0, 1}
    dead = (vals == 0).mean()
    assert dead > 0.05, dead  # steep heads: most far blocks are dead
    # the diagonal blocks are always live
    for qt in range(T // 128):
        assert (m[:, :, qt, 2 * qt + 1] == 1).all()


def test_attention_bwd_all_dead_map_zeroes(fb):
    """A map that marks every block dead: the backward must finish and produce exact zeros."""
    B, T, H, dh = 1, 256, 2, 128
    dev = torch.device("cuda")
    d = H * dh
    qkv = torch.randn(B * T, 3 * d, device=dev).to(torch.bfloat16)
    do = torch.randn(B * T, d, device=dev).to(torch.bfloat16)
    o = torch.empty(B * T, d, dtype=torch.bfloat16, device=dev)
    lse2 = torch.empty(B * H * T, dtype=torch.float32, device=dev)
    fb.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse2.data_ptr(), None, B, T, H, dh, 1, fb.stream_handle())
    live = torch.zeros(B * H * (T // 128) * (T // 64), dtype=torch.uint8, device=dev)
    dqkv = torch.full_like(qkv, 3.0)
    work = torch.empty(int(fb.lib().fb_attn_bwd_work_floats(B, T, H, dh)), dtype=torch.float32, device=dev)
    fb.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse2.data_ptr(), live.data_ptr(),
            dqkv.data_ptr(), work.data_ptr(), B, T, H, dh, 1, fb.stream_handle())
    torch.cuda.synchronize()
    assert (dqkv.float() == 0).all()


@pytest.mark.parametrize("rows,d", [(256, 512), (100, 768), (64, 2048), (33, 128), (5003, 2048), (20011, 512),
                                    (9001, 768)])
def test_layernorm(fb, rows, d):
    """fb_ln_fwd / fb_ln_bwd vs torch; d = 512 / 768 take the warp-per-row backward (grid-looped at
    the larger row counts), the others the CTA-per-row one."""
    torch.manual_seed(1)
    dev = torch.device("cuda")
    x = torch.randn(rows, d, device=dev) * 2 + 0.5
    gamma = torch.randn(d, device=dev)
    beta = torch.randn(d, device=dev)
    y = torch.empty(rows, d, dtype=torch.bfloat16, device=dev)
    mean = torch.empty(rows, device=dev)
    rstd = torch.empty(rows, device=dev)
    fb.call("fb_ln_fwd", x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(), mean.data_ptr(),
            rstd.data_ptr(), rows, d, fb.stream_handle())
    xr = x.clone().requires_grad_()
    gr = gamma.clone().requires_grad_()
    br = beta.clone().requires_grad_()
    ref = F.layer_norm(xr, (d,), gr, br, 1e-5)
    torch.cuda.synchronize()
    torch.testing.assert_close(y.float(), ref, atol=3e-2, rtol=1e-2)
    dy = torch.randn(rows, d, device=dev)
    dres = torch.randn(rows, d, device=dev)
    ref.backward(dy)
    dx = torch.empty_like(x)
    dxb = torch.empty(rows, d, dtype=torch.bfloat16, device=dev)
    dg = torch.zeros(d, device=dev)
    db = torch.ones(d, device=dev)  # accumulates
    work = torch.empty(2 * 592 * d, device=dev)
    fb.call("fb_ln_bwd", x.data_ptr(), gamma.data_ptr(), mean.data_ptr(), rstd.data_ptr(), dy.data_ptr(),
            dres.data_ptr(), dx.data_ptr(), dxb.data_ptr(), dg.data_ptr(), db.data_ptr(), work.data_ptr(), rows, d,
            fb.stream_handle())
    torch.cuda.synchronize()
    torch.testing.assert_close(dx, xr.grad + dres, atol=1e-4, rtol=1e-4)
    torch.testing.assert_close(dxb.float(), dx, atol=2e-2, rtol=1e-2)
    torch.testing.assert_close(dg, gr.grad, atol=1e-3, rtol=1e-4)
    torch.testing.assert_close(db, br.grad + 1, atol=1e-3, rtol=1e-4)


def test_embedding(fb):
    torch.manual_seed(2)
    dev = torch.device("cuda")
    V, d, B, T = 300, 256, 4, 64
    emb = torch.randn(V, d, device=dev)
    pos = torch.randn(T, d, device=dev)
    tok = torch.randint(0, V, (B * T,), device=dev, dtype=torch.int32)
    x = torch.empty(B * T, d, device=dev)
    for p in (None, pos):
        fb.call("fb_embed_fwd", tok.data_ptr(), emb.data_ptr(), fb.ptr(p), x.data_ptr(), B * T, T, d, fb.stream_handle())
        ref = emb[tok.long()] + (pos.repeat(B, 1) if p is not None else 0)
        torch.cuda.synchronize()
        assert torch.equal(x, ref)
    dx = torch.randn(B * T, d, device=dev)
    ge = torch.zeros(V, d, device=dev)
    gp = torch.zeros(T, d, device=dev)
    fb.call("fb_embed_bwd", tok.data_ptr(), dx.data_ptr(), ge.data_ptr(), gp.data_ptr(), B * T, T, d, V,
            fb.stream_handle())
    ref = torch.zeros(V, d, device=dev).index_add_(0, tok.long(), dx)
    torch.cuda.synchronize()
    torch.testing.assert_close(ge, ref, atol=1e-4, rtol=1e-5)
    torch.testing.assert_close(gp, dx.view(B, T, d).sum(0), atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("V,d,B,T,skew", [(300, 256, 4, 64, False), (32000, 2048, 8, 2048, True), (64, 16, 4, 16, False),
                                          (48, 24, 3, 16, True)])
def test_embedding_bwd_sorted_is_deterministic(fb, V, d, B, T, skew):
    """the sorted-token segment sum gives the same bits on every run and equals
    the fixed-order (ascending position) sum of the rows of each token."""
    torch.manual_seed(3)
    dev = torch.device("cuda")
    n = B * T
    tok = torch.randint(0, V, (n,), device=dev, dtype=torch.int32)
    if skew:  # one dominant id, as in real text
        tok[torch.rand(n, device=dev) < 0.3] = 7
    dx = torch.randn(n, d, device=dev)
    wb = int(fb.lib().fb_embed_bwd_work_bytes(n, V))
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    outs = []
    for _ in range(3):
        ge = torch.full((V, d), 0.5, device=dev)
        gp = torch.full((T, d), 0.25, device=dev)
        fb.call("fb_embed_bwd_sorted", tok.data_ptr(), dx.data_ptr(), ge.data_ptr(), gp.data_ptr(), n, T, d, V,
                work.data_ptr(), wb, fb.stream_handle())
        outs.append((ge.clone(), gp.clone()))
    torch.cuda.synchronize()
    for ge, gp in outs[1:]:
        assert torch.equal(ge, outs[0][0]) and torch.equal(gp, outs[0][1])
    ge, gp = outs[0]
    ref = torch.zeros(V, d, dtype=torch.float64, device=dev).index_add_(0, tok.long(), dx.double()) + 0.5
    torch.testing.assert_close(ge.double(), ref, atol=1e-3 * (n / V) ** 0.5 + 1e-4, rtol=1e-5)
    torch.testing.assert_close(gp.double(), dx.double().view(B, T, d).sum(0) + 0.25, atol=1e-4, rtol=1e-5)
    # the exact fixed-order f32 sum for a few ids: the run's rows (ascending positions) in 8
    # contiguous ranges, each summed in order, the range sums added in order (d % 8 == 0),
    # or one sequential sum (d % 8 != 0)
    t_cpu, dx_cpu = tok.cpu().numpy(), dx.cpu().numpy()
    for v in [7] + list(np.unique(t_cpu)[:3]):
        rows = np.nonzero(t_cpu == v)[0]
        if rows.size == 0:
            continue
        n_r = rows.size
        ranges = [rows[n_r * w // 8: n_r * (w + 1) // 8] for w in range(8)] if d % 8 == 0 else [rows]
        parts = []
        for rg in ranges:
            acc = np.zeros(d, np.float32)
            for r in rg:
                acc += dx_cpu[r]
            parts.append(acc)
        tot = parts[0].copy()
        for p_ in parts[1:]:
            tot += p_
        assert np.array_equal(ge[v].cpu().numpy(), np.float32(0.5) + tot), v


@pytest.mark.parametrize("V,d,B,T", [(256, 512, 3, 64), (32000, 512, 2, 1024), (32000, 2048, 4, 2048), (48, 24, 3, 16),
                                     (32000, 768, 33, 128)])
def test_lmhead_cross_entropy(fb, V, d, B, T):
    """fb_lmhead_ce: LM head GEMM + mean next-token CE with no f32 logits tensor,
    in two row chunks (row0 > 0), against torch fp32 on the same bf16 operands:
    loss rel <= 1e-5, dlogits within bf16 rounding (atol 1e-6 / rtol 2e-2)."""
    torch.manual_seed(3)
    dev = torch.device("cuda")
    M = B * T
    x = (torch.randn(M, d, device=dev) * 0.5).to(torch.bfloat16)
    w = (torch.randn(V, d, device=dev) * (3.0 / d ** 0.5)).to(torch.bfloat16)
    tok = torch.randint(0, V, (M,), device=dev, dtype=torch.int32)
    scale = 1.0 / (B * (T - 1))
    dl = torch.empty(M, V, dtype=torch.bfloat16, device=dev)
    row_loss = torch.empty(M, dtype=torch.float64, device=dev)
    h = (M // 2 + 7) // 8 * 8
    nw = int(fb.lib().fb_lmhead_ce_work_floats(max(h, M - h), V))
    work = torch.empty(nw, dtype=torch.float32, device=dev)
    for r0, n in [(0, h), (h, M - h)]:
        fb.call("fb_lmhead_ce", x[r0:].data_ptr(), w.data_ptr(), tok.data_ptr(), r0, n, T, V, d, scale, 1,
                dl[r0:].data_ptr(), work.data_ptr(), nw, row_loss.data_ptr(), fb.stream_handle())
    lg = (x.float() @ w.float().t()).view(B, T, V).requires_grad_()
    ref = F.cross_entropy(lg[:, :-1].reshape(-1, V), tok.view(B, T)[:, 1:].reshape(-1).long())
    ref.backward()
    torch.cuda.synchronize()
    assert row_loss.view(B, T)[:, -1].abs().max().item() == 0.0
    assert row_loss.sum().item() * scale == pytest.approx(ref.item(), rel=1e-5)
    torch.testing.assert_close(dl.float(), lg.grad.view(M, V), atol=1e-6, rtol=2e-2)


@pytest.mark.parametrize("B,T,H,dh", [(8, 2048, 16, 128), (16, 1024, 8, 64), (1, 512, 4, 128)])
def test_outproj_dgrad_rowdot_feeds_attention_bwd(fb, B, T, H, dh):
    """dO = dY W_proj with D = rowsum(bf16(dO) o O) fused into the GEMM epilogue (fb_gemm_bf16_rowdot):
    dO is bit-identical to the plain bf16 GEMM, D matches torch, and fb_attn_bwd_ex(FB_ATTN_D_READY)
    gives the same dQ/dK/dV as fb_attn_bwd (which forms D itself) up to f32 summation order."""
    torch.manual_seed(3)
    dev = torch.device("cuda")
    d, M = H * dh, B * T
    dY = (torch.randn(M, d, device=dev) * 0.5).to(torch.bfloat16)
    W = (torch.randn(d, d, device=dev) * d ** -0.5).to(torch.bfloat16)   # proj weight [out][in], MN-major B for dgrad
    O = torch.randn(M, d, device=dev).to(torch.bfloat16)
    dO_plain = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
    dO = torch.empty_like(dO_plain)
    D = torch.full((B * H * T,), float("nan"), device=dev)
    fb.call("fb_gemm_bf16", M, d, d, dY.data_ptr(), d, 0, W.data_ptr(), d, 1, dO_plain.data_ptr(), d, fb.EPI["bf16"],
            None, None, 0, fb.stream_handle())
    rc = fb.lib().fb_gemm_bf16_rowdot(M, d, d, dY.data_ptr(), d, 0, W.data_ptr(), d, 1, dO.data_ptr(), d,
                                      O.data_ptr(), d, D.data_ptr(), T, dh, fb.stream_handle())
    if M < 256 or (M // 256) * (d // 256) < 74:  # only the 2-SM kernel fuses; the model then falls back
        assert rc == fb.FB_UNSUPPORTED
        return
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.equal(dO, dO_plain)
    ref = (dO.float() * O.float()).view(B, T, H, dh).sum(-1).permute(0, 2, 1).reshape(-1)
    torch.testing.assert_close(D, ref, atol=1e-3, rtol=1e-4)
    # attention backward with the fused D vs with its own pre-pass
    qkv = torch.randn(M, 3 * d, device=dev).to(torch.bfloat16)
    o = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
    lse2 = torch.empty(B * H * T, dtype=torch.float32, device=dev)
    live = torch.empty(B * H * (T // 128) * (T // 64), dtype=torch.uint8, device=dev)
    fb.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse2.data_ptr(), live.data_ptr(), B, T, H, dh, 1,
            fb.stream_handle())
    rc = fb.lib().fb_gemm_bf16_rowdot(M, d, d, dY.data_ptr(), d, 0, W.data_ptr(), d, 1, dO.data_ptr(), d,
                                      o.data_ptr(), d, D.data_ptr(), T, dh, fb.stream_handle())
    assert rc == 0
    work = torch.empty(int(fb.lib().fb_attn_bwd_work_floats(B, T, H, dh)), dtype=torch.float32, device=dev)
    work[: B * H * T].copy_(D)
    work[B * H * T:].fill_(123.0)  # garbage accumulator and box counters: the call must not depend on them
    g1 = torch.empty_like(qkv)
    g2 = torch.empty_like(qkv)
    fb.call("fb_attn_bwd_ex", qkv.data_ptr(), o.data_ptr(), dO.data_ptr(), lse2.data_ptr(), live.data_ptr(),
            g1.data_ptr(), work.data_ptr(), B, T, H, dh, 1, 1, fb.stream_handle())
    work2 = torch.empty_like(work)
    fb.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), dO.data_ptr(), lse2.data_ptr(), live.data_ptr(),
            g2.data_ptr(), work2.data_ptr(), B, T, H, dh, 1, fb.stream_handle())
    torch.cuda.synchronize()
    torch.testing.assert_close(work[: B * H * T], work2[: B * H * T], atol=1e-3, rtol=1e-4)
    torch.testing.assert_close(g1.float(), g2.float(), atol=2e-2, rtol=2e-2)


@pytest.mark.parametrize("B,T,H,dh", [(2, 512, 4, 128), (2, 1024, 3, 64), (1, 2048, 16, 128), (2, 2048, 12, 64)])
def test_attention_bwd_deterministic_mode(fb, B, T, H, dh):
    """The tcgen05 backward adds each query block's dQ partials in descending key-block order
    (per-box counters) and writes bf16 dQ itself: every run is bitwise equal, whatever
    fb_set_deterministic says (ABI 3), and no dQ byte of the output is left from before the call
    (dqkv pre-filled with NaN)."""
    torch.manual_seed(9)
    dev = torch.device("cuda")
    d = H * dh
    qkv = torch.randn(B * T, 3 * d, device=dev).to(torch.bfloat16)
    do = torch.randn(B * T, d, device=dev).to(torch.bfloat16)
    o = torch.empty(B * T, d, dtype=torch.bfloat16, device=dev)
    lse2 = torch.empty(B * H * T, dtype=torch.float32, device=dev)
    live = torch.empty(B * H * (T // 128) * (T // 64), dtype=torch.uint8, device=dev)
    st = fb.stream_handle()
    fb.call("fb_attn_fwd", qkv.data_ptr(), o.data_ptr(), lse2.data_ptr(), live.data_ptr(), B, T, H, dh, 1, st)
    outs = []
    for det in (0, 1, 1, 0):
        fb.call("fb_set_deterministic", det)
        nw = int(fb.lib().fb_attn_bwd_work_floats(B, T, H, dh))
        work = torch.full((nw,), float("nan"), dtype=torch.float32, device=dev)
        dqkv = torch.full_like(qkv, float("nan"))
        fb.call("fb_attn_bwd", qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse2.data_ptr(), live.data_ptr(),
                dqkv.data_ptr(), work.data_ptr(), B, T, H, dh, 1, st)
        outs.append(dqkv)
    fb.call("fb_set_deterministic", 1)  # the library default
    torch.cuda.synchronize()
    assert torch.isfinite(outs[0].float()).all()
    for x in outs[1:]:
        assert torch.equal(outs[0], x)
