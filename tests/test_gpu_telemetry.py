"""§8(f) drop-ins on the GPU: compute_round_norms, the fused server_step_with_norms and
evaluate_mean_ce, against values produced by the reference (tests/golden/norms_eval.npz)."""
import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


def test_compute_round_norms_vs_reference():
    from paper_2405_10853_b200.params import ParamVector
    from paper_2405_10853_b200.telemetry import compute_round_norms
    g, a = golden("norms_eval.npz"), golden("agg.npz")
    w, wk, nk = a["k8_w"], a["k8_wk"], a["k8_nk"]
    deltas = [w.astype(np.float64) - wk[k].astype(np.float64) for k in range(8)]
    weights = [int(n) / int(nk.sum()) for n in nk]
    rn = compute_round_norms(ParamVector(w), deltas, weights, ParamVector(a["k8_det_0.7_0.9_1_m"]), list(range(8)))
    assert rn.global_norm == pytest.approx(float(g["global_norm"]), rel=1e-12)
    assert rn.avg_client_norm == pytest.approx(float(g["avg_client_norm"]), rel=1e-9)
    assert rn.pseudograd_norm == pytest.approx(float(g["pseudograd_norm"]), rel=1e-6)
    assert rn.momentum_norm == pytest.approx(float(g["momentum_norm"]), rel=1e-12)
    np.testing.assert_allclose([rn.per_client_norms[k] for k in range(8)], g["per_client"], rtol=1e-12)


def test_fused_step_with_norms_bitwise_and_norms():
    from paper_2405_10853_b200.fedopt import (AggregatorState, DeviceClientUpdate, DeviceVector, ServerOptState,
                                              server_step_with_norms)
    g, a = golden("norms_eval.npz"), golden("agg.npz")
    w, m, wk, nk = a["k8_w"], a["k8_m"], a["k8_wk"], a["k8_nk"]
    W = torch.from_numpy(w).cuda()
    agg = AggregatorState(1, w.size, deterministic=True)
    for k in a["k8_arrival"]:
        agg.accumulate(DeviceClientUpdate(int(k), 1, int(nk[k]), torch.from_numpy(wk[k]).cuda(), W))
    opt = ServerOptState(DeviceVector(torch.from_numpy(m).cuda()), 0.7, 0.9, True)
    w2, opt2, rn = server_step_with_norms(opt, DeviceVector(W), agg, 1)
    assert np.array_equal(w2.data.view(np.uint32), a["k8_det_0.7_0.9_1_w"].view(np.uint32))
    assert np.array_equal(opt2.momentum.data.view(np.uint32), a["k8_det_0.7_0.9_1_m"].view(np.uint32))
    assert rn.global_norm == pytest.approx(float(g["global_norm"]), rel=1e-12)
    assert rn.pseudograd_norm == pytest.approx(float(g["pseudograd_norm"]), rel=1e-6)
    assert rn.momentum_norm == pytest.approx(float(g["momentum_norm"]), rel=1e-12)
    np.testing.assert_allclose([rn.per_client_norms[k] for k in range(8)], g["per_client"], rtol=1e-12)


def test_evaluate_mean_ce_vs_reference():
    from paper_2405_10853_b200 import data
    from paper_2405_10853_b200.config import TinyLMConfig
    from paper_2405_10853_b200.model import LossEvaluator
    from paper_2405_10853_b200.trainer import evaluate_mean_ce
    g = golden("norms_eval.npz")
    cfg = TinyLMConfig(vocab_size=256, context_len=128, n_layers=1, d_model=128, n_heads=2, seed=21)
    ev = LossEvaluator(cfg)
    corpus = data.tokenize_bytes(data.synth_corpus(99, 60_000), 128, 256)
    split = data.split_corpus(corpus, 2, 99, 0.1)
    ce = evaluate_mean_ce(ev, g["eval_params"], corpus, split.validation, 8, 3)
    assert abs(ce - float(g["eval_ce"])) <= 2e-2, (ce, float(g["eval_ce"]))


@pytest.mark.parametrize("n,offset", [(1_000_003, 0), (77_777, 1), (1023, 0), (5, 0)])
def test_round_norms_partial_warps_and_unaligned(n, offset):
    """The per-client norms are warp reductions: shapes whose last grid-stride iteration leaves a
    partial warp (n / 4 not a multiple of 32), the unaligned scalar-load path (offset by one
    float: ADVICE r1) and n < 4 must all give the f64 norms and the bit-exact step."""
    import ctypes as C
    from oracle import fedopt_ref
    from paper_2405_10853_b200 import ext
    rng = np.random.default_rng(n)
    K = 5
    w = rng.normal(0, 0.02, n).astype(np.float32)
    m = rng.normal(0, 1e-3, n).astype(np.float32)
    wk = [(w + rng.normal(0, 2e-3, n)).astype(np.float32) for _ in range(K)]
    nk = [1000 + 7 * k for k in range(K)]

    def dev(a):  # `offset` floats into a fresh allocation: 16-byte alignment broken when offset = 1
        t = torch.zeros(a.size + 4, dtype=torch.float32, device="cuda")
        t[offset:offset + a.size] = torch.from_numpy(a).cuda()
        return t[offset:offset + a.size]

    W, M, WK = dev(w), dev(m), [dev(x) for x in wk]
    wo, mo = dev(np.zeros(n, np.float32)), dev(np.zeros(n, np.float32))
    stats = torch.zeros(6 + K, dtype=torch.float64, device="cuda")
    bad = torch.empty(1, dtype=torch.int64, device="cuda")
    ext.call("fb_fedagg_round_norms_f32", (C.c_void_p * K)(*[t.data_ptr() for t in WK]), (C.c_int64 * K)(*nk), K, 1,
             W.data_ptr(), M.data_ptr(), wo.data_ptr(), mo.data_ptr(), n, 0.7, 0.9, 1, stats.data_ptr(),
             bad.data_ptr(), ext.stream_handle())
    s = stats.cpu().numpy()
    ref_w, ref_m = fedopt_ref.fed_round(w, m, wk, nk, 0.7, 0.9, True)
    assert np.array_equal(wo.cpu().numpy().view(np.uint32), ref_w.view(np.uint32))
    assert np.array_equal(mo.cpu().numpy().view(np.uint32), ref_m.view(np.uint32))
    assert int(bad.item()) >= n
    p = np.array(nk, np.float64) / sum(nk)
    avg = sum(p[k] * wk[k].astype(np.float64) for k in range(K))
    w64 = w.astype(np.float64)
    np.testing.assert_allclose(s[3], w64 @ w64, rtol=1e-12)
    np.testing.assert_allclose(s[4], avg @ avg, rtol=1e-9)
    np.testing.assert_allclose(s[5], (w64 - avg) @ (w64 - avg), rtol=1e-6)
    np.testing.assert_allclose(s[6:], [x.astype(np.float64) @ x.astype(np.float64) for x in wk], rtol=1e-12)
