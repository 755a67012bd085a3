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
