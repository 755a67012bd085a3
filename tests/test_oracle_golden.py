"""Pin the CPU oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py) and against the reference's own known answers."""
import json
import math
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN, golden
from oracle import data_ref, fedopt_ref, localopt_ref, model_ref, round_ref

torch.set_num_threads(1)


@pytest.mark.parametrize("tag", ["k8", "k5", "k1", "k13"])
@pytest.mark.parametrize("mode", ["det", "stream"])
def test_aggregation_bitwise_vs_reference(tag, mode):
    g = golden("agg.npz")
    w, m, wk, nk, arr = g[f"{tag}_w"], g[f"{tag}_m"], g[f"{tag}_wk"], g[f"{tag}_nk"], g[f"{tag}_arrival"]
    deltas = [w.astype(np.float64) - wk[k].astype(np.float64) for k in arr]
    pg = fedopt_ref.finalize_deltas(deltas, [nk[k] for k in arr], list(arr), deterministic=(mode == "det"))
    assert np.array_equal(pg.view(np.uint64), g[f"{tag}_pg_{mode}"].view(np.uint64))
    for eta, mu, nes in [(0.7, 0.9, True), (0.1, 0.9, False), (1.0, 0.0, True)]:
        key = f"{tag}_{mode}_{eta}_{mu}_{int(nes)}"
        w2, m2 = fedopt_ref.server_step(w, m, pg, eta, mu, nes)
        assert np.array_equal(w2.view(np.uint32), g[key + "_w"].view(np.uint32))
        assert np.array_equal(m2.view(np.uint32), g[key + "_m"].view(np.uint32))


def test_server_step_hand_recurrence():
    # reference tests/test_fedopt.py:179-186
    w, m = fedopt_ref.server_step(np.array([1.0], np.float32), np.zeros(1, np.float32), np.array([0.5]), 0.1, 0.9)
    assert m[0] == pytest.approx(0.5) and float(w[0]) == pytest.approx(0.905, rel=1e-6)


def test_adamw_bitwise_vs_reference():
    g = golden("adamw.npz")
    p = g["p0"]
    m1 = np.zeros_like(p)
    m2 = np.zeros_like(p)
    for t in range(g["grads"].shape[0]):
        p, m1, m2, u = localopt_ref.adamw(p, g["grads"][t], m1, m2, t + 1, float(g["lrs"][t]),
                                          float(g["beta1"]), float(g["beta2"]), float(g["eps"]), float(g["wd"]))
        assert np.array_equal(p, g["p"][t]) and np.array_equal(m1, g["m1"][t]) and np.array_equal(m2, g["m2"][t])
        assert u == g["applied"][t]
    c, raw = localopt_ref.clip(g["clip_in"], 1.0)
    assert raw == float(g["clip_raw"]) and np.array_equal(c, g["clip_out"])
    assert np.array_equal(localopt_ref.micro_mean(list(g["micro"])), g["micro_avg"])


def test_schedule_vs_reference():
    with open(os.path.join(GOLDEN, "sched.json")) as fh:
        rows = json.load(fh)
    for r in rows:
        for s, lr in zip(r["steps"], r["lr"]):
            assert localopt_ref.lr_at(*r["cfg"], s) == lr


def test_data_indices_vs_reference():
    g = golden("data.npz")
    text = data_ref.markov_bytes(99, 400_000)
    assert np.array_equal(np.frombuffer(text[:512], np.uint8), g["markov_head"])
    import hashlib
    assert hashlib.sha256(text).hexdigest() == str(g["markov_sha"])
    tok = data_ref.tokens_of(text)
    n = data_ref.n_samples(tok, 128)
    assert n == int(g["n_samples"])
    val, shards = data_ref.split(n, 2, 99, 0.05)
    assert np.array_equal(val, g["val"])
    for k in range(2):
        assert np.array_equal(shards[k], g[f"shard{k}"])
        order = data_ref.client_order(shards[k], k, 99)
        assert np.array_equal(order, g[f"order{k}"])
        got = []
        for off in (0, 4, 37):
            cur = off * 16
            for _ in range(3):
                got.append(data_ref.gather(tok, 128, data_ref.batch_rows(order, cur, 16)))
                cur += 16
        assert np.array_equal(np.stack(got), g[f"batches{k}"])
    tok8 = data_ref.tokens_of(text)
    val8, shards8 = data_ref.split(data_ref.n_samples(tok8, 1024), 8, 99, 0.05)
    assert np.array_equal(val8, g["c8_val"]) and np.array_equal(np.stack(shards8), g["c8_shards"])


@pytest.mark.parametrize("tag,cfg", [("micro", (32, 8, 2, 8, 2, True, 5)),
                                     ("h3", (48, 16, 1, 24, 3, True, 9)),
                                     ("nopos", (32, 8, 1, 16, 2, False, 4))])
def test_model_vs_reference(tag, cfg):
    g = golden("model.npz")
    V, ctx, L, d, H, alibi, seed = cfg
    assert [n for n, _ in model_ref.manifest(V, ctx, L, d, alibi)] == list(g[f"{tag}_names"])
    init = model_ref.init_flat(V, ctx, L, d, seed, alibi)
    assert np.array_equal(init, g[f"{tag}_init"])
    loss, grad = model_ref.loss_and_grad(g[f"{tag}_params"], g[f"{tag}_batch"], V, ctx, L, d, H, alibi)
    assert abs(loss - float(g[f"{tag}_loss"])) <= 1e-6
    np.testing.assert_allclose(grad, g[f"{tag}_grad"], rtol=1e-4, atol=1e-7)


def test_c1_init_bitwise():
    g = golden("model.npz")
    init = model_ref.init_flat(256, 128, 2, 512, 1234)
    import hashlib
    assert init.size == int(g["c1_init_n"])
    assert hashlib.sha256(init.tobytes()).hexdigest() == str(g["c1_init_sha"])


def test_train_round_vs_reference():
    g = golden("round.npz")
    raw = (np.arange(4096) % 64).astype(np.uint8).tobytes()
    tok = data_ref.tokens_of(raw)
    shard = np.arange(data_ref.n_samples(tok, 16))
    order = data_ref.client_order(shard, 0, 7)
    w, tele = round_ref.train_round(
        g["params"], tok, 16, order, shard.size, (64, 16, 1, 16, 2, True),
        dict(beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=1e-5, clip_norm=1.0),
        (1e-3, 5, 500, 0.01), local_steps=4, schedule_offset=4, batch_size=4, micro_batches=2)
    delta = g["params"].astype(np.float64) - w.astype(np.float64)
    np.testing.assert_allclose(delta, g["delta"], rtol=1e-4, atol=1e-9)
    np.testing.assert_allclose(np.array(tele), g["tele"], rtol=1e-5)


def test_c1_three_rounds_and_round2_is_chaotic():
    """The oracle reproduces the reference's 3-round C1 run (c1.npz) and, from start weights
    perturbed by 1e-4 relative (40x below bf16 resolution), its own round-2 round-mean loss
    moves by > 0.3: the reference algorithm is chaotic at the round-2 grad-norm spikes, which
    is why free-running GPU rounds 2-3 are bounded by this envelope and the strict 2e-2 bound
    is applied from a common start model (tests/test_gpu_round_parity.py)."""
    import torch
    from oracle import fedopt_ref
    torch.set_num_threads(min(8, os.cpu_count() or 1))
    g = golden("c1.npz")
    tok = data_ref.tokens_of(data_ref.markov_bytes(99, 400_000))
    _, shards = data_ref.split(data_ref.n_samples(tok, 128), 2, 99, 0.05)
    orders = [data_ref.client_order(s, k, 99) for k, s in enumerate(shards)]
    opt = dict(beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=1e-5, clip_norm=1.0)

    def run(w):
        m = np.zeros_like(w)
        means = []
        for rnd in (1, 2, 3):
            ws = []
            for k, s in enumerate(shards):
                wk, tele = round_ref.train_round(w, tok, 128, orders[k], s.size, (256, 128, 2, 512, 8, True), opt,
                                                 (1e-3, 2, 1000, 0.1), local_steps=4, schedule_offset=(rnd - 1) * 4,
                                                 batch_size=16, micro_batches=1)
                ws.append(wk)
                means.append(np.mean([t[1] for t in tele]))
            w, m = fedopt_ref.fed_round(w, m, ws, [s.size for s in shards], 1.0, 0.0, True)
        return np.array(means)

    w0 = model_ref.init_flat(256, 128, 2, 512, 1234)
    np.testing.assert_allclose(run(w0), g["mean_losses"], atol=2e-3)
    pert = (w0 * (1 + 1e-4 * np.random.default_rng(1).standard_normal(w0.size))).astype(np.float32)
    d = np.abs(run(pert) - g["mean_losses"])
    assert d[:2].max() < 2e-3          # round 1: insensitive
    assert d[2] > 0.3                  # round 2, client 0: the spike moves the round mean by ~0.35
