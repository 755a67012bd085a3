"""The reference's own aggregation / server-step tests, replayed against the drop-in
(reference tests/test_fedopt.py), plus bitwise parity of host-format updates."""
import itertools

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


def api():
    from paper_2405_10853_b200 import fedopt, params
    return fedopt, params


def upd(cid, rnd, n_k, delta):
    f, _ = api()
    return f.ClientUpdate(cid, rnd, n_k, np.asarray(delta, dtype=np.float64))


@pytest.mark.parametrize("tag", ["k8", "k5", "k1", "k13"])
@pytest.mark.parametrize("det", [True, False])
def test_host_updates_bitwise(tag, det):
    f, P = api()
    g = golden("agg.npz")
    w, m, wk, nk, arr = g[f"{tag}_w"], g[f"{tag}_m"], g[f"{tag}_wk"], g[f"{tag}_nk"], g[f"{tag}_arrival"]
    agg = f.AggregatorState(1, w.size, deterministic=det)
    for k in arr:
        agg.accumulate(upd(int(k), 1, int(nk[k]), w.astype(np.float64) - wk[k].astype(np.float64)))
    pg = agg.finalize()
    mode = "det" if det else "stream"
    assert np.array_equal(np.asarray(pg).view(np.uint64), g[f"{tag}_pg_{mode}"].view(np.uint64))
    for eta, mu, nes in [(0.7, 0.9, True), (0.1, 0.9, False), (1.0, 0.0, True)]:
        opt = f.ServerOptState(P.ParamVector(m), eta, mu, nes)
        w2, opt2 = f.server_step(opt, P.ParamVector(w), pg, 1)
        key = f"{tag}_{mode}_{eta}_{mu}_{int(nes)}"
        assert np.array_equal(w2.data.view(np.uint32), g[key + "_w"].view(np.uint32))
        assert np.array_equal(opt2.momentum.data.view(np.uint32), g[key + "_m"].view(np.uint32))
        # numpy pseudo-gradient in -> same result
        w3, _ = f.server_step(opt, P.ParamVector(w), np.asarray(pg), 1)
        assert w3.bitwise_equal(w2)


def test_device_updates_bitwise():
    f, P = api()
    g = golden("agg.npz")
    w, m, wk, nk, arr = g["k8_w"], g["k8_m"], g["k8_wk"], g["k8_nk"], g["k8_arrival"]
    W = torch.from_numpy(w).cuda()
    agg = f.AggregatorState(1, w.size, deterministic=True)
    for k in arr:
        agg.accumulate(f.DeviceClientUpdate(int(k), 1, int(nk[k]), torch.from_numpy(wk[k]).cuda(), W))
    opt = f.ServerOptState(f.DeviceVector(torch.from_numpy(m).cuda()), 0.7, 0.9, True)
    w2, opt2 = f.server_step(opt, f.DeviceVector(W), agg.finalize(), 1)
    assert np.array_equal(w2.data.view(np.uint32), g["k8_det_0.7_0.9_1_w"].view(np.uint32))
    assert np.array_equal(opt2.momentum.data.view(np.uint32), g["k8_det_0.7_0.9_1_m"].view(np.uint32))


@pytest.mark.parametrize("device_updates", [True, False])
def test_weighted_sum_is_the_reference_running_sum(device_updates):
    """AggregatorState.weighted_sum (fedopt.py:95): the f64 running sum of n_k * delta_k in
    arrival order, bitwise — for device end weights and for host f64 deltas."""
    f, P = api()
    g = golden("agg.npz")
    w, wk, nk, arr = g["k13_w"], g["k13_wk"], g["k13_nk"], g["k13_arrival"]
    W = torch.from_numpy(w).cuda()
    agg = f.AggregatorState(1, w.size, deterministic=True)
    ref = np.zeros(w.size)
    for k in arr:
        delta = w.astype(np.float64) - wk[k].astype(np.float64)
        ref += int(nk[k]) * delta
        u = (f.DeviceClientUpdate(int(k), 1, int(nk[k]), torch.from_numpy(wk[k]).cuda(), W) if device_updates
             else f.ClientUpdate(int(k), 1, int(nk[k]), delta))
        agg.accumulate(u)
    assert np.array_equal(agg.weighted_sum.view(np.uint64), ref.view(np.uint64))


class TestReferenceAggregatorTests:
    def test_first_contribution(self):
        f, _ = api()
        agg = f.AggregatorState(1, 2)
        agg.accumulate(upd(0, 1, 2, [1.0, 0.0]))
        assert agg.weighted_sum.tolist() == [2.0, 0.0] and agg.total_weight == 2 and agg.contributors == {0}

    def test_errors(self):
        f, P = api()
        from paper_2405_10853_b200.errors import AggregationError, ParamError
        agg = f.AggregatorState(1, 1)
        agg.accumulate(upd(3, 1, 1, [1.0]))
        with pytest.raises(AggregationError, match="duplicate"):
            agg.accumulate(upd(3, 1, 1, [2.0]))
        with pytest.raises(AggregationError, match="round"):
            f.AggregatorState(1, 1).accumulate(upd(0, 2, 1, [1.0]))
        with pytest.raises(ParamError):
            f.AggregatorState(1, 2).accumulate(upd(0, 1, 1, [1.0]))
        with pytest.raises(AggregationError):
            f.AggregatorState(0, 1).finalize()

    def test_means(self, rng):
        f, _ = api()
        delta = rng.normal(size=13)
        agg = f.AggregatorState(2, 13)
        agg.accumulate(upd(5, 2, 937, delta))
        assert np.array_equal(np.asarray(agg.finalize()), delta)
        agg = f.AggregatorState(0, 2)
        agg.accumulate(upd(0, 0, 3, [1.0, 2.0])).accumulate(upd(1, 0, 3, [3.0, 4.0]))
        assert np.asarray(agg.finalize()).tolist() == [2.0, 3.0]
        agg = f.AggregatorState(0, 1)
        agg.accumulate(upd(0, 0, 1, [4.0])).accumulate(upd(1, 0, 3, [0.0]))
        assert np.asarray(agg.finalize()).tolist() == [1.0]

    def test_orders_and_merge(self, rng):
        f, _ = api()
        ups = [upd(i, 1, int(n), rng.normal(size=5)) for i, n in enumerate(rng.integers(1, 50, size=3))]
        ref = sum(u.n_k * u.delta for u in ups) / sum(u.n_k for u in ups)
        for perm in itertools.permutations(ups):
            agg = f.AggregatorState(1, 5)
            for u in perm:
                agg.accumulate(u)
            assert np.allclose(np.asarray(agg.finalize()), ref, rtol=1e-6)
        ups = [upd(i, 1, int(n), rng.normal(size=7)) for i, n in enumerate(rng.integers(1, 100, size=8))]
        res = []
        for s in range(10):
            agg = f.AggregatorState(1, 7, deterministic=True)
            for i in np.random.default_rng(s).permutation(8):
                agg.accumulate(ups[i])
            res.append(np.asarray(agg.finalize()))
        assert all(np.array_equal(r.view(np.uint64), res[0].view(np.uint64)) for r in res)
        whole = f.AggregatorState(1, 7)
        for u in ups:
            whole.accumulate(u)
        for mask in (1, 37, 200, 254):
            a, b = f.AggregatorState(1, 7), f.AggregatorState(1, 7)
            for i, u in enumerate(ups):
                (a if mask & (1 << i) else b).accumulate(u)
            mg = a.merge(b)
            assert mg.total_weight == whole.total_weight and mg.contributors == set(range(8))
            assert np.allclose(np.asarray(mg.finalize()), np.asarray(whole.finalize()), rtol=1e-6)

    def test_server_step_known_answers(self):
        f, P = api()
        from paper_2405_10853_b200.errors import ParamError
        w, _ = f.server_step(f.ServerOptState.fresh(2, 1.0, 0.0), P.ParamVector(np.ones(2, np.float32)), np.ones(2))
        assert w.data.tolist() == [0.0, 0.0]
        w, o2 = f.server_step(f.ServerOptState.fresh(1, 0.1, 0.9), P.ParamVector(np.ones(1, np.float32)), np.array([0.5]))
        assert o2.momentum.data[0] == pytest.approx(0.5) and float(w.data[0]) == pytest.approx(0.905, rel=1e-6)
        opt = f.ServerOptState(P.ParamVector(np.array([2.0], np.float32)), 0.1, 0.5, True)
        w = P.ParamVector(np.ones(1, np.float32))
        for t in range(5):
            w, opt = f.server_step(opt, w, np.zeros(1))
            assert P.l2_norm(opt.momentum) == pytest.approx(2.0 * 0.5 ** (t + 1), rel=1e-6)
        with pytest.raises(ParamError, match="round 9"):
            f.server_step(f.ServerOptState.fresh(1, 1.0, 0.0), P.ParamVector(np.array([3.0e38], np.float32)),
                          np.array([-3.0e38]), round_num=9)
        with pytest.raises(ParamError):
            f.ServerOptState.fresh(1, eta=0.0, mu=0.5)
        with pytest.raises(ParamError):
            f.ServerOptState.fresh(1, eta=0.1, mu=1.0)
