"""Round driver, Flower façade and device checkpoint on the GPU."""
import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


def _c1():
    from paper_2405_10853_b200 import data
    from paper_2405_10853_b200.config import AdamWConfig, ScheduleConfig, TinyLMConfig
    cfg = TinyLMConfig(vocab_size=256, context_len=128, n_layers=2, d_model=512, n_heads=8, seed=1234)
    corpus = data.tokenize_bytes(data.synth_corpus(99, 400_000), 128, 256)
    return cfg, corpus, data.split_corpus(corpus, 2, 99, 0.05), AdamWConfig(), ScheduleConfig(1e-3, 2, 1000, 0.1)


def test_federation_round1_vs_reference(tmp_path):
    from paper_2405_10853_b200.checkpoint import read_checkpoint
    from paper_2405_10853_b200.federation import Federation
    g = golden("c1.npz")
    cfg, corpus, split, adamw, sched = _c1()
    fed = Federation(cfg, adamw, sched, corpus, split, batch_size=16, micro_batches=1, local_steps=4, server_eta=1.0,
                     server_mu=0.0, eval_batches=2)
    w, opt = fed.init_state()
    res = fed.run_round(w, opt, 1, checkpoint_path=tmp_path / "r1.fedp")
    means = [res.client_metrics[k]["mean_loss"] for k in range(2)]
    assert np.max(np.abs(np.array(means) - g["mean_losses"][:2])) <= 2e-2
    err = np.abs(res.params.tensor.cpu().numpy()[::1009] - g["w_sub"][0])
    assert np.median(err) <= 5e-4
    assert res.norms.pseudograd_norm > 0 and len(res.norms.per_client_norms) == 2
    assert np.isfinite(res.val_loss) and res.val_loss < 5.6
    assert res.checkpoint.wait() > 0
    ck = read_checkpoint(tmp_path / "r1.fedp")
    assert ck["round"] == 1 and ck["global"].bitwise_equal(res.params.to_param_vector())
    res2 = fed.run_round(res.params, res.opt, 2)
    assert all(np.isfinite(res2.client_metrics[k]["mean_loss"]) for k in range(2))


def test_flower_facade_fit_and_aggregate():
    from paper_2405_10853_b200 import data
    from paper_2405_10853_b200.flower import B200Client, FedOptStrategy
    from paper_2405_10853_b200.model import LossEvaluator
    cfg, corpus, split, adamw, sched = _c1()
    ev = LossEvaluator(cfg)
    clients = [B200Client(k, ev, data.BatchIterator(corpus, split.shards[k], 16, 99), adamw, sched, local_steps=2,
                          batch_size=16) for k in range(2)]
    params = clients[0].get_parameters()
    strat = FedOptStrategy(ev, params, eta=0.7, mu=0.9, nesterov=True)
    results = [c.fit(params, {"server_round": 1}) for c in clients]
    new_params, metrics = strat.aggregate_fit(1, results, [])
    assert len(new_params) == len(params) and metrics["n_contributors"] == 2
    assert abs(sum(metrics["weights"].values()) - 1.0) < 1e-12
    assert all(np.isfinite(a).all() for a in new_params)


def test_async_checkpoint_of_device_vectors(tmp_path):
    """(f)4: the round-boundary checkpoint snapshots device vectors with async D2H copies on a
    side stream (the caller continues at once) and writes the same bytes as the host encoder."""
    from paper_2405_10853_b200.checkpoint import decode_sections, encode_sections, write_checkpoint_async
    from paper_2405_10853_b200.fedopt import DeviceVector
    from paper_2405_10853_b200.params import ParamVector
    n = 10_000_019
    w = torch.randn(n, device="cuda")
    m = torch.randn(n, device="cuda") * 1e-3
    w2 = w * 2  # produced on the current stream right before the snapshot
    h = write_checkpoint_async({"round": 7, "global": DeviceVector(w2), "momentum": DeviceVector(m),
                                "server_opt": {"eta": 0.7, "mu": 0.9, "nesterov": True}}, tmp_path / "a.fedp")
    nbytes = h.wait()
    raw = open(tmp_path / "a.fedp", "rb").read()
    assert nbytes == len(raw)
    want = encode_sections({"round": 7, "global": ParamVector(w2.cpu().numpy()),
                            "momentum": ParamVector(m.cpu().numpy()),
                            "server_opt": {"eta": 0.7, "mu": 0.9, "nesterov": True}})
    assert raw == want
    dec = decode_sections(raw)
    assert dec["global"].bitwise_equal(ParamVector(w2.cpu().numpy())) and dec["round"] == 7


def test_concurrent_clients_match_sequential():
    """Federation(concurrent_clients=2): this GPU's clients train two at a time on their own
    streams; with the deterministic kernels the round's global model is bitwise the
    sequential one (same per-client computations, same fused round end)."""
    from paper_2405_10853_b200.federation import Federation
    from paper_2405_10853_b200.model import set_deterministic
    cfg, corpus, split, adamw, sched = _c1()
    kw = dict(batch_size=16, micro_batches=2, local_steps=3, server_eta=0.7, server_mu=0.9)
    set_deterministic(True)
    try:
        outs = []
        for P in (1, 2):
            fed = Federation(cfg, adamw, sched, corpus, split, concurrent_clients=P, **kw)
            w, opt = fed.init_state()
            res = fed.run_round(w, opt, 1)
            res = fed.run_round(res.params, res.opt, 2)
            outs.append((res.params.tensor.cpu().numpy(), res.opt.momentum.tensor.cpu().numpy(), res.client_metrics))
    finally:
        set_deterministic(True)
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert np.array_equal(outs[0][1].view(np.uint32), outs[1][1].view(np.uint32))
    assert outs[0][2] == outs[1][2]
