"""Model / round parity on the B200 through the public drop-in API.

Tolerances (bf16 tensor-core GEMMs vs the reference's fp32 CPU model):
  * loss of one micro-batch: |dL| <= 2e-2 absolute
  * gradient: ||g - g_ref|| <= 5e-2 ||g_ref||  and cosine >= 0.998
  * round-mean loss after each round: <= 2e-2 absolute (BASELINE north star)
Index work (cursor, lr) is exact."""
import math

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import data_ref, model_ref

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("V,ctx,L,d,H,alibi,B,T", [(256, 128, 2, 128, 2, True, 2, 128),
                                                   (320, 128, 1, 256, 2, True, 2, 128),
                                                   (256, 384, 2, 192, 3, False, 1, 384),
                                                   (512, 256, 1, 768, 12, True, 1, 256)])
def test_loss_and_grad_vs_oracle(V, ctx, L, d, H, alibi, B, T):
    from paper_2405_10853_b200.config import TinyLMConfig
    from paper_2405_10853_b200.model import LossEvaluator
    cfg = TinyLMConfig(vocab_size=V, context_len=ctx, n_layers=L, d_model=d, n_heads=H, use_alibi=alibi, seed=7)
    ev = LossEvaluator(cfg)
    rng = np.random.default_rng(0)
    p = ev.init_params().data.copy()
    p += rng.normal(0, 0.02, p.size).astype(np.float32)  # non-zero head
    batch = rng.integers(0, V, size=(B, T))
    loss, grad = ev.loss_and_grad(p, batch)
    torch.set_num_threads(8)
    ref_loss, ref_grad = model_ref.loss_and_grad(p, batch, V, ctx, L, d, H, alibi)
    assert abs(loss - ref_loss) <= 2e-2, (loss, ref_loss)
    rel = np.linalg.norm(grad - ref_grad) / np.linalg.norm(ref_grad)
    cos = float(np.dot(grad, ref_grad) / (np.linalg.norm(grad) * np.linalg.norm(ref_grad)))
    assert rel <= 5e-2 and cos >= 0.998, (rel, cos)
    # per-tensor check (every manifest entry gets a gradient)
    for e in ev.manifest:
        g, r = grad[e.offset:e.offset + e.size], ref_grad[e.offset:e.offset + e.size]
        if np.linalg.norm(r) > 1e-6:
            assert np.linalg.norm(g - r) <= 0.1 * np.linalg.norm(r) + 1e-6, e.tensor_name
    assert ev.loss(p, batch) == pytest.approx(loss, abs=1e-6)


def test_untrained_loss_is_log_vocab():
    from paper_2405_10853_b200.config import TinyLMConfig
    from paper_2405_10853_b200.model import LossEvaluator
    cfg = TinyLMConfig(vocab_size=256, context_len=128, n_layers=2, d_model=128, n_heads=2)
    ev = LossEvaluator(cfg)
    loss = ev.loss(ev.init_params(), np.random.default_rng(0).integers(0, 256, size=(4, 128)))
    assert loss == pytest.approx(math.log(256), abs=1e-3)


def test_token_range_error():
    from paper_2405_10853_b200.config import TinyLMConfig
    from paper_2405_10853_b200.errors import TokenRangeError
    from paper_2405_10853_b200.model import LossEvaluator
    ev = LossEvaluator(TinyLMConfig(vocab_size=64, context_len=128, n_layers=1, d_model=64, n_heads=1))
    b = np.zeros((2, 128), dtype=np.int64)
    b[1, 3] = 64
    with pytest.raises(TokenRangeError, match=r"row 1, position 3"):
        ev.loss(ev.init_params(), b)


def _c1_world():
    from paper_2405_10853_b200 import data
    from paper_2405_10853_b200.config import AdamWConfig, ScheduleConfig, TinyLMConfig
    cfg = TinyLMConfig(vocab_size=256, context_len=128, n_layers=2, d_model=512, n_heads=8, seed=1234)
    corpus = data.tokenize_bytes(data.synth_corpus(99, 400_000), 128, 256)
    split = data.split_corpus(corpus, 2, 99, 0.05)
    return cfg, corpus, split, AdamWConfig(), ScheduleConfig(base_lr=1e-3, warmup_steps=2, t_max=1000, alpha_f=0.1)


def test_c1_round1_free_running_vs_reference():
    """C1: 2 clients x 4 steps x 16x128, FedAvg — round 1 through the drop-in
    API (train_round -> AggregatorState -> server_step) against the reference run."""
    from paper_2405_10853_b200 import data
    from paper_2405_10853_b200.config import TrainTask, lr_at
    from paper_2405_10853_b200.fedopt import AggregatorState, DeviceVector, ServerOptState, server_step
    from paper_2405_10853_b200.model import LossEvaluator
    from paper_2405_10853_b200.trainer import train_round
    g = golden("c1.npz")
    cfg, corpus, split, adamw, sched = _c1_world()
    ev = LossEvaluator(cfg)
    w = DeviceVector(torch.from_numpy(ev.init_params().data.copy()).cuda())
    opt = ServerOptState(DeviceVector(torch.zeros(len(w), device="cuda")), 1.0, 0.0, True)
    its = [data.BatchIterator(corpus, s, 16, 99) for s in split.shards]
    agg = AggregatorState(1, len(w), deterministic=True)
    tele_all, means = [], []
    for k in range(2):
        upd, tele = train_round(w, its[k], ev, adamw, sched, TrainTask(1, k, 4, 0, 16, 1, {"data": 99}, "k"))
        assert its[k].cursor == 4 * 16
        assert [t.lr for t in tele] == [lr_at(sched, s) for s in range(4)]
        assert upd.n_k == split.shards[k].n_k
        agg.accumulate(upd)
        tele_all.append([[t.step, t.loss, t.grad_norm_raw, t.grad_norm_applied, t.lr, t.param_norm] for t in tele])
        means.append(upd.local_metrics["mean_loss"])
    w, opt = server_step(opt, w, agg.finalize(), 1)
    tele_all, ref = np.array(tele_all), g["tele"][:2]
    assert np.max(np.abs(tele_all[:, :, 1] - ref[:, :, 1])) <= 2e-2
    assert np.max(np.abs(np.array(means) - g["mean_losses"][:2])) <= 2e-2
    assert np.array_equal(tele_all[:, :, 4], ref[:, :, 4])          # lr exact
    np.testing.assert_allclose(tele_all[:, :, 5], ref[:, :, 5], rtol=2e-3)  # param norm
    np.testing.assert_allclose(tele_all[:, :, 2], ref[:, :, 2], rtol=2e-2)  # raw grad norm
    err = np.abs(w.tensor.cpu().numpy()[::1009] - g["w_sub"][0])
    assert np.median(err) <= 5e-4 and err.max() <= 1e-2, (np.median(err), err.max())


def test_c1_round2_teacher_forced_vs_oracle():
    """Round 2 of C1 hits two loss spikes (grad norm 22.9 and 59.4 in the fp32 reference).
    Free-running bf16 and fp32 trajectories separate there (fresh-moment AdamW turns
    0.5% gradient noise into sign flips of tiny coordinates), so round 2 is checked
    teacher-forced: our loss/grad at the oracle's exact params and batch of every step."""
    from paper_2405_10853_b200.model import LossEvaluator
    from oracle import fedopt_ref, localopt_ref
    torch.set_num_threads(16)
    g = golden("c1.npz")
    cfg, corpus, split, adamw, sched = _c1_world()
    ev = LossEvaluator(cfg)
    tok = corpus.tokens
    orders = [data_ref.client_order(s.indices, k, 99) for k, s in enumerate(split.shards)]
    w = model_ref.init_flat(256, 128, 2, 512, 1234)
    m = np.zeros_like(w)
    for rnd in (1, 2):
        ws = []
        for k in range(2):
            p, m1, m2 = w.copy(), np.zeros_like(w), np.zeros_like(w)
            cur = (rnd - 1) * 64
            for s in range(4):
                batch = data_ref.gather(tok, 128, data_ref.batch_rows(orders[k], cur, 16))
                cur += 16
                lo, go = model_ref.loss_and_grad(p, batch, 256, 128, 2, 512, 8)
                assert lo == pytest.approx(float(g["tele"][2 * (rnd - 1) + k, s, 1]), abs=1e-4)
                if rnd == 2:
                    lg, gg = ev.loss_and_grad(p, batch)
                    assert abs(lg - lo) <= 1e-2, (k, s, lg, lo)
                    assert np.linalg.norm(gg - go) <= 2e-2 * np.linalg.norm(go), (k, s)
                go, _ = localopt_ref.clip(go, 1.0)
                p, m1, m2, _ = localopt_ref.adamw(p, go, m1, m2, s + 1, localopt_ref.lr_at(1e-3, 2, 1000, 0.1, (rnd - 1) * 4 + s))
            ws.append(p)
        w, m = fedopt_ref.fed_round(w, m, ws, [s.n_k for s in split.shards], 1.0, 0.0, True)
