"""Generate golden fixtures by running the REFERENCE (fedforge) in the build container.

Run from the repo root:  python tests/golden/make_golden.py
Requires /root/reference (read-only) — only this script touches it; the fixtures it
writes (tests/golden/*.npz / *.json) are what travels to the GPU box.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/reference/pkg/src")
torch.set_num_threads(1)

from fedforge import data as rdata  # noqa: E402
from fedforge import fedopt as rfed  # noqa: E402
from fedforge import localopt as ropt  # noqa: E402
from fedforge import model as rmodel  # noqa: E402
from fedforge import trainer as rtrain  # noqa: E402
from fedforge.messages import TrainTask  # noqa: E402
from fedforge.params import ParamVector, l2_norm  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_agg():
    out = {}
    for tag, K, N, seed in [("k8", 8, 4099, 0), ("k5", 5, 1031, 1), ("k1", 1, 257, 2), ("k13", 13, 515, 3)]:
        rng = np.random.default_rng(seed)
        w = rng.normal(0, 0.02, N).astype(np.float32)
        m = rng.normal(0, 1e-3, N).astype(np.float32)
        wks = [(w + rng.normal(0, 2e-3, N)).astype(np.float32) for _ in range(K)]
        nks = [1000 + 7 * k for k in range(K)]
        ids = list(rng.permutation(K))  # arrival order != id order
        out[f"{tag}_w"], out[f"{tag}_m"] = w, m
        out[f"{tag}_wk"] = np.stack(wks)
        out[f"{tag}_nk"] = np.array(nks)
        out[f"{tag}_arrival"] = np.array(ids)
        for det in (True, False):
            agg = rfed.AggregatorState(1, N, deterministic=det)
            for k in ids:
                agg.accumulate(rfed.ClientUpdate(int(k), 1, nks[k], w.astype(np.float64) - wks[k].astype(np.float64)))
            pg = agg.finalize()
            out[f"{tag}_pg_{'det' if det else 'stream'}"] = pg
            for eta, mu, nes in [(0.7, 0.9, True), (0.1, 0.9, False), (1.0, 0.0, True)]:
                opt = rfed.ServerOptState(ParamVector(m), eta, mu, nes)
                w2, opt2 = rfed.server_step(opt, ParamVector(w), pg, 1)
                key = f"{tag}_{'det' if det else 'stream'}_{eta}_{mu}_{int(nes)}"
                out[key + "_w"] = w2.data.copy()
                out[key + "_m"] = opt2.momentum.data.copy()
    np.savez_compressed(os.path.join(OUT, "agg.npz"), **out)


def gen_adamw():
    rng = np.random.default_rng(11)
    n, steps = 1024, 7
    cfg = ropt.AdamWConfig(weight_decay=0.01)
    p0 = rng.normal(size=n).astype(np.float32)
    grads = [rng.normal(size=n).astype(np.float32) * (10 ** rng.uniform(-6, 1, n)).astype(np.float32)
             for _ in range(steps)]
    grads[3][:5] = 0.0
    lrs = [1e-3 * (i + 1) for i in range(steps)]
    st = ropt.AdamWState.fresh(n, cfg)
    p = ParamVector(p0)
    ps, m1s, m2s, us = [], [], [], []
    for g, lr in zip(grads, lrs):
        p, st, u = ropt.adamw_step(st, p, ParamVector(g), lr)
        ps.append(p.data.copy()); m1s.append(st.m1.data.copy()); m2s.append(st.m2.data.copy()); us.append(u)
    # clip + micro mean
    gbig = (rng.normal(size=n) * 3).astype(np.float32)
    clipped, raw = ropt.clip_grad(ParamVector(gbig), 1.0)
    micro = [rng.normal(size=n).astype(np.float32) for _ in range(4)]
    acc = ropt.MicrobatchAccumulator(n)
    for g in micro:
        acc.add(ParamVector(g))
    np.savez_compressed(os.path.join(OUT, "adamw.npz"), p0=p0, grads=np.stack(grads), lrs=np.array(lrs),
                        p=np.stack(ps), m1=np.stack(m1s), m2=np.stack(m2s), applied=np.array(us),
                        clip_in=gbig, clip_out=clipped.data.copy(), clip_raw=raw,
                        micro=np.stack(micro), micro_avg=acc.average().data.copy(),
                        beta1=cfg.beta1, beta2=cfg.beta2, eps=cfg.eps, wd=cfg.weight_decay)


def gen_sched():
    rows = [(4e-4, 100, 88000, 1e-6), (3e-4, 100, 15000, 1e-5), (3e-4, 100, 13400, 1e-1),
            (2e-4, 100, 24800, 1e-1), (1e-3, 2, 1000, 0.1)]
    out = []
    for r in rows:
        s = ropt.ScheduleConfig(base_lr=r[0], warmup_steps=r[1], t_max=r[2], alpha_f=r[3])
        steps = [0, 1, 2, 50, 99, 100, 101, 500, 999, 1000, 5000, 13399, 13400, 24799, 24800, 88000, 100000]
        out.append({"cfg": r, "steps": steps, "lr": [ropt.lr_at(s, t) for t in steps]})
    with open(os.path.join(OUT, "sched.json"), "w") as fh:
        json.dump(out, fh)


def gen_data():
    out = {}
    text = rdata.synth_corpus(99, 400_000, "markov")
    out["markov_head"] = np.frombuffer(text[:512], dtype=np.uint8)
    out["markov_sha"] = np.array(hashlib.sha256(text).hexdigest())
    corpus = rdata.tokenize_bytes(text, 128, 256)
    split = rdata.split_corpus(corpus, 2, 99, 0.05)
    out["n_samples"] = corpus.n_samples
    out["val"] = split.validation
    for s in split.shards:
        out[f"shard{s.shard_id}"] = s.indices
        it = rdata.BatchIterator(corpus, s, 16, 99)
        out[f"order{s.shard_id}"] = it._order
        rows = []
        for off in (0, 4, 37):  # schedule offsets: seek(offset * micro * B)
            it.seek(off * 1 * 16)
            for _ in range(3):
                x, _ = it.next_batch()
                rows.append(x)
        out[f"batches{s.shard_id}"] = np.stack(rows)
    # 8-client split at a different seq len (C2-like, smaller corpus)
    corpus8 = rdata.tokenize_bytes(text, 1024, 32000)
    split8 = rdata.split_corpus(corpus8, 8, 99, 0.05)
    out["c8_val"] = split8.validation
    out["c8_shards"] = np.stack([s.indices for s in split8.shards])
    np.savez_compressed(os.path.join(OUT, "data.npz"), **out)


def gen_model():
    out = {}
    for tag, cfg in [
        ("micro", rmodel.TinyLMConfig(vocab_size=32, context_len=8, n_layers=2, d_model=8, n_heads=2, seed=5)),
        ("h3", rmodel.TinyLMConfig(vocab_size=48, context_len=16, n_layers=1, d_model=24, n_heads=3, seed=9)),
        ("nopos", rmodel.TinyLMConfig(vocab_size=32, context_len=8, n_layers=1, d_model=16, n_heads=2, use_alibi=False, seed=4)),
    ]:
        ev = rmodel.LossEvaluator(cfg)
        p = ev.init_params()
        rng = np.random.default_rng(7)
        pert = (p.data + rng.normal(0, 0.05, len(p)).astype(np.float32)).astype(np.float32)
        batch = rng.integers(0, cfg.vocab_size, size=(3, cfg.context_len))
        loss, grad = ev.loss_and_grad(ParamVector(pert), batch)
        out[f"{tag}_init"] = p.data.copy()
        out[f"{tag}_params"] = pert
        out[f"{tag}_batch"] = batch
        out[f"{tag}_loss"] = loss
        out[f"{tag}_grad"] = grad
        out[f"{tag}_names"] = np.array([e.tensor_name for e in ev.manifest.entries])
    c1 = rmodel.TinyLMConfig(vocab_size=256, context_len=128, n_layers=2, d_model=512, n_heads=8, seed=1234)
    p = rmodel.LossEvaluator(c1).init_params()
    out["c1_init_sha"] = np.array(sha(p.data))
    out["c1_init_n"] = len(p)
    out["c1_init_sub"] = p.data[::997].copy()
    np.savez_compressed(os.path.join(OUT, "model.npz"), **out)


def gen_round():
    """train_round on the reference's own test world (tests/test_trainer.py:171-200)."""
    cfg = rmodel.TinyLMConfig(vocab_size=64, context_len=16, n_layers=1, d_model=16, n_heads=2, seed=3)
    raw = (np.arange(4096) % 64).astype(np.uint8).tobytes()
    corpus = rdata.tokenize_bytes(raw, 16, vocab_size=64)
    shard = rdata.ShardSpec(0, np.arange(corpus.n_samples))
    ev = rmodel.LossEvaluator(cfg)
    params = ev.init_params()
    adamw = ropt.AdamWConfig()
    sched = ropt.ScheduleConfig(base_lr=1e-3, warmup_steps=5, t_max=500, alpha_f=0.01)
    task = TrainTask(round=2, client_id=0, local_steps=4, schedule_offset=4, batch_size=4,
                     micro_batches=2, seeds={"data": 7}, blob_key="k")
    it = rdata.BatchIterator(corpus, shard, 4, seed=7)
    upd, tele = rtrain.train_round(params, it, ev, adamw, sched, task)
    np.savez_compressed(os.path.join(OUT, "round.npz"), params=params.data, delta=upd.delta,
                        n_k=upd.n_k, tele=np.array([[t.step, t.loss, t.grad_norm_raw, t.grad_norm_applied, t.lr, t.param_norm] for t in tele]),
                        cursor=it.cursor)


def gen_c1():
    """C1: 2 clients x 4 steps x 16x128, FedAvg; 3 rounds of telemetry."""
    cfg = rmodel.TinyLMConfig(vocab_size=256, context_len=128, n_layers=2, d_model=512, n_heads=8, seed=1234)
    text = rdata.synth_corpus(99, 400_000, "markov")
    corpus = rdata.tokenize_bytes(text, 128, 256)
    split = rdata.split_corpus(corpus, 2, 99, 0.05)
    adamw = ropt.AdamWConfig()
    sched = ropt.ScheduleConfig(base_lr=1e-3, warmup_steps=2, t_max=1000, alpha_f=0.1)
    ev = rmodel.LossEvaluator(cfg)
    w = ev.init_params()
    opt = rfed.ServerOptState.fresh(len(w), 1.0, 0.0, True)
    its = [rdata.BatchIterator(corpus, s, 16, 99) for s in split.shards]
    tele_all, wsub, mean_losses = [], [], []
    for rnd in (1, 2, 3):
        agg = rfed.AggregatorState(rnd, len(w), deterministic=True)
        for k, s in enumerate(split.shards):
            task = TrainTask(rnd, k, 4, (rnd - 1) * 4, 16, 1, {"data": 99}, "k")
            upd, tele = rtrain.train_round(w, its[k], ev, adamw, sched, task)
            agg.accumulate(upd)
            tele_all.append([[t.step, t.loss, t.grad_norm_raw, t.grad_norm_applied, t.lr, t.param_norm] for t in tele])
            mean_losses.append(upd.local_metrics["mean_loss"])
        w, opt = rfed.server_step(opt, w, agg.finalize(), rnd)
        wsub.append(w.data[::1009].copy())
    np.savez_compressed(os.path.join(OUT, "c1.npz"), tele=np.array(tele_all), w_sub=np.stack(wsub),
                        mean_losses=np.array(mean_losses), w_norm=l2_norm(w))


def gen_norms_eval():
    """compute_round_norms (metrics.py:177-215) and evaluate_mean_ce (trainer.py:117-135)."""
    from fedforge.metrics import compute_round_norms
    g = np.load(os.path.join(OUT, "agg.npz"))
    w, m, wk, nk = g["k8_w"], g["k8_m"], g["k8_wk"], g["k8_nk"]
    deltas = [w.astype(np.float64) - wk[k].astype(np.float64) for k in range(8)]
    weights = [int(n) / int(nk.sum()) for n in nk]
    mom = g["k8_det_0.7_0.9_1_m"]
    rn = compute_round_norms(ParamVector(w), deltas, weights, ParamVector(mom), list(range(8)))
    cfg = rmodel.TinyLMConfig(vocab_size=256, context_len=128, n_layers=1, d_model=128, n_heads=2, seed=21)
    ev = rmodel.LossEvaluator(cfg)
    rng = np.random.default_rng(3)
    params = (ev.init_params().data + rng.normal(0, 0.05, ev.n_params).astype(np.float32)).astype(np.float32)
    corpus = rdata.tokenize_bytes(rdata.synth_corpus(99, 60_000, "markov"), 128, 256)
    split = rdata.split_corpus(corpus, 2, 99, 0.1)
    ce = rtrain.evaluate_mean_ce(ev, ParamVector(params), corpus, split.validation, 8, 3)
    np.savez_compressed(os.path.join(OUT, "norms_eval.npz"), global_norm=rn.global_norm,
                        per_client=np.array([rn.per_client_norms[k] for k in range(8)]),
                        avg_client_norm=rn.avg_client_norm, momentum_norm=rn.momentum_norm,
                        pseudograd_norm=rn.pseudograd_norm, eval_params=params, eval_ce=ce)


def gen_ckpt():
    """A FEDP blob encoded by the reference (params.encode_sections)."""
    from fedforge.params import encode_sections
    rng = np.random.default_rng(4)
    sections = {"round": 3, "global": ParamVector(rng.normal(size=257).astype(np.float32)),
                "momentum": ParamVector(rng.normal(size=257).astype(np.float32)),
                "server_opt": {"eta": 0.7, "mu": 0.9, "nesterov": True}, "lr": 0.25,
                "delta": rng.normal(size=31), "config_hash": "abc"}
    with open(os.path.join(OUT, "ckpt_ref.fedp"), "wb") as fh:
        fh.write(encode_sections(sections))


if __name__ == "__main__":
    which = sys.argv[1:] or ["agg", "adamw", "sched", "data", "model", "round", "c1", "norms_eval", "ckpt"]
    for name in which:
        globals()["gen_" + name]()
        print("wrote", name)
