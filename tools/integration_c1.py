"""C1 round through the two integration paths of INTEGRATION.md §1, timed on one GPU.

(a) "import swap": what the UNMODIFIED fedforge runtime does around the drop-in calls:
    ClientWorker.execute (cluster.py:170-203) materialises update.delta (f64, host) and
    encodes the FEDP update blob; the server decodes it (cluster.py:385-394), accumulates
    host ClientUpdates, finalizes, server_step, then compute_round_norms over the host
    deltas (cluster.py:519-525).
(b) fast path: federation.Federation — end weights stay in HBM, one fused
    aggregation + outer step + round norms pass.
Both produce the same global model (bitwise). Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import data  # noqa: E402
from paper_2405_10853_b200.checkpoint import decode_sections, encode_sections  # noqa: E402
from paper_2405_10853_b200.config import AdamWConfig, ScheduleConfig, TinyLMConfig, TrainTask  # noqa: E402
from paper_2405_10853_b200.federation import Federation  # noqa: E402
from paper_2405_10853_b200.fedopt import AggregatorState, ClientUpdate, ServerOptState, server_step  # noqa: E402
from paper_2405_10853_b200.model import LossEvaluator, set_deterministic  # noqa: E402
from paper_2405_10853_b200.params import ParamVector  # noqa: E402
from paper_2405_10853_b200.telemetry import compute_round_norms  # noqa: E402
from paper_2405_10853_b200.trainer import train_round  # noqa: E402

cfg = TinyLMConfig(vocab_size=256, context_len=128, n_layers=2, d_model=512, n_heads=8, seed=1234)
corpus = data.tokenize_bytes(data.synth_corpus(99, 400_000), 128, 256)
split = data.split_corpus(corpus, 2, 99, 0.05)
adamw, sched = AdamWConfig(), ScheduleConfig(1e-3, 2, 1000, 0.1)
ev = LossEvaluator(cfg)
w0 = ev.init_params()
set_deterministic(True)  # both paths train bit-identical clients, so their global models can be compared bitwise


def swap_round():
    its = [data.BatchIterator(corpus, s, 16, 99) for s in split.shards]
    t0 = time.perf_counter()
    blobs = []
    t_train = 0.0
    for k in range(2):
        a = time.perf_counter()
        u, tele = train_round(w0, its[k], ev, adamw, sched, TrainTask(1, k, 4, 0, 16, 1, {"data": 99}, "k"))
        t_train += time.perf_counter() - a
        blobs.append(encode_sections({"round": 1, "client_id": k, "n_k": u.n_k, "delta": u.delta,
                                      "local_metrics": u.local_metrics}))
    agg = AggregatorState(1, len(w0), deterministic=True)
    for b in blobs:
        s = decode_sections(b)
        agg.accumulate(ClientUpdate(s["client_id"], s["round"], s["n_k"], s["delta"], s["local_metrics"]))
    weights = agg.weights()
    opt = ServerOptState.fresh(len(w0), 1.0, 0.0, True)
    w1, opt1 = server_step(opt, w0, agg.finalize(), 1)
    ordered = sorted(agg.updates, key=lambda u: u.client_id)
    compute_round_norms(w0, [u.delta for u in ordered], [weights[u.client_id] for u in ordered], opt1.momentum,
                        [u.client_id for u in ordered])
    return time.perf_counter() - t0, t_train, w1, sum(len(b) for b in blobs)


def fast_round():
    fed = Federation(cfg, adamw, sched, corpus, split, batch_size=16, micro_batches=1, local_steps=4, server_eta=1.0,
                     server_mu=0.0)
    w, opt = fed.init_state()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = fed.run_round(w, opt, 1)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, res.params


swap_round()
fast_round()  # warm-up both
ts, ttrain, w_swap, blob_bytes = swap_round()
tf, w_fast = fast_round()
same = ParamVector(w_fast.tensor.cpu().numpy()).bitwise_equal(w_swap)
print(json.dumps({"config": "C1 (2 clients x 4 steps x 16 x 128, FedAvg)", "n_params": len(w0),
                  "import_swap_round_s": round(ts, 4), "import_swap_train_s": round(ttrain, 4),
                  "update_blob_bytes": blob_bytes, "federation_round_s": round(tf, 4),
                  "global_model_bitwise_equal": bool(same)}))
