"""Teacher-forced C1 diagnostic: at each oracle step of round 2, compare our GPU
loss/grad with the fp32 oracle's at identical params and batch."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import data_ref, fedopt_ref, localopt_ref, model_ref  # noqa: E402
from paper_2405_10853_b200.config import TinyLMConfig  # noqa: E402
from paper_2405_10853_b200.model import LossEvaluator  # noqa: E402

torch.set_num_threads(16)
V, ctx, L, d, H = 256, 128, 2, 512, 8
text = data_ref.markov_bytes(99, 400_000)
tok = data_ref.tokens_of(text)
val, shards = data_ref.split(data_ref.n_samples(tok, 128), 2, 99, 0.05)
orders = [data_ref.client_order(s, k, 99) for k, s in enumerate(shards)]
ev = LossEvaluator(TinyLMConfig(vocab_size=V, context_len=ctx, n_layers=L, d_model=d, n_heads=H, seed=1234))
w = model_ref.init_flat(V, ctx, L, d, 1234)
m = np.zeros_like(w)
for rnd in (1, 2):
    ws = []
    for k in range(2):
        p = w.copy()
        m1 = np.zeros_like(p)
        m2 = np.zeros_like(p)
        cur = (rnd - 1) * 4 * 16
        for s in range(4):
            batch = data_ref.gather(tok, 128, data_ref.batch_rows(orders[k], cur, 16))
            cur += 16
            lo, go = model_ref.loss_and_grad(p, batch, V, ctx, L, d, H)
            lg, gg = ev.loss_and_grad(p, batch)
            rel = np.linalg.norm(gg - go) / np.linalg.norm(go)
            sign = np.mean(np.sign(gg) == np.sign(go))
            lr = localopt_ref.lr_at(1e-3, 2, 1000, 0.1, (rnd - 1) * 4 + s)
            go_c, raw = localopt_ref.clip(go, 1.0)
            gg_c, raw2 = localopt_ref.clip(gg.astype(np.float32), 1.0)
            p2, _, _, _ = localopt_ref.adamw(p, gg_c, m1, m2, s + 1, lr)
            p, m1, m2, _ = localopt_ref.adamw(p, go_c, m1, m2, s + 1, lr)
            print(f"r{rnd} c{k} s{s}: loss {lo:.5f} ours {lg:.5f} | grad rel {rel:.2e} sign-agree {sign:.4f} "
                  f"| |g| {raw:.3f} vs {raw2:.3f} | param-step diff rel {np.linalg.norm(p2 - p) / np.linalg.norm(p - w):.3e}")
        ws.append(p)
    w, m = fedopt_ref.fed_round(w, m, ws, [s.size for s in shards], 1.0, 0.0, True)
