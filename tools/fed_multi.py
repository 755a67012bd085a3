"""torchrun --nproc-per-node G tools/fed_multi.py: two C1 rounds (K = 4 clients) of the Federation
driver on G GPUs (clients sharded over ranks, peer-memory round end); prints the aggregator
used, the round-2 client mean losses and the global-model norm (compare with --nproc-per-node 1)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import data  # noqa: E402
from paper_2405_10853_b200.config import AdamWConfig, ScheduleConfig, TinyLMConfig  # noqa: E402
from paper_2405_10853_b200.federation import Federation  # noqa: E402

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
cfg = TinyLMConfig(vocab_size=256, context_len=128, n_layers=2, d_model=512, n_heads=8, seed=1234)
corpus = data.tokenize_bytes(data.synth_corpus(99, 400_000), 128, 256)
K = 4
split = data.split_corpus(corpus, K, 99, 0.05)
kw = dict(batch_size=16, micro_batches=1, local_steps=4, server_eta=0.7, server_mu=0.9)
fed = Federation(cfg, AdamWConfig(), ScheduleConfig(1e-3, 2, 1000, 0.1), corpus, split, **kw)
w, opt = fed.init_state()
res = fed.run_round(w, opt, 1)
ck_path = os.environ.get("FED_CKPT", "/tmp/fed_multi_r2.fedp")
res = fed.run_round(res.params, res.opt, 2, checkpoint_path=ck_path)
losses = torch.zeros(K, dtype=torch.float64, device="cuda")
for k, mtr in res.client_metrics.items():
    losses[k] = mtr["mean_loss"]
dist.all_reduce(losses)
w_multi = res.params.tensor.clone()
kind = type(fed.agg).__name__
if rank == 0:
    from paper_2405_10853_b200.checkpoint import read_checkpoint
    res.checkpoint.wait()
    ck = read_checkpoint(ck_path)
    n = res.norms
    print(json.dumps({"world": world, "aggregator": kind, "round2_client_mean_losses": [round(float(x), 5) for x in
                      losses.tolist()], "w_norm": float(w_multi.double().norm()), "finite": bool(torch.isfinite(w_multi).all()),
                      "ckpt_momentum_len": len(ck["momentum"]), "ckpt_global_len": len(ck["global"]),
                      "ckpt_momentum_norm": float(np.linalg.norm(np.asarray(ck["momentum"].data, np.float64))),
                      "norms": {"global": n.global_norm, "avg_client": n.avg_client_norm, "pseudograd": n.pseudograd_norm,
                                "momentum": n.momentum_norm,
                                "per_client": [n.per_client_norms[k] for k in sorted(n.per_client_norms)]}}),
          flush=True)
dist.destroy_process_group()
