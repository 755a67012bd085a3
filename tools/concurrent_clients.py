"""Small-config utilisation experiment: P clients of C2 or
C3 trained CONCURRENTLY on one GPU, one host thread + one CUDA stream each (ctypes releases
the GIL), against the same clients trained one after another. Prints one JSON line per P:
aggregate tokens/s and the fraction of sustained bf16 (algorithmic FLOPs).

    python tools/concurrent_clients.py c2 [steps]"""
import json
import os
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2405_10853_b200 import data, ext  # noqa: E402
from paper_2405_10853_b200.config import AdamWConfig, ScheduleConfig, TinyLMConfig, TrainTask  # noqa: E402
from paper_2405_10853_b200.fedopt import DeviceVector  # noqa: E402
from paper_2405_10853_b200.model import LossEvaluator, init_params_host  # noqa: E402
from paper_2405_10853_b200.trainer import ClientSession, device_corpus  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
c = bench.CONFIGS[name]
ext.lib()
_, _, tf_sus, _ = bench.peaks()
cfg = TinyLMConfig(vocab_size=c["V"], context_len=c["T"], n_layers=c["L"], d_model=c["d"], n_heads=c["H"], seed=1234)
corpus = data.tokenize_bytes(data.synth_corpus(99, c["n_bytes"]), c["T"], c["V"])
split = data.split_corpus(corpus, c["K"], 99, 0.05)
w0 = DeviceVector(torch.from_numpy(init_params_host(cfg)).cuda())
tokens_step = c["B"] * c["micro"] * c["T"]
fl_tok = bench.flops_per_token(c)
MAXP = 4
evs = [LossEvaluator(cfg) for _ in range(MAXP)]
streams = [torch.cuda.Stream() for _ in range(MAXP)]


def client_run(k, nsteps, barrier=None):
    with torch.cuda.stream(streams[k]):
        it = data.BatchIterator(corpus, split.shards[k], c["B"], 99)
        device_corpus(it, evs[k].device)
        sess = ClientSession(evs[k], it, AdamWConfig(), ScheduleConfig(*c["sched"]))
        sess.begin(w0, TrainTask(1, k, nsteps, 0, c["B"], c["micro"], {"data": 99}, "cc"))
        if barrier is not None:
            barrier.wait()
        for s in range(nsteps):
            sess.step(s)
        sess.finish()
        torch.cuda.current_stream().synchronize()


for k in range(MAXP):  # warm-up: workspaces, tensor maps, corpus upload
    client_run(k, 1)
torch.cuda.synchronize()
for P in (1, 2, 4):
    bar = threading.Barrier(P + 1)
    ths = [threading.Thread(target=client_run, args=(k, steps, bar)) for k in range(P)]
    for t in ths:
        t.start()
    bar.wait()
    t0 = time.perf_counter()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tps = P * steps * tokens_step / dt
    print(json.dumps({"config": name, "concurrent_clients": P, "steps_each": steps, "wall_s": round(dt, 3),
                      "tokens_per_s": round(tps, 1), "tflops": round(tps * fl_tok / 1e12, 1),
                      "frac_sustained_bf16": round(tps * fl_tok / 1e12 / tf_sus, 3)}), flush=True)
