"""torchrun --nproc-per-node G tools/multi_gpu_check.py
Round-end exchange, both multi-GPU forms, must be bit-identical to the single-GPU fused
aggregation: (a) NCCL all-to-all of client slices + shard-local fused kernel + all-gather,
(b) the single fused kernel over NVLink peer memory (PeerAggregator). Also reports each
form's time (max over ranks) for N params, K clients."""
import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_10853_b200 import ext  # noqa: E402
from paper_2405_10853_b200.dist import (PeerAggregator, ShardedAggregator, clients_of,  # noqa: E402
                                        reduce_round_end)

N = int(os.environ.get("CHK_N", "70542336"))
K = int(os.environ.get("CHK_K", "8"))
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
ext.lib()


def client(k):
    g = torch.Generator(device="cuda").manual_seed(100 + k)
    return w + torch.empty(N, device="cuda").normal_(0, 2e-3, generator=g)


g0 = torch.Generator(device="cuda").manual_seed(7)
w = torch.empty(N, device="cuda").normal_(0, 0.02, generator=g0)
m = torch.empty(N, device="cuda").normal_(0, 1e-3, generator=g0)
nk = {k: 1000 + 7 * k for k in range(K)}
agg = ShardedAggregator(N, K)
mine = {k: client(k) for k in clients_of(rank, world, K)}
for _ in range(2):
    agg.exchange(mine)
    w_new, m_shard = agg.step(w, m[agg.lo:agg.hi].contiguous(), nk, 0.7, 0.9, True)
torch.cuda.synchronize()
dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 5
for _ in range(reps):
    agg.exchange(mine)
    w_new, m_shard = agg.step(w, m[agg.lo:agg.hi].contiguous(), nk, 0.7, 0.9, True)
e1.record()
torch.cuda.synchronize()
ms = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
dist.all_reduce(ms, op=dist.ReduceOp.MAX)
stats_nccl, bad_nccl = reduce_round_end(agg.stats, agg.bad)
# (b) fused over NVLink peer memory: copy-engine staged pull (default) and direct SM pull
res_peer = {}  # both forms explicitly (the product default "auto" picks one per world size)
for mode in ("ce", "sm"):
    peer = PeerAggregator(N, K, pull=mode, chunk=int(os.environ.get("CHK_CHUNK", str(1 << 25))),
                          ce_clients=int(os.environ["CHK_CE"]) if "CHK_CE" in os.environ else None)
    for k, t in mine.items():
        peer.client_buffer(k).copy_(t)
    m_sh = m[peer.lo:peer.hi].contiguous()
    for _ in range(2):
        w_peer, m_peer = peer.step(w, m_sh, nk, 0.7, 0.9, True)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    for _ in range(reps):
        w_peer, m_peer = peer.step(w, m_sh, nk, 0.7, 0.9, True)
    e1.record()
    torch.cuda.synchronize()
    t_ms = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
    dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    st_sum, bad_sum = reduce_round_end(peer.stats, peer.bad)
    # an injected NaN in the last client's last-shard element must surface as that global index
    kn = K - 1
    if kn % world == rank:
        peer.client_buffer(kn)[N - 3] = float("nan")
    w_nan, _ = peer.step(w, m_sh, nk, 0.7, 0.9, True)
    _, bad_nan = reduce_round_end(peer.stats, peer.bad)
    res_peer[mode] = (float(t_ms), w_peer.clone(), m_peer.clone(), st_sum, bad_sum, bad_nan)
    del peer
    torch.cuda.empty_cache()
ms_peer, w_peer, m_peer = res_peer["ce"][:3]
ms_peer_sm, w_peer_sm, m_peer_sm = res_peer["sm"][:3]
# single-GPU reference on every rank (all clients regenerated locally)
allc = [client(k) for k in range(K)]
ptrs = (C.c_void_p * K)(*[t.data_ptr() for t in allc])
nks = (C.c_int64 * K)(*[nk[k] for k in range(K)])
wr, mr = torch.empty_like(w), torch.empty_like(m)
stats1 = torch.zeros(6 + K, dtype=torch.float64, device="cuda")
ext.call("fb_fedagg_round_norms_f32", ptrs, nks, K, 1, w.data_ptr(), m.data_ptr(), wr.data_ptr(), mr.data_ptr(), N, 0.7,
         0.9, 1, stats1.data_ptr(), None, ext.stream_handle())
torch.cuda.synchronize()
s1 = stats1.cpu().numpy()
import numpy as np  # noqa: E402
norms_ok = all(np.allclose(x, s1, rtol=1e-9, atol=0) for x in (stats_nccl, res_peer["ce"][3], res_peer["sm"][3]))
bad_ok = bad_nccl >= N and res_peer["ce"][4] >= N and res_peer["sm"][4] >= N and \
    res_peer["ce"][5] == N - 3 and res_peer["sm"][5] == N - 3
ok_w = torch.equal(w_new.view(torch.int32), wr.view(torch.int32))
ok_m = torch.equal(m_shard.view(torch.int32), mr[agg.lo:agg.hi].view(torch.int32))
ok_pw = torch.equal(w_peer.view(torch.int32), wr.view(torch.int32))
ok_pm = torch.equal(m_peer.view(torch.int32), mr[agg.lo:agg.hi].view(torch.int32))
ok_sm = torch.equal(w_peer_sm.view(torch.int32), wr.view(torch.int32)) and torch.equal(
    m_peer_sm.view(torch.int32), mr[agg.lo:agg.hi].view(torch.int32))
ok_st = bool(np.allclose(res_peer["ce"][3][:3], res_peer["sm"][3][:3], rtol=1e-12, atol=0))
flags = torch.tensor([int(ok_w), int(ok_m), int(ok_pw), int(ok_pm), int(ok_sm), int(ok_st), int(norms_ok),
                      int(bad_ok)], device="cuda")
dist.all_reduce(flags, op=dist.ReduceOp.MIN)
per_rank_bytes = 4 * N * len(mine) * (world - 1) / world + 4 * N * (world - 1) / world
if rank == 0:
    print(json.dumps({"world": world, "N": N, "K": K, "bit_identical_w": bool(flags[0]), "bit_identical_m": bool(flags[1]),
                      "peer_bit_identical_w": bool(flags[2]), "peer_bit_identical_m": bool(flags[3]),
                      "peer_sm_bit_identical": bool(flags[4]), "peer_stats_ce_vs_sm_close": bool(flags[5]),
                      "round_norms_match_1gpu": bool(flags[6]), "first_bad_global_index": bool(flags[7]),
                      "peer_sm_ms": round(ms_peer_sm, 3),
                      "exchange_ms": round(float(ms), 3), "peer_fused_ms": round(ms_peer, 3),
                      "peer_nvlink_in_bytes_per_rank": int(4 * (N // world) * (K - len(mine))),
                      "peer_nvlink_in_gbs_per_rank": round(4 * (N // world) * (K - len(mine)) / (ms_peer / 1e3) / 1e9, 1),
                      "nvlink_bytes_per_rank_per_dir": int(per_rank_bytes),
                      "nvlink_gbs_per_rank": round(per_rank_bytes / (float(ms) / 1e3) / 1e9, 1)}), flush=True)
dist.destroy_process_group()
