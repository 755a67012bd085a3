"""NVLink pull-rate probe (G = 2): how fast can one rank READ a peer's HBM?

Compares the copy engines (cudaMemcpyAsync from a symmetric-memory peer view, 1 and 4
streams) with SM loads (a torch reduction over the peer view) on the same bytes, to size
the headroom of the fused peer-memory round end (fb_fedagg_step_f32_peers, ~430 GB/s).

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nvlink_pull.py [GB]
"""
import json
import os
import sys

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    gb = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl")
    n = int(gb * 2**30) // 4
    buf = symm.empty(n, dtype=torch.float32, device="cuda")
    buf.normal_()
    h = symm.rendezvous(buf, dist.group.WORLD)
    peer = h.get_buffer((rank + 1) % world, (n,), torch.float32)
    dst = torch.empty(n, dtype=torch.float32, device="cuda")
    h.barrier(channel=0)
    nbytes = 4 * n
    res = {"rank": rank, "bytes": nbytes}
    res["ce_1stream_gbs"] = nbytes / timed(lambda: dst.copy_(peer)) / 1e6
    streams = [torch.cuda.Stream() for _ in range(4)]

    def ce4():
        cur = torch.cuda.current_stream()
        q = n // 4
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                dst[i * q:(i + 1) * q].copy_(peer[i * q:(i + 1) * q])
        for s in streams:
            cur.wait_stream(s)
    res["ce_4stream_gbs"] = nbytes / timed(ce4) / 1e6
    out = torch.empty((), dtype=torch.float32, device="cuda")
    res["sm_sum_gbs"] = nbytes / timed(lambda: torch.sum(peer, 0, out=out)) / 1e6
    res["sm_local_sum_gbs"] = nbytes / timed(lambda: torch.sum(buf, 0, out=out)) / 1e6
    res["sm_add_gbs"] = nbytes / timed(lambda: torch.add(buf, peer, out=dst)) / 1e6  # peer read only
    h.barrier(channel=1)
    allr = [None] * world
    dist.all_gather_object(allr, res)
    if rank == 0:
        for r in allr:
            print(json.dumps(r))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
