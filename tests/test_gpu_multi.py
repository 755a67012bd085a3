"""Multi-GPU round end (needs >= 2 GPUs on the box; skipped otherwise).

Runs tools/multi_gpu_check.py under torchrun: the NCCL form (ShardedAggregator), the
copy-engine staged peer pull and the direct SM peer pull (PeerAggregator) must all be
bit-identical to the single-GPU fused aggregation, including ragged last chunks."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.gpu
@pytest.mark.parametrize("n,chunk", [(1_000_003, 100_000), (8_388_611, 1 << 25)])
def test_peer_round_end_bit_identical(n, chunk):
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    env = dict(os.environ, CHK_N=str(n), CHK_CHUNK=str(chunk), CHK_K="8")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(ROOT, "tools", "multi_gpu_check.py")]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [x for x in out.stdout.splitlines() if x.startswith("{")][-1]
    r = json.loads(line)
    for key in ("bit_identical_w", "bit_identical_m", "peer_bit_identical_w", "peer_bit_identical_m",
                "peer_sm_bit_identical", "peer_stats_ce_vs_sm_close"):
        assert r[key], (key, r)
