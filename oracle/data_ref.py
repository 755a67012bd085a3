"""Oracle: the data index contract (numpy PCG64; integer, bit-exact).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates
  * tokenize_bytes / TokenizedCorpus.samples  /root/reference/pkg/src/fedforge/data.py:42-58
  * split_corpus                              data.py:85-109
  * BatchIterator order / seek / next_batch   data.py:132-161
  * synth_corpus("markov")                    data.py:164-203
"""
from __future__ import annotations

import numpy as np

_ALPHA = np.arange(33, 97, dtype=np.uint8)
_CUM = np.cumsum([0.55, 0.25, 0.15, 0.05])


def markov_bytes(seed: int, n_bytes: int) -> bytes:
    rng = np.random.default_rng(seed)
    n = _ALPHA.size
    succ = np.empty((n, 4), dtype=np.int64)
    for s in range(n):
        succ[s] = rng.choice(n, size=4, replace=False)
    pick = np.searchsorted(_CUM, rng.random(n_bytes), side="left")
    state = int(rng.integers(0, n))
    out = np.empty(n_bytes, dtype=np.int64)
    sl = succ.tolist()
    pl = pick.tolist()
    for i in range(n_bytes):
        out[i] = state
        state = sl[state][pl[i]]
    return _ALPHA[out].tobytes()


def tokens_of(text: bytes) -> np.ndarray:
    return np.frombuffer(text, dtype=np.uint8).astype(np.uint16)


def n_samples(tokens: np.ndarray, seq_len: int) -> int:
    return tokens.size // seq_len


def split(n: int, n_clients: int, seed: int, val_frac: float):
    perm = np.random.default_rng(seed).permutation(n)
    nv = int(val_frac * n)
    rest = perm[nv:]
    per = rest.size // n_clients
    shards = [np.sort(rest[k * per:(k + 1) * per]) for k in range(n_clients)]
    return np.sort(perm[:nv]), shards


def client_order(shard_indices: np.ndarray, shard_id: int, seed: int) -> np.ndarray:
    p = np.random.default_rng([seed & 0xFFFFFFFFFFFFFFFF, shard_id]).permutation(shard_indices.size)
    return shard_indices[p]


def batch_rows(order: np.ndarray, cursor: int, batch: int) -> np.ndarray:
    return order[(cursor + np.arange(batch)) % order.size]


def gather(tokens: np.ndarray, seq_len: int, rows: np.ndarray) -> np.ndarray:
    ns = tokens.size // seq_len
    return tokens[: ns * seq_len].reshape(ns, seq_len)[rows]
