"""Oracle: TinyLM forward / backward from a flat f32 vector (torch CPU fp32).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates
  * TinyLMConfig + manifest order     /root/reference/pkg/src/fedforge/model.py:28-43, :184-190
  * alibi_slopes / alibi_bias         model.py:46-72
  * init_weights                      model.py:123-141
  * Block.forward / TinyLM.forward    model.py:88-102, :143-150
  * mean next-token CE                model.py:222-229
  * loss_and_grad                     model.py:237-250
Functional (no nn.Module); autograd supplies the backward.
"""
from __future__ import annotations

import functools
import math

import numpy as np
import torch
import torch.nn.functional as F


def manifest(V, ctx, L, d, use_alibi=True):
    """[(name, shape)] in the reference's named_parameters() order."""
    ent = [("embed.weight", (V, d))]
    if not use_alibi:
        ent.append(("pos_embed.weight", (ctx, d)))
    for i in range(L):
        p = f"blocks.{i}."
        ent += [(p + "ln1.weight", (d,)), (p + "ln1.bias", (d,)),
                (p + "qkv.weight", (3 * d, d)), (p + "attn_proj.weight", (d, d)),
                (p + "ln2.weight", (d,)), (p + "ln2.bias", (d,)),
                (p + "mlp_fc.weight", (4 * d, d)), (p + "mlp_proj.weight", (d, 4 * d))]
    ent += [("ln_f.weight", (d,)), ("ln_f.bias", (d,)), ("head.weight", (V, d))]
    return ent


def n_params(V, ctx, L, d, use_alibi=True):
    return sum(int(np.prod(s)) for _, s in manifest(V, ctx, L, d, use_alibi))


def init_flat(V, ctx, L, d, seed, use_alibi=True) -> np.ndarray:
    gen = torch.Generator().manual_seed(seed)
    std_r = 0.02 / math.sqrt(2 * L)
    parts = []
    for name, shape in manifest(V, ctx, L, d, use_alibi):
        t = torch.empty(shape, dtype=torch.float32)
        if name == "head.weight":
            t.zero_()
        elif name.endswith("attn_proj.weight") or name.endswith("mlp_proj.weight"):
            t.normal_(0.0, std_r, generator=gen)
        elif "ln" in name:
            t.fill_(1.0) if name.endswith("weight") else t.zero_()
        else:
            t.normal_(0.0, 0.02, generator=gen)
        parts.append(t.reshape(-1))
    return torch.cat(parts).numpy()


def slopes(H):
    return np.array([2.0 ** (-8.0 * (h + 1) / H) for h in range(H)])


@functools.lru_cache(maxsize=4)
def attn_bias(H, T, use_alibi=True):
    """(H, T, T) f32 bias; built once per shape like the reference's registered buffer (model.py:115-121)."""
    i = np.arange(T)[:, None]
    j = np.arange(T)[None, :]
    if use_alibi:
        b = -slopes(H)[:, None, None] * (i - j).astype(np.float64)[None]
    else:
        b = np.zeros((H, T, T))
    b[:, j > i] = -np.inf
    return torch.from_numpy(b.astype(np.float32))


def _views(flat, V, ctx, L, d, use_alibi, dtype):
    out, off = {}, 0
    for name, shape in manifest(V, ctx, L, d, use_alibi):
        n = int(np.prod(shape))
        out[name] = flat[off:off + n].view(shape)
        off += n
    return out


def loss_and_grad(flat32: np.ndarray, tokens: np.ndarray, V, ctx, L, d, H, use_alibi=True,
                  dtype=torch.float32, want_grad=True):
    """Mean CE over B*(T-1) positions and (optionally) the flat gradient."""
    p = torch.tensor(np.asarray(flat32), dtype=dtype, requires_grad=want_grad)
    W = _views(p, V, ctx, L, d, use_alibi, dtype)
    tok = torch.from_numpy(np.asarray(tokens).astype(np.int64))
    B, T = tok.shape
    dh = d // H
    x = W["embed.weight"][tok]
    if not use_alibi:
        x = x + W["pos_embed.weight"][torch.arange(T)]
    bias = attn_bias(H, ctx, use_alibi).to(dtype)[:, :T, :T]
    for i in range(L):
        pre = f"blocks.{i}."
        h = F.layer_norm(x, (d,), W[pre + "ln1.weight"], W[pre + "ln1.bias"], 1e-5)
        qkv = h @ W[pre + "qkv.weight"].t()
        q, k, v = qkv.split(d, dim=2)
        q = q.view(B, T, H, dh).transpose(1, 2)
        k = k.view(B, T, H, dh).transpose(1, 2)
        v = v.view(B, T, H, dh).transpose(1, 2)
        s = (q @ k.transpose(-2, -1)) / math.sqrt(dh) + bias
        y = (torch.softmax(s, dim=-1) @ v).transpose(1, 2).reshape(B, T, d)
        x = x + y @ W[pre + "attn_proj.weight"].t()
        h = F.layer_norm(x, (d,), W[pre + "ln2.weight"], W[pre + "ln2.bias"], 1e-5)
        x = x + F.gelu(h @ W[pre + "mlp_fc.weight"].t()) @ W[pre + "mlp_proj.weight"].t()
    logits = F.layer_norm(x, (d,), W["ln_f.weight"], W["ln_f.bias"], 1e-5) @ W["head.weight"].t()
    loss = F.cross_entropy(logits[:, :-1].reshape(-1, V), tok[:, 1:].reshape(-1))
    if not want_grad:
        return float(loss.detach())
    loss.backward()
    return float(loss.detach()), p.grad.detach().numpy().copy()
