"""Model / optimizer / schedule / task configuration types.

Same fields, defaults and validation as the reference so they are consumed
unchanged: TinyLMConfig (fedforge/model.py:28-43), AdamWConfig
(localopt.py:22-38), ScheduleConfig + lr_at (localopt.py:99-129), TrainTask
(messages.py:45-56), StepTelemetry (trainer.py:44-51).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from .errors import ParamError


@dataclass(frozen=True)
class TinyLMConfig:
    vocab_size: int = 256
    context_len: int = 64
    n_layers: int = 2
    d_model: int = 64
    n_heads: int = 4
    use_alibi: bool = True
    seed: int = 1234

    def __post_init__(self):
        if self.d_model % self.n_heads != 0:
            raise ParamError(f"d_model={self.d_model} not divisible by n_heads={self.n_heads}")
        if self.context_len < 2:
            raise ParamError(f"context_len must be >= 2, got {self.context_len}")

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_heads


@dataclass(frozen=True)
class AdamWConfig:
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 1e-5
    clip_norm: float = 1.0

    def __post_init__(self):
        if not 0 <= self.beta1 < 1 or not 0 <= self.beta2 < 1:
            raise ParamError(f"betas must be in [0, 1): {self.beta1}, {self.beta2}")
        if self.eps <= 0:
            raise ParamError(f"eps must be positive, got {self.eps}")
        if self.weight_decay < 0:
            raise ParamError(f"weight_decay must be >= 0, got {self.weight_decay}")
        if self.clip_norm <= 0:
            raise ParamError(f"clip_norm must be positive, got {self.clip_norm}")


@dataclass(frozen=True)
class ScheduleConfig:
    base_lr: float
    warmup_steps: int = 100
    t_max: int = 10_000
    alpha_f: float = 1e-6

    def __post_init__(self):
        if self.base_lr <= 0:
            raise ParamError(f"base_lr must be positive, got {self.base_lr}")
        if not 0 <= self.warmup_steps < self.t_max:
            raise ParamError(f"need 0 <= warmup_steps < t_max, got {self.warmup_steps}, {self.t_max}")
        if not 0 <= self.alpha_f <= 1:
            raise ParamError(f"alpha_f must be in [0, 1], got {self.alpha_f}")


def lr_at(sched: ScheduleConfig, global_step: int) -> float:
    """Warmup then cosine to alpha_f * base_lr; evaluated on the host in f64 and
    shipped to the device per step (the schedule clock survives rounds)."""
    if global_step < 0:
        raise ParamError(f"global_step must be >= 0, got {global_step}")
    if global_step < sched.warmup_steps:
        return sched.base_lr * (global_step + 1) / sched.warmup_steps
    if global_step >= sched.t_max:
        return sched.base_lr * sched.alpha_f
    frac = (global_step - sched.warmup_steps) / (sched.t_max - sched.warmup_steps)
    return sched.base_lr * (sched.alpha_f + (1.0 - sched.alpha_f) * (0.5 * (1.0 + math.cos(math.pi * frac))))


@dataclass(frozen=True)
class TrainTask:
    round: int
    client_id: int
    local_steps: int
    schedule_offset: int
    batch_size: int
    micro_batches: int
    seeds: dict = field(default_factory=dict)
    blob_key: str = ""


@dataclass(frozen=True)
class StepTelemetry:
    step: int
    loss: float
    grad_norm_raw: float
    grad_norm_applied: float
    lr: float
    param_norm: float
