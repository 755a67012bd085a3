"""Flower-style façade over the drop-in API (BASELINE north star: "Flower-style fit /
aggregate_fit"). Parameters travel as Flower does — a list of numpy arrays in model
manifest order — and map onto the reference entry points:
  fit            -> train_round            (fedforge/trainer.py:54-114)
  aggregate_fit  -> AggregatorState + server_step  (fedforge/fedopt.py:58-201)
"""
from __future__ import annotations

import numpy as np

from .config import AdamWConfig, ScheduleConfig, TrainTask
from .data import BatchIterator
from .fedopt import AggregatorState, ClientUpdate, DeviceVector, ServerOptState, server_step
from .model import LossEvaluator
from .params import ParamVector
from .trainer import train_round


def to_arrays(flat: np.ndarray, evaluator: LossEvaluator) -> list:
    return [flat[e.offset:e.offset + e.size].reshape(e.shape).copy() for e in evaluator.manifest]


def from_arrays(arrays) -> np.ndarray:
    return np.concatenate([np.asarray(a, dtype=np.float32).reshape(-1) for a in arrays])


class B200Client:
    """NumPyClient-like: fit(parameters, config) -> (parameters, num_examples, metrics)."""

    def __init__(self, client_id: int, evaluator: LossEvaluator, batches: BatchIterator, adamw: AdamWConfig,
                 sched: ScheduleConfig, *, local_steps: int, batch_size: int, micro_batches: int = 1):
        self.cid, self.ev, self.batches = client_id, evaluator, batches
        self.adamw, self.sched = adamw, sched
        self.S, self.B, self.micro = local_steps, batch_size, micro_batches

    def get_parameters(self, config=None):
        return to_arrays(self.ev.init_params().data, self.ev)

    def fit(self, parameters, config: dict):
        rnd = int(config.get("server_round", 1))
        steps = int(config.get("local_steps", self.S))
        offset = int(config.get("schedule_offset", (rnd - 1) * self.S))
        task = TrainTask(rnd, self.cid, steps, offset, self.B, self.micro, {}, "")
        upd, tele = train_round(ParamVector(from_arrays(parameters)), self.batches, self.ev, self.adamw, self.sched,
                                task)
        w_end = upd.w_end.cpu().numpy()
        metrics = dict(upd.local_metrics)
        metrics["client_id"] = self.cid
        return to_arrays(w_end, self.ev), upd.n_k, metrics


class FedOptStrategy:
    """aggregate_fit(server_round, results, failures) -> (parameters, metrics): the
    sample-weighted pseudo-gradient and a FedAvg / Nesterov outer step."""

    def __init__(self, evaluator: LossEvaluator, initial_parameters, *, eta: float = 1.0, mu: float = 0.0,
                 nesterov: bool = True, deterministic: bool = True):
        self.ev = evaluator
        self.w = ParamVector(from_arrays(initial_parameters))
        self.opt = ServerOptState.fresh(len(self.w), eta, mu, nesterov)
        self.det = deterministic

    def aggregate_fit(self, server_round: int, results, failures):
        if not results:
            return None, {"failures": len(failures)}
        agg = AggregatorState(server_round, len(self.w), deterministic=self.det)
        g = self.w.as_f64()
        for i, (params, n_k, metrics) in enumerate(results):
            cid = int(metrics.get("client_id", i))
            agg.accumulate(ClientUpdate(cid, server_round, int(n_k), g - from_arrays(params).astype(np.float64)))
        self.w, self.opt = server_step(self.opt, self.w, agg.finalize(), server_round)
        return to_arrays(self.w.data, self.ev), {"n_contributors": len(results), "failures": len(failures),
                                                  "weights": agg.weights()}
