"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This package is a from-scratch CPU restatement of the reference's (fedforge,
arXiv 2405.10853) federated-round hot path. It is the *checker*: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it. The product package
``paper_2405_10853_b200`` never imports it and has no CPU fallback.

Parity pinning: every function here is checked against golden vectors produced
by running the *reference itself* in the build container
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src/fedforge``)
and against the reference's own known-answer tests (scalar AdamW oracle,
scalar server-step oracle, hand recurrence 0.905, ...). See
``tests/test_oracle_golden.py``.

Modules
  fedopt_ref   aggregation (streaming / deterministic pairwise tree) + server step
  localopt_ref AdamW (f64 math, f32 materialisation), clip, lr schedule, micro-mean
  data_ref     byte tokenizer, seeded split, per-client order, batch rows, Markov corpus
  model_ref    TinyLM forward/backward on torch CPU fp32 from a flat vector
  round_ref    train_round and one full federated round
"""
