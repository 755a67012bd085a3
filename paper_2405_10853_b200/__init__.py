"""B200-native (sm_100a) federated generative pre-training round — a drop-in
for the reference `fedforge` hot path (client train_round, server
AggregatorState/server_step) built on hand-written tcgen05/TMA CUDA behind
the C ABI in include/fedb200.h."""
__version__ = "0.1.0"
