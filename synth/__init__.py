"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package is the ONLY code the CUDA path and the oracle have in common. It draws
random numbers and lays out trajectories; it holds none of the method's arithmetic
(no masks, no advantages, no softmax, no loss). Values the method derives from these
inputs (old/ref log-probs) are built by the caller from an implementation's output
plus the noise drawn here.
"""
from .trajectories import TrajBatch, make_batch, CONFIGS, WorkloadConfig, concat_batches, slice_batch, split_rows
from .logits import make_logits, make_noise, bf16_round
from .lmhead import make_lmhead

__all__ = [
    "TrajBatch", "make_batch", "CONFIGS", "WorkloadConfig", "concat_batches", "slice_batch", "split_rows",
    "make_logits", "make_noise", "bf16_round", "make_lmhead",
]
