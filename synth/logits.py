"""Seeded synthetic LM-head logits and per-row noise.

Recipe: per row z = 2*N(0,1); one "preferred" token gets
+U[4,14]; the target is the preferred token with probability 0.8, else uniform in [0, V).
Values are rounded to the logits dtype (bf16 round-to-nearest-even via torch). Columns [V, ld)
of a padded row hold a large sentinel so that a kernel reading past V is caught by parity.

torch is used here only as a seeded random-number source and for device placement.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

PAD_SENTINEL = 1.0e4


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def make_logits(n_rows: int, V: int, *, ld: Optional[int] = None, dtype: str = "bf16", seed: int = 0,
                device: str = "cpu", uniform_rows: Sequence[int] = (), rows_per_chunk: int = 2048,
                scale: float = 2.0, out: Optional[torch.Tensor] = None):
    """Return (logits [n_rows, ld] in dtype, targets int32 [n_rows]) on `device`."""
    ld = V if ld is None else ld
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32}[dtype]
    g = _gen(device, seed)
    if out is None:
        out = torch.empty((n_rows, ld), dtype=tdt, device=device)
    targets = torch.empty(n_rows, dtype=torch.int32, device=device)
    for r0 in range(0, n_rows, rows_per_chunk):
        r1 = min(n_rows, r0 + rows_per_chunk)
        n = r1 - r0
        z = torch.randn((n, V), generator=g, device=device, dtype=torch.float32) * scale
        pref = torch.randint(0, V, (n,), generator=g, device=device)
        bump = torch.rand((n,), generator=g, device=device) * 10.0 + 4.0
        z[torch.arange(n, device=device), pref] += bump
        pick = torch.rand((n,), generator=g, device=device) < 0.8
        other = torch.randint(0, V, (n,), generator=g, device=device)
        targets[r0:r1] = torch.where(pick, pref, other).to(torch.int32)
        out[r0:r1, :V] = z.to(tdt)
        if ld > V:
            out[r0:r1, V:] = PAD_SENTINEL
    for r in uniform_rows:
        if 0 <= r < n_rows:
            out[r, :V] = 0
    return out, targets


def make_noise(n: int, sigma: float, seed: int, device: str = "cpu") -> torch.Tensor:
    """N(0, sigma^2) float32 noise, used to build old/ref log-probs from a policy's log-probs."""
    g = _gen(device, seed)
    return (torch.randn(n, generator=g, device=device, dtype=torch.float32) * sigma)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bf16 (RNE) and return them widened back to float64."""
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def widen(logits: torch.Tensor) -> np.ndarray:
    """Exact widening of bf16/fp32 logits to float64 numpy (what the oracle consumes)."""
    return logits.detach().to("cpu").to(torch.float64).numpy()
