"""Seeded LM-head inputs for the fused LM-head forward (NEXT-1): final hidden states
h ~ N(0, 1) and a head matrix W ~ N(0, (2/sqrt(d))^2), both rounded to bf16, so the logits z = h W^T have
standard deviation ~2 like the logits recipe; targets uniform in [0, V). torch is only the seeded RNG."""
from __future__ import annotations

import torch


def make_lmhead(n_rows: int, vocab: int, hidden_dim: int, *, seed: int = 0, device: str = "cpu"):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    h = torch.randn((n_rows, hidden_dim), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    w = (torch.randn((vocab, hidden_dim), generator=g, device=device, dtype=torch.float32)
         * (2.0 / hidden_dim ** 0.5)).to(torch.bfloat16)
    y = torch.randint(0, vocab, (n_rows,), generator=g, device=device, dtype=torch.int64).to(torch.int32)
    return h, w, y
