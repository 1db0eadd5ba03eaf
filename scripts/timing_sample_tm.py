"""Experiment: per-CTA timeline of the ring sampler's first row (build with -DOTK_STM_TIMING, OTK_LIB=that .so):
launch spread (globaltimer, ns) and clock64 phases (ns at SM_MHZ): start -> consumer warp 1 has chunk 0 (first
bulk-TMA latency), -> it has finished the row (streaming), -> the search warp has the row, -> token written (search).
Columns: min / median / max over CTAs."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2601_07376_b200 as otk
from synth import make_logits
ctx = otk.Context(0)
mhz = float(os.environ.get("SM_MHZ", "1965"))
for n in (96, 128, 148):
    bufs = [make_logits(n, 151936, dtype="bf16", seed=3 + k, device="cuda")[0] for k in range(8)]
    u = torch.rand(n, device="cuda")
    buf = (ctypes.c_ulonglong * (256 * 8))()
    for it in range(8):
        otk.otk_sample_tokens(ctx, bufs[it], u)
        torch.cuda.synchronize()
    otk._lib.otk_debug_stm(buf)
    a = np.array(buf, dtype=np.int64).reshape(256, 8)[:n]
    cols = ["start:%d/%d/%d" % tuple(np.percentile(a[:, 0] - a[:, 0].min(), [0, 50, 100]))]
    for i, name in ((2, "first"), (3, "stream"), (4, "handoff"), (5, "search")):
        d = (a[:, i] - a[:, i - 1]) * 1e3 / mhz
        cols.append(f"{name}:{int(d.min())}/{int(np.median(d))}/{int(d.max())}")
    end = a[:, 0] - a[:, 0].min() + (a[:, 5] - a[:, 1]) * 1e3 / mhz
    cols.append("end:%d/%d/%d" % tuple(np.percentile(end, [0, 50, 100])))
    print(n, " ".join(cols), flush=True)
