"""Experiment: stamps of every CTA of the decode sampler (build with -DOTK_SDEC_TIMING, OTK_LIB=that .so): the
launch spread (globaltimer at each CTA's start, ns) and per-CTA phase durations from clock64 (SM cycles -> ns at the
SM clock): 0-1 load + segment pass, 1-2 push + wait for the row's partials, 2-3 peer reads + max, 3-4 masses +
scan, 4-5 crossing partial, 5-6 search (crossing warp) / exit. Each column: min / median / max over the launch's CTAs."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2601_07376_b200 as otk
from synth import make_logits
ctx = otk.Context(0)
mhz = float(os.environ.get("SM_MHZ", "1965"))
for n in (1, 16, 32):
    lg, _ = make_logits(n, 151936, dtype="bf16", seed=3, device="cuda")
    u = torch.rand(n, device="cuda")
    buf = (ctypes.c_ulonglong * (256 * 8))()
    for it in range(4):
        torch.cuda._sleep(200000)   # a busy GPU ahead of the launch, as inside a decode step
        otk.otk_sample_tokens(ctx, lg, u)
        torch.cuda.synchronize()
        otk._lib.otk_debug_sdec(buf)
        a = np.array(buf, dtype=np.int64).reshape(256, 8)
        a = a[a[:, 0] > 0]
        a = a[a[:, 0] >= a[:, 0].max() - 100000]       # this launch's CTAs (stale entries are older)
        cols = ["start:%d/%d/%d" % tuple(np.percentile(a[:, 0] - a[:, 0].min(), [0, 50, 100]))]
        for i, name in ((1, "seg"), (2, "xchg"), (3, "R"), (4, "scan"), (5, "X"), (6, "end")):
            d = (a[:, 1 + i] - a[:, i]) * 1e3 / mhz
            cols.append(f"{name}:{int(d.min())}/{int(np.median(d))}/{int(d.max())}")
        end = a[:, 0] - a[:, 0].min() + (a[:, 7] - a[:, 1]) * 1e3 / mhz
        cols.append("end:%d/%d/%d" % tuple(np.percentile(end, [0, 50, 100])))
        print(n, it, len(a), " ".join(cols), flush=True)
