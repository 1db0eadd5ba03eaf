"""Time otk_sample_tokens on decode batches (V = 151936 bf16): CUDA events, buffers cycled so the
logits of an iteration are not L2-resident from the previous one (total > L2 for the larger batches).
Usage: python scripts/perf_sample.py [--rows 256,1024,4096] [--iters 20]"""
import os, sys, json, argparse
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_07376_b200 as otk
from synth import make_logits
ap = argparse.ArgumentParser(); ap.add_argument("--rows", default="128,256,1024,4096"); ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
torch.cuda.set_device(0)
ctx = otk.Context(0)
V = 151936
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6532.2
for n in [int(r) for r in a.rows.split(",")]:
    nb = max(2, -(-400_000_000 // (n * V * 2)))        # cycle >= 400 MB of logits (> L2)
    nb = min(nb, 8)
    bufs = [make_logits(n, V, dtype="bf16", seed=7 + k, device="cuda", rows_per_chunk=4096)[0] for k in range(nb)]
    u = torch.rand(n, device="cuda")
    res = {}
    for mode in ("sample", "greedy"):
        toks = torch.empty(n, dtype=torch.int32, device="cuda")
        lps = torch.empty(n, dtype=torch.float32, device="cuda")
        def fn(k):
            otk.otk_sample_tokens(ctx, bufs[k % nb], u, greedy=mode == "greedy", out=dict(tokens=toks, logp=lps))
        for k in range(3): fn(k)
        torch.cuda.synchronize()
        # the launches are captured in a CUDA graph, so the time is the kernels' (not the Python binding's)
        g = torch.cuda.CUDAGraph()
        s_ = torch.cuda.Stream()
        s_.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_):
            with torch.cuda.graph(g, stream=s_):
                for k in range(a.iters): fn(k)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        g.replay()
        ev[1].record(); torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / a.iters
        by = n * (2 * V + 12)
        res[mode] = dict(us=round(ms * 1e3, 1), GBps=round(by / ms / 1e6, 1), frac=round(by / ms / 1e6 / peak, 4),
                         rows_per_s=round(n / ms * 1e3))
    # greedy without logp (no exponentials)
    toks = torch.empty(n, dtype=torch.int32, device="cuda")
    def fg(k):
        otk.otk_sample_tokens(ctx, bufs[k % nb], greedy=True, want_logp=False, out=dict(tokens=toks))
    for k in range(3): fg(k)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        with torch.cuda.graph(g, stream=s_):
            for k in range(a.iters): fg(k)
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(); g.replay(); ev[1].record(); torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / a.iters
    by = n * (2 * V + 4)
    res["greedy_nologp"] = dict(us=round(ms * 1e3, 1), GBps=round(by / ms / 1e6, 1), frac=round(by / ms / 1e6 / peak, 4))
    print(json.dumps(dict(rows=n, bufs=nb, **res)), flush=True)
    del bufs
ctx.check()
