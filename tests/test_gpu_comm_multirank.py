"""The library's batch-sharded exchanges at several ranks on the one-GPU box: otk_comm_* / otk_batch_* bound to an
in-process fake NCCL (tests/fake_nccl, via $OTK_NCCL_LIB; ranks are threads sharing the device — real NCCL refuses
two ranks on one device). PolicyLossStep(collectives="otk") on P = 2 and 3 contiguous trajectory shards (groups
straddling the ranks) must equal the unsharded step: global token count exact, advantages and dlogits bit-exact,
loss statistics to the fp64 summation order. Runs in a subprocess so the fake is what the library binds."""
import json
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")

SCRIPT = r'''
import json, os, sys, threading
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2601_07376_b200 as otk
from paper_2601_07376_b200.dist import plan_batch_shards, traj_costs
from paper_2601_07376_b200.step import MicroBatch, PolicyLossStep
from synth import make_logits, make_noise
from synth.trajectories import random_small_batch
from tests.test_dist_gloo import _sub_batch
P, credit = int(sys.argv[1]), sys.argv[2]
torch.cuda.set_device(0)
rng = np.random.default_rng(11)
tb = random_small_batch(rng, 24, max_segs=8, max_len=40, num_groups=4)
tb.group_id = (np.arange(24) % 4).astype(np.int32)      # every group straddles the ranks
V, N, dev = 4096, tb.num_rows, "cuda"
ctx0 = otk.Context(0)
logits, targets = make_logits(N, V, dtype="bf16", seed=3, device=dev)
lp = otk.otk_logprob_entropy_fwd(ctx0, logits, targets)["logp"]
old = (lp + make_noise(N, 0.05, 1, device=dev)).contiguous()
ref = (lp + make_noise(N, 0.1, 2, device=dev)).contiguous()
cfg = otk.LossCfg()
def make_step(ctx, b, **kw):
    db = otk.traj_batch_to_device(b, dev)
    return PolicyLossStep(ctx, db, torch.from_numpy(b.group_id).to(dev), 4, torch.from_numpy(b.turn_offsets).to(dev),
                          torch.from_numpy(b.turn_rewards).to(dev), V, cfg, credit=credit, gamma=0.9, **kw)
st0 = make_step(ctx0, tb)
dl0 = torch.empty_like(logits)
st0.run([MicroBatch(0, N, logits, targets, old, ref, dl0)])
torch.cuda.synchronize()
plan = plan_batch_shards(traj_costs(tb, V), P)
counts = [b1 - b0 for b0, b1 in plan]
seg_counts = [int(tb.seg_offsets[b1] - tb.seg_offsets[b0]) for b0, b1 in plan]
uid = otk.otk_comm_unique_id()
res = [None] * P
def worker(r):
    try:
        torch.cuda.set_device(0)
        with torch.cuda.stream(torch.cuda.Stream()):
            ctx = otk.Context(0)
            otk.otk_comm_init(ctx, uid, P, r)
            b0, b1 = plan[r]
            r0, r1 = int(tb.tok_offsets[b0]), int(tb.tok_offsets[b1])
            st = make_step(ctx, _sub_batch(tb, b0, b1), collectives="otk", global_num_traj=counts, global_num_groups=4,
                           global_num_segments=seg_counts)
            dl = torch.empty(r1 - r0, V, dtype=logits.dtype, device=dev)
            st.run([MicroBatch(0, r1 - r0, logits[r0:r1], targets[r0:r1], old[r0:r1], ref[r0:r1], dl)])
            torch.cuda.current_stream().synchronize()
            ctx.check()
            res[r] = dict(stats=otk.stats_dict(st.stats), n_loss=int(st.masks["n_loss"].item()),
                          adv=st.adv_used.cpu().numpy().tolist(),
                          dl_equal=bool(torch.equal(dl, dl0[r0:r1])), size=otk.otk_comm_size(ctx))
            otk.otk_comm_destroy(ctx)
    except Exception as e:  # reported to the parent
        res[r] = dict(error=repr(e))
th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
for t in th: t.start()
for t in th: t.join(180)
E = st0.adv_used.cpu().numpy()
if credit == "turn":
    offs = [int(tb.seg_offsets[b0]) for b0, _ in plan]
    ref_adv = [E[o:o + n].tolist() for o, n in zip(offs, seg_counts)]
else:
    ref_adv = [E[b0:b1].tolist() for b0, b1 in plan]
print(json.dumps(dict(ref=otk.stats_dict(st0.stats), n_loss=int(st0.masks["n_loss"].item()), ranks=res, ref_adv=ref_adv)))
'''


def _fake(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    so = str(tmp_path / "libfake_nccl.so")
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", os.path.join(CUDA, "include"),
                    os.path.join(ROOT, "tests", "fake_nccl", "fake_nccl.cc"), "-o", so, "-L",
                    os.path.join(CUDA, "lib64"), "-lcudart"], check=True, capture_output=True, text=True)
    return so


@pytest.mark.parametrize("P,credit", [(2, "trajectory"), (3, "trajectory"), (2, "turn")])
def test_batch_sharded_step_over_the_library_comm(tmp_path, P, credit):
    so = _fake(tmp_path)
    script = tmp_path / "run.py"
    script.write_text(SCRIPT.replace("ROOT", repr(ROOT), 1))
    env = dict(os.environ, OTK_NCCL_LIB=so, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, str(script), str(P), credit], capture_output=True, text=True, timeout=600,
                       env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    ref, ranks = out["ref"], out["ranks"]
    assert all(x is not None and "error" not in x for x in ranks), ranks
    for k, x in enumerate(ranks):
        assert x["size"] == [P, k]
        assert x["n_loss"] == out["n_loss"]                 # global token count (exchange 1)
        assert x["adv"] == out["ref_adv"][k]                # group statistics over the union (exchange 2), bit-exact
        assert x["dl_equal"]                                # every gradient row bit-exact
        assert x["stats"]["n_tokens"] == ref["n_tokens"]    # exchange 3
        for f in ("loss", "kl_sum", "entropy_sum", "n_clipped"):
            assert abs(x["stats"][f] - ref[f]) <= 1e-12 * max(1.0, abs(ref[f])), (f, x["stats"][f], ref[f])


SCRIPT_EMPTY = r'''
import json, sys, threading
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2601_07376_b200 as otk
torch.cuda.set_device(0)
gid = np.array([0, 1, 0, 2, 1], dtype=np.int32)
ret = np.array([1.0, 0.0, -1.0, 2.0, 0.5])
counts = [3, 0, 2]                       # rank 1 holds no trajectory
ctx0 = otk.Context(0)
ref = otk.otk_group_advantages(ctx0, torch.from_numpy(gid).cuda(), 3, returns=torch.from_numpy(ret).cuda())
ref = {k: ref[k].cpu().numpy().tolist() for k in ("adv", "group_mean", "group_std", "group_size")}
uid = otk.otk_comm_unique_id()
res = [None] * 3
def worker(r):
    try:
        torch.cuda.set_device(0)
        with torch.cuda.stream(torch.cuda.Stream()):
            ctx = otk.Context(0)
            otk.otk_comm_init(ctx, uid, 3, r)
            b0 = sum(counts[:r])
            g = torch.from_numpy(gid[b0:b0 + counts[r]].copy()).cuda()
            x = torch.from_numpy(ret[b0:b0 + counts[r]].copy()).cuda()
            o = otk.otk_batch_group_advantages(ctx, g, x, counts, 3)
            torch.cuda.current_stream().synchronize()
            ctx.check()
            res[r] = {k: o[k].cpu().numpy().tolist() for k in ("adv_all", "adv", "group_mean", "group_std", "group_size")}
            otk.otk_comm_destroy(ctx)
    except Exception as e:
        res[r] = dict(error=repr(e))
th = [threading.Thread(target=worker, args=(r,)) for r in range(3)]
for t in th: t.start()
for t in th: t.join(120)
print(json.dumps(dict(ref=ref, ranks=res)))
'''


def test_group_advantages_with_an_empty_rank(tmp_path):
    """otk_batch_group_advantages at 3 ranks with counts [3, 0, 2] (a rank without trajectories: its broadcasts are
    skipped, its slice is empty): every rank gets the single-GPU statistics of the whole batch, bit for bit."""
    so = _fake(tmp_path)
    script = tmp_path / "run_empty.py"
    script.write_text(SCRIPT_EMPTY.replace("ROOT", repr(ROOT), 1))
    env = dict(os.environ, OTK_NCCL_LIB=so, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    ref, ranks = out["ref"], out["ranks"]
    b0 = [0, 3, 3]
    for k, x in enumerate(ranks):
        assert x is not None and "error" not in x, x
        assert x["adv_all"] == ref["adv"]
        assert x["adv"] == ref["adv"][b0[k]:b0[k] + [3, 0, 2][k]]
        for f in ("group_mean", "group_std", "group_size"):
            assert x[f] == ref[f], f
