import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2601_07376_b200 as otk
from oracle import oracle_ref as O
from tests.gpu_common import row_problem, oracle_cfg
V, n, scale = 151936, 24, 1/0.7
d, h = row_problem(n, V, dtype="f32", seed=7*V+n, force_clip=3, logit_scale=scale, uniform_rows=(1,))
ctx = otk.Context(0)
cfg = otk.LossCfg(kl_beta=0.04, kl_type=3, logit_scale=scale)
N = int(h["mask"].sum())
nl = torch.tensor([N], dtype=torch.int64, device="cuda")
got = otk.otk_policy_loss_fwd_bwd(ctx, d["logits"], d["targets"], d["mask"], d["row_traj"], d["adv"], d["old"], d["ref"], nl, cfg)
ctx.check()
want = O.policy_loss_fwd_bwd(h["wide"], h["targets"], h["mask"], h["row_traj"], h["adv"], h["old"], h["ref"], N, oracle_cfg(cfg))
g = got["dlogits"].double().cpu().numpy()
for j in range(n):
    if not h["mask"][j]: continue
    w = want["dlogits"][j]; c = want["coef"][j]
    tol = 1e-5*np.abs(w) + 1e-5*abs(c) + 1e-30
    r = np.abs(g[j]-w)/tol
    k = int(np.argmax(r))
    print(j, "ratio %.3f" % r[k], "col", k, "target", h["targets"][j], "got %.9e want %.9e coef %.4e x %.4f" % (g[j,k], w[k], c, h["wide"][j,k]),
          "logp gpu %.7f or %.7f" % (got["logp"][j].item(), want["logp"][j]))
