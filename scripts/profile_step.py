"""One warm-up + N evaluations of a config (for ncu launch lists / full captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthgen  # noqa: E402
import paper_1110_2921_b200 as vf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--p", type=int, default=0)
ap.add_argument("--depth", type=int, default=0)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--m2l", default="")
a = ap.parse_args()
if a.m2l:
    os.environ["VFMM_M2L"] = a.m2l
c = synthgen.CONFIGS[a.config]
f = synthgen.make(a.config)
ev = vf.Evaluator(p=a.p or c["p"], depth=a.depth or c["depth"], image_levels=3, sigma=f.sigma,
                  box_lo=f.box_lo, box_len=f.box_len)
pos = torch.from_numpy(f.pos).cuda()
gam = torch.from_numpy(f.gamma).cuda()
for _ in range(1 + a.steps):
    v, s = ev.evaluate(pos, gam)
ev.sync_status()
torch.cuda.synchronize()
print("stats", ev.stats())
