"""Diagnostic (GPU): FP32 rounding of the two classical-scheme P2P accumulations
(VFMM_P2P=cross: per-pair gamma_j x d; default: staged s_j = gamma_j x x_j) against the
float64 oracles.  Prints relative L2 errors; test infrastructure (uses oracle/)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synthgen  # noqa: E402
from oracle import fmm_ref as F  # noqa: E402
import paper_1110_2921_b200 as vf  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def run(field, **kw):
    ev = vf.Evaluator(sigma=field.sigma, box_lo=field.box_lo, box_len=field.box_len, **kw)
    pos = torch.from_numpy(np.ascontiguousarray(field.pos)).cuda()
    gam = torch.from_numpy(np.ascontiguousarray(field.gamma)).cuda()
    v, s = ev.evaluate(pos, gam)
    ev.sync_status()
    out = v.cpu().numpy().astype(np.float64), s.cpu().numpy().astype(np.float64)
    ev.close()
    return out


cases = []
f1 = synthgen.jitter(synthgen.taylor_green(12), seed=5)
o1 = oracle.direct(f1.pos, f1.gamma, f1.sigma, f1.box_lo, f1.box_len, 0, 0)
cases.append(("TG12 jitter depth1 near-only vs direct", f1,
              dict(p=2, depth=1, image_levels=0, mode=vf.MODE_NEAR_ONLY), o1))
for name, depth, p, lam in [("c1", 2, 4, 3), ("iso16", 2, 6, 2), ("iso32", 3, 6, 1)]:
    f = synthgen.make("c1") if name == "c1" else synthgen.isotropic(int(name[3:]), seed=7)
    o = F.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, depth, p, lam, 0)
    cases.append((f"{name} depth{depth} p{p} FMM vs fp64 FMM oracle", f,
                   dict(p=p, depth=depth, image_levels=lam), (o[0], o[1])))
for mode in ["cross", "sj"]:
    os.environ["VFMM_P2P"] = mode
    for label, f, kw, (vo, so) in cases:
        v, s = run(f, **kw)
        print(f"{mode:5s} {label:48s} u {rel(v, vo):.3e}  sdot {rel(s, so):.3e}", flush=True)
