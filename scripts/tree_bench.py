"""Treecode (vfmm_evaluate_tree) vs the uniform FMM (vfmm_evaluate) on one
configuration: device ms per evaluation (CUDA events, after warm-up), the interaction counts,
and the difference between the two (both approximate Eqs. 5 / 8).  Usage:
  python scripts/tree_bench.py --config c3 --p 10 --theta 0.5 --ncrit 64 [--clustered N]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthgen  # noqa: E402
import paper_1110_2921_b200 as vf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--clustered", type=int, default=0)
    ap.add_argument("--p", type=int, default=10)
    ap.add_argument("--depth", type=int, default=0)
    ap.add_argument("--theta", type=float, default=0.5)
    ap.add_argument("--ncrit", type=int, default=64)
    ap.add_argument("--lam", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    f = synthgen.clustered(a.clustered) if a.clustered else synthgen.make(a.config)
    ev = vf.Evaluator(p=a.p, depth=a.depth, image_levels=a.lam, sigma=f.sigma, box_lo=f.box_lo,
                      box_len=f.box_len)
    pos = torch.from_numpy(f.pos).cuda()
    gam = torch.from_numpy(f.gamma).cuda()
    out = {"field": f.name, "n": pos.shape[1], "p": a.p, "theta": a.theta, "ncrit": a.ncrit,
           "lam": a.lam}
    for name, fn in (("fmm", lambda: ev.evaluate(pos, gam)),
                     ("tree", lambda: ev.evaluate_tree(pos, gam, a.theta, a.ncrit))):
        r = fn()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(a.reps):
            r = fn()
        t1.record()
        torch.cuda.synchronize()
        st = ev.stats()
        out[name] = {"ms": t0.elapsed_time(t1) / a.reps, "depth": st["depth_used"],
                     "ms_p2p": st["ms_p2p"], "pairs": st["n_p2p_pairs"], "m2l": st["n_m2l"]}
        out[name + "_v"] = r
    v1, s1 = out.pop("fmm_v")
    v2, s2 = out.pop("tree_v")
    out["tree_vs_fmm_u"] = float((v1 - v2).norm() / v1.norm())
    out["tree_vs_fmm_s"] = float((s1 - s2).norm() / s1.norm())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
