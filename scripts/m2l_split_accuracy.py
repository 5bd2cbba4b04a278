#!/usr/bin/env python3
"""Order-split tcgen05 M2L (m2l_tc.cu, VFMM_M2L_SPLIT): accuracy and M2L time per split degree.

For each configuration and each split degree n0 (terms whose local and multipole degrees are
both below n0 keep the 3-product FP16 split, the rest run hi x hi alone; "full" = every term
split), one evaluation on the GPU:
  * relative L2 difference of u and dgamma/dt from the "full" run over all particles,
  * relative L2 error against O1 (float64 direct sum, 27^3 images) on stratified targets
    (c4: the committed golden values),
  * the M2L phase time (vfmm_get_stats).
One JSON line per (config, p, n0).

    python scripts/m2l_split_accuracy.py [--configs c3 c4] [--splits full 8 7 6 5 4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="*", default=["c3", "c4"])
    ap.add_argument("--ps", nargs="*", type=int, default=[10, 13])
    ap.add_argument("--splits", nargs="*", default=["full", "8", "7", "6", "5", "4"])
    ap.add_argument("--targets", type=int, default=16)
    a = ap.parse_args()
    import numpy as np
    import torch

    import oracle
    import synthgen
    import paper_1110_2921_b200 as vf

    def rel(x, y):
        return float(np.linalg.norm(x - y) / np.linalg.norm(y))

    for cfg in a.configs:
        c = synthgen.CONFIGS[cfg]
        f = synthgen.make(cfg)
        t0 = time.time()
        if cfg in ("c4", "c5"):
            g = json.load(open(os.path.join(ROOT, "tests", "golden", f"{cfg}_lam3_s0_o1.json")))
            tg = np.array(g["targets"], np.int64)
            vo, so = np.array(g["vel"]), np.array(g["dgamma"])
        else:
            tg = synthgen.sample_targets(f.pos.shape[1], a.targets, n_lattice=f.n)
            vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 3, 0,
                                   targets=tg, batched=True)
        print(f"# {cfg}: O1 reference on {len(tg)} targets ({time.time() - t0:.0f} s)",
              flush=True)
        pos = torch.from_numpy(f.pos).cuda()
        gam = torch.from_numpy(f.gamma).cuda()
        vel = torch.empty_like(pos)
        dg = torch.empty_like(pos)
        for p in a.ps:
            ref = None
            for sp in a.splits:
                os.environ["VFMM_M2L_SPLIT"] = sp
                ev = vf.Evaluator(p=p, depth=c["depth"], image_levels=3, sigma=f.sigma,
                                  box_lo=f.box_lo, box_len=f.box_len)
                ms = 0.0
                for r in range(4):
                    ev.evaluate_into(pos, gam, vel, dg)
                    if r >= 1:
                        ms += ev.stats()["ms_m2l"] / 3
                ev.sync_status()
                v = vel.cpu().numpy().astype(np.float64)
                s = dg.cpu().numpy().astype(np.float64)
                ev.close()
                if ref is None:
                    ref = (v, s)
                print(json.dumps({
                    "config": cfg, "p": p, "split": sp, "ms_m2l": round(ms, 3),
                    "u_vs_full": rel(v, ref[0]), "sdot_vs_full": rel(s, ref[1]),
                    "u_vs_o1": rel(v[:, tg], vo), "sdot_vs_o1": rel(s[:, tg], so)}), flush=True)
    os.environ.pop("VFMM_M2L_SPLIT", None)


if __name__ == "__main__":
    main()
