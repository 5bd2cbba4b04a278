#!/usr/bin/env python3
"""Bench records for the BASELINE.json configurations besides the headline c4 line: c1, c2,
c3 at p in {4, 6, 8, 10} (and 13), c5 -- each with its parity number from the same run.

Per (config, p): device ms per evaluation (CUDA events around `reps` back-to-back evaluate
calls after warm-up, inputs resident) and the relative L2 error of u and dgamma/dt against
the oracle O1 (float64 direct sum over the same 27^3 image cube) on a stratified target sample
(c1: all 4096 targets; c5: the committed golden values, tests/golden/).  One JSON line each.

    python scripts/bench_sweep.py [--configs c1 c2 c3 c5] [--targets 32]
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
    ap.add_argument("--configs", nargs="*", default=["c1", "c2", "c3", "c5"])
    ap.add_argument("--targets", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import numpy as np
    import torch

    import oracle
    import synthgen
    import paper_1110_2921_b200 as vf

    sweeps = {"c1": [4, 6, 8, 10, 13], "c2": [6, 10], "c3": [4, 6, 8, 10, 13], "c5": [10, 13]}
    for cfg in a.configs:
        c = synthgen.CONFIGS[cfg]
        f = synthgen.make(cfg)
        n = f.pos.shape[1]
        t0 = time.time()
        if cfg == "c5":
            g = json.load(open(os.path.join(ROOT, "tests", "golden", "c5_lam3_s0_o1.json")))
            tg = np.array(g["targets"], np.int64)
            vo, so = np.array(g["vel"]), np.array(g["dgamma"])
            src = "golden O1 (tests/golden/c5_lam3_s0_o1.json)"
        else:
            tg = np.arange(n) if n <= 4096 else synthgen.sample_targets(n, a.targets, n_lattice=f.n)
            vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 3, 0, targets=tg,
                                   batched=True)
            src = f"O1 on {len(tg)} stratified targets, {time.time() - t0:.0f} s"
        pos = torch.from_numpy(f.pos).cuda()
        gam = torch.from_numpy(f.gamma).cuda()
        vel = torch.empty_like(pos)
        dg = torch.empty_like(pos)
        for p in sweeps[cfg]:
            ev = vf.Evaluator(p=p, depth=c["depth"], image_levels=3, sigma=f.sigma,
                              box_lo=f.box_lo, box_len=f.box_len)
            for _ in range(3):
                ev.evaluate_into(pos, gam, vel, dg)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                ev.evaluate_into(pos, gam, vel, dg)
            e1.record()
            torch.cuda.synchronize()
            ev.sync_status()
            ms = e0.elapsed_time(e1) / a.reps
            st = ev.stats()
            v = vel.cpu().numpy().astype(np.float64)[:, tg]
            s = dg.cpu().numpy().astype(np.float64)[:, tg]
            eu = float(np.linalg.norm(v - vo) / np.linalg.norm(vo))
            es = float(np.linalg.norm(s - so) / np.linalg.norm(so))
            print(json.dumps({"config": cfg, "n": int(n), "p": p, "depth": c["depth"],
                              "image_levels": 3, "ms_per_eval": round(ms, 4),
                              "phase_ms": {k[3:]: round(x, 4) for k, x in st.items()
                                           if k.startswith("ms_") and x},
                              "rel_l2_u": eu, "rel_l2_dgamma": es, "oracle": src}), flush=True)
            ev.close()


if __name__ == "__main__":
    main()
