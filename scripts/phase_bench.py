#!/usr/bin/env python3
"""Per-phase device times (vfmm_get_stats CUDA events) of the bench workload under a set of
environment variants -- a measurement knob sweep, not the bench line.

    python scripts/phase_bench.py --config c4 --variants "VFMM_P2P_CFG=b3u1" "VFMM_M2L=simt"
Each variant runs in a fresh process (the library reads the knobs at launch time)."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg, p, depth, reps):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import synthgen
    import paper_1110_2921_b200 as vf

    c = synthgen.CONFIGS[cfg]
    f = synthgen.make(cfg)
    ev = vf.Evaluator(p=p or c["p"], depth=depth or c["depth"], image_levels=3, sigma=f.sigma,
                      box_lo=f.box_lo, box_len=f.box_len)
    pos = torch.from_numpy(f.pos).cuda()
    gam = torch.from_numpy(f.gamma).cuda()
    vel = torch.empty_like(pos)
    dg = torch.empty_like(pos)
    acc = {}
    for r in range(reps + 2):
        ev.evaluate_into(pos, gam, vel, dg)
        st = ev.stats()
        if r >= 2:
            for k, v in st.items():
                if k.startswith("ms_"):
                    acc[k] = acc.get(k, 0.0) + v / reps
    ev.sync_status()
    print(json.dumps({k: round(v, 4) for k, v in acc.items()}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--p", type=int, default=0)
    ap.add_argument("--depth", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", nargs="*", default=[""])
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        return child(a.config, a.p, a.depth, a.reps)
    for v in a.variants:
        env = dict(os.environ)
        for kv in v.split():
            k, _, val = kv.partition("=")
            env[k] = val
        out = subprocess.run([sys.executable, __file__, "--child", "--config", a.config,
                              "--p", str(a.p), "--depth", str(a.depth), "--reps", str(a.reps)],
                             env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
        print(f"{v or 'default'}: {line}", flush=True)


if __name__ == "__main__":
    main()
