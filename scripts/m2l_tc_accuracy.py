#!/usr/bin/env python3
"""M2L engine accuracy on the GPU (investigation): local expansions per level and the
velocity / stretching of the tcgen05 engines (f16, tf32) and the SIMT engine against the
float64 step-by-step FMM oracle (same algorithm, so only arithmetic separates them).

    python scripts/m2l_tc_accuracy.py [--n 32] [--depth 3] [--p 10] [--lam 1]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import synthgen  # noqa: E402
from oracle import fmm_ref as F  # noqa: E402
import paper_1110_2921_b200 as vf  # noqa: E402


def pack(C, p, scale_n):
    out = np.zeros(C.shape[:2] + ((p + 1) ** 2,))
    for n in range(p + 1):
        out[..., n * n] = C[..., F.kidx(n, 0)].real * scale_n[n]
        for m in range(1, n + 1):
            out[..., n * n + 2 * m - 1] = C[..., F.kidx(n, m)].real * scale_n[n]
            out[..., n * n + 2 * m] = C[..., F.kidx(n, m)].imag * scale_n[n]
    return out


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--depth", type=int, default=3)
    ap.add_argument("--p", type=int, default=10)
    ap.add_argument("--lam", type=int, default=1)
    ap.add_argument("--seed", type=int, default=21)
    args = ap.parse_args()
    f = synthgen.isotropic(args.n, seed=args.seed)
    p, L = args.p, args.depth
    vo, so, st = F.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, L, p, args.lam,
                            return_stages=True)
    dev = torch.device("cuda:0")
    pos = torch.from_numpy(f.pos).to(dev)
    gam = torch.from_numpy(f.gamma).to(dev)
    res = {}
    for eng in ("simt", "f16", "tf32"):
        os.environ["VFMM_M2L"] = eng
        ev = vf.Evaluator(p=p, depth=L, image_levels=args.lam, sigma=f.sigma, box_lo=f.box_lo,
                          box_len=f.box_len)
        v, s = ev.evaluate(pos, gam)
        ev.sync_status()
        v = v.cpu().numpy().astype(np.float64)
        s = s.cpu().numpy().astype(np.float64)
        line = [f"{eng:5s} u {rel(v, vo):.3e} sdot {rel(s, so):.3e} |"]
        for l in range(1, L + 1):
            al = f.box_len / (1 << l)
            got = ev.debug_expansions(1, l)[..., 1:]
            want = pack(st["L"][l], p, al ** (np.arange(p + 1.0) + 1))[..., 1:]
            line.append(f"L{l} {rel(got, want):.2e}")
        res[eng] = (v, s)
        print(" ".join(line), flush=True)
        ev.close()
    for eng in ("f16", "tf32"):
        print(f"{eng} vs simt: u {rel(res[eng][0], res['simt'][0]):.3e} "
              f"sdot {rel(res[eng][1], res['simt'][1]):.3e}")


if __name__ == "__main__":
    main()
