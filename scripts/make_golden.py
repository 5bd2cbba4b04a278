#!/usr/bin/env python3
"""Write tests/golden/<cfg>_lam3_o1.json: oracle O1 (float64 direct periodic sum, oracle/ only)
at the benched image count -- the 27^3 cube, image_levels = 3 ("3^3 x 3^3 x 3^3
- 1" images, :361 "27^3 periodic images") -- for a seeded stratified sample of targets of the
full-size configurations c4 / c5 (BASELINE.json configs[3], [4]).

Calls only oracle/ and synthgen/ (the seeded input generators).  Nothing here comes from the
CUDA path.  vfmm_oracle_eval_batched gives bitwise vfmm_oracle_eval's result
(tests/test_oracle_pins.py::test_batched_oracle_is_bitwise_the_plain_one).

    python scripts/make_golden.py c4 [--targets 16] [--threads 8]

About 1 h per configuration on 8 AVX-512 cores (1.06e13 / 2 pair evaluations).
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synthgen  # noqa: E402


def field_digest(f):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(f.pos, np.float32).tobytes())
    h.update(np.ascontiguousarray(f.gamma, np.float32).tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--targets", type=int, default=16)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--image-levels", type=int, default=3)
    ap.add_argument("--scheme", type=int, default=0)
    args = ap.parse_args()
    f = synthgen.make(args.cfg)
    n = f.pos.shape[1]
    tg = synthgen.sample_targets(n, args.targets, n_lattice=f.n)
    t0 = time.time()
    vel, dg = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, args.image_levels,
                            args.scheme, targets=tg, nthreads=args.threads, batched=True,
                            native=True)
    dt = time.time() - t0
    out = {
        "_source": ("oracle O1 (oracle/oracle.c vfmm_oracle_eval_batched, float64 direct sum over "
                    "the image cube) written by scripts/make_golden.py; no CUDA involved"),
        "cite": "PAPER.md:81 Eq.(5), :100 Eq.(8), :164/:361 27^3 images; SURVEY.md 8(c) O1",
        "config": args.cfg, "field": f.name, "n": int(n), "sigma": f.sigma,
        "box_lo": f.box_lo, "box_len": f.box_len, "image_levels": args.image_levels,
        "scheme": args.scheme, "field_sha256": field_digest(f),
        "targets": tg.tolist(), "vel": vel.tolist(), "dgamma": dg.tolist(),
        "oracle_seconds": dt, "threads": args.threads or os.cpu_count(),
    }
    path = os.path.join(ROOT, "tests", "golden",
                        f"{args.cfg}_lam{args.image_levels}_s{args.scheme}_o1.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote {path} in {dt:.0f} s")


if __name__ == "__main__":
    main()
