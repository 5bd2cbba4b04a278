#!/usr/bin/env python3
"""Numerical model of the tensor-core M2L's arithmetic (investigation, not a test).

Emulates, in numpy, the scaled 3xFP16 split of m2l_tc.cu on one level of a real field:
balanced operators Ahat = T / (rs cs) and multipoles Mhat = M cs s split into half hi + lo,
exact products, an accumulator chain per MMA (16 products + accumulator) rounded to FP32
toward zero (the tensor core's truncation) or to nearest, flushed into round-to-nearest FP32
registers every `flush` chain -- against the float64 result and against a plain FP32
(round-to-nearest) gather-GEMM like the SIMT kernel.

    python scripts/m2l_precision.py [--n 32] [--depth 3] [--p 10]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402
from oracle import fmm_ref as F  # noqa: E402


def pack_vec(C, p):
    """complex [.., full] -> packed real [.., (p+1)^2]"""
    out = np.zeros(C.shape[:-1] + ((p + 1) ** 2,))
    for n in range(p + 1):
        out[..., n * n] = C[..., F.kidx(n, 0)].real
        for m in range(1, n + 1):
            out[..., n * n + 2 * m - 1] = C[..., F.kidx(n, m)].real
            out[..., n * n + 2 * m] = C[..., F.kidx(n, m)].imag
    return out


def pack_op(A, p):
    nc = (p + 1) ** 2
    P = np.zeros((nc, nc))
    for n in range(p + 1):
        for m in range(n + 1):
            for part in range(1 if m == 0 else 2):
                j = n * n + (0 if m == 0 else 2 * m - 1 + part)
                v = np.zeros((p + 1) ** 2, np.complex128)
                c = 1.0 if part == 0 else 1j
                v[F.kidx(n, m)] = c
                if m > 0:
                    v[F.kidx(n, -m)] = (-1) ** m * np.conj(c)
                P[:, j] = pack_vec(A @ v, p)
    return P


def pow2_ceil(x):
    return np.where(x > 0, 2.0 ** np.ceil(np.log2(np.where(x > 0, x, 1.0))), 1.0)


def half_split(x):
    h = x.astype(np.float16).astype(np.float64)
    lo = (x - h).astype(np.float16).astype(np.float64)
    return h, lo


def to32(x, rz):
    y = x.astype(np.float32)
    if rz:
        over = np.abs(y.astype(np.float64)) > np.abs(x)
        y = np.where(over, np.nextafter(y, np.float32(0)), y)
    return y.astype(np.float64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--depth", type=int, default=3)
    ap.add_argument("--p", type=int, default=10)
    ap.add_argument("--level", type=int, default=0)
    args = ap.parse_args()
    p, L = args.p, args.depth
    lev = args.level or L
    nc = (p + 1) ** 2
    f = synthgen.isotropic(args.n, seed=21)
    t0 = time.time()
    _, _, st = F.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, L, p, 0,
                          return_stages=True)
    a = f.box_len / (1 << lev)
    M = pack_vec(st["M"][lev] / (a ** np.array([n for n in range(p + 1) for _ in range(2 * n + 1)])), p)
    print(f"fp64 FMM stages {time.time() - t0:.1f} s; level {lev}: {M.shape[0]} cells")
    # operators for all 316 offsets, packed real, scaled (a = 1)
    offs = [(x, y, z) for x in range(-3, 4) for y in range(-3, 4) for z in range(-3, 4)
            if max(abs(x), abs(y), abs(z)) > 1]
    T = {o: pack_op(F.m2l_matrix(-np.array(o, np.float64), p), p) for o in offs}
    allT = np.stack(list(T.values()))
    cs = pow2_ceil(np.abs(allT).max(axis=(0, 1)))          # column scale over slots and rows
    rs = pow2_ceil((np.abs(allT) / cs).max(axis=(0, 2)))    # row scale of the column-scaled rows
    mx = np.abs(M * cs).max()
    s = 2.0 ** (14 - np.frexp(mx)[1])
    side = 1 << lev
    ncell = side ** 3
    # target cell -> list of (offset, source cell), Morton order, periodic
    dec = [F._m_decode(c, lev) for c in range(ncell)]
    enc = {d: c for c, d in enumerate(dec)}
    lists = []
    for t in range(ncell):
        tx, ty, tz = dec[t]
        px, py, pz = tx >> 1, ty >> 1, tz >> 1
        lst = []
        for sx in range(2 * px - 2, 2 * px + 4):
            for sy in range(2 * py - 2, 2 * py + 4):
                for sz in range(2 * pz - 2, 2 * pz + 4):
                    o = (sx - tx, sy - ty, sz - tz)
                    if max(abs(o[0]), abs(o[1]), abs(o[2])) <= 1:
                        continue
                    lst.append((o, enc[(sx % side, sy % side, sz % side)]))
        lists.append(lst)
    nl = len(lists[0])
    src = np.array([[c for _, c in lst] for lst in lists])          # [t][189]
    ops = [[o for o, _ in lst] for lst in lists]
    # exact and emulated sums, vectorised over the target cells of one parity (same offset order)
    Ahat = {o: T[o] / (rs[:, None] * cs[None, :]) for o in offs}
    Ah = {o: half_split(Ahat[o]) for o in offs}
    Mh_hi, Mh_lo = half_split(M * cs * s)
    exact = np.zeros((ncell, 3, nc))
    f32 = np.zeros((ncell, 3, nc))
    # strategy: (rounding of the MMA chain, flush granularity, cross terms in their own chain)
    strategies = {"rz_group3": ("rz", "group3", False), "rz_offset": ("rz", "offset", False),
                  "rz_kc": ("rz", "kc", False), "rz_group3_sepx": ("rz", "group3", True),
                  "rz_offset_sepx": ("rz", "offset", True), "rn_group3": ("rn", "group3", False)}
    results = {k: np.zeros((ncell, 3, nc)) for k in strategies}
    t0 = time.time()
    par = np.array([(d[0] & 1) | ((d[1] & 1) << 1) | ((d[2] & 1) << 2) for d in dec])
    for pi in range(8):
        tc = np.nonzero(par == pi)[0]
        olist = ops[tc[0]]
        assert all(ops[t] == olist for t in tc)
        acc = {k: np.zeros((len(tc), 3, nc)) for k in strategies}
        ch = {k: np.zeros((len(tc), 3, nc)) for k in strategies}
        chx = {k: np.zeros((len(tc), 3, nc)) for k in strategies}
        e = np.zeros((len(tc), 3, nc))
        g = np.zeros((len(tc), 3, nc), np.float32)

        def flush(k):
            acc[k] = to32(acc[k] + ch[k], False)
            acc[k] = to32(acc[k] + chx[k], False)
            ch[k][:] = 0
            chx[k][:] = 0

        for i, o in enumerate(olist):
            sc = src[tc, i]
            Ms = M[sc]
            e += Ms @ T[o].T
            g = (g + (Ms.astype(np.float32) @ T[o].T.astype(np.float32))).astype(np.float32)
            hi, lo = Ah[o]
            bh, bl = Mh_hi[sc], Mh_lo[sc]
            for kc in range(2):
                for ks in range(4):
                    k0 = kc * 64 + ks * 16
                    if k0 >= nc:
                        continue
                    sl = slice(k0, min(k0 + 16, nc))
                    phh = bh[..., sl] @ hi[:, sl].T
                    phl = bl[..., sl] @ hi[:, sl].T
                    plh = bh[..., sl] @ lo[:, sl].T
                    for k, (rnd, fl, sepx) in strategies.items():
                        rz = rnd == "rz"
                        ch[k] = to32(ch[k] + phh, rz)
                        if sepx:
                            chx[k] = to32(chx[k] + phl, rz)
                            chx[k] = to32(chx[k] + plh, rz)
                        else:
                            ch[k] = to32(ch[k] + phl, rz)
                            ch[k] = to32(ch[k] + plh, rz)
                for k, (rnd, fl, sepx) in strategies.items():
                    if fl == "kc":
                        flush(k)
            for k, (rnd, fl, sepx) in strategies.items():
                if fl == "offset" or (fl == "group3" and (i % 3 == 2 or i == len(olist) - 1)):
                    flush(k)
        exact[tc] = e
        f32[tc] = g
        for k in strategies:
            results[k][tc] = acc[k] * rs[None, None, :nc] / s
    print(f"emulation {time.time() - t0:.1f} s")
    nrm = np.linalg.norm(exact[..., 1:])

    def err(x):
        return np.linalg.norm((x - exact)[..., 1:]) / nrm

    print(f"fp32 RN gather-GEMM (SIMT-like): {err(f32.astype(np.float64)):.3e}")
    for k, v in results.items():
        print(f"3xFP16 {k}: {err(v):.3e}")


if __name__ == "__main__":
    main()
