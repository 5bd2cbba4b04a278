"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for arXiv:1110.2921's hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The CUDA product
(``paper_1110_2921_b200``) never imports it and shares no code with it.

Contents
--------
* ``liboracle.so`` (``oracle/oracle.c``): double-precision direct periodic
  image summation of the regularized Biot-Savart velocity (Eq. 5)
  and vortex stretching (Eq. 8), scalar kernels zeta/g/f/q
  (PAPER.md:76, :86), and the Morton-ordered uniform octree (bit-exact contract).
* ``fmm_ref`` : a step-by-step float64 numpy FMM (P2M, M2M, periodic images,
  M2L, L2L, L2P, P2P) following PAPER.md Eqs. (10)-(15) in Cheng et al.'s
  nomenclature, used for per-stage parity.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path(native: bool = False) -> str:
    return os.path.join(_HERE, "liboracle_native.so" if native else "liboracle.so")


def build(force: bool = False, native: bool = False) -> str:
    """Compile liboracle.so with gcc (-O3 -fopenmp -ffp-contract=off, no fast-math;
    -fno-math-errno only drops errno writes, results are unchanged).  native=True builds a
    -march=native copy (liboracle_native.so) for long runs on this host only (same source,
    same IEEE operations: see test_batched_oracle_is_bitwise_the_plain_one)."""
    import subprocess

    out = lib_path(native)
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call([
            "gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fno-math-errno",
            "-fPIC", "-shared", *(["-march=native", "-mprefer-vector-width=512"] if native else []), "-o", out, src, "-lm",
        ])
    return out


_LIBS = {}


def _lib(native: bool = False):
    if native not in _LIBS:
        path = build(native=native)
        L = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        L.vfmm_oracle_kernels.argtypes = [ctypes.c_double, ctypes.c_double, dp, dp, dp, dp]
        L.vfmm_oracle_kernels.restype = None
        for fn in (L.vfmm_oracle_eval, L.vfmm_oracle_eval_batched, L.vfmm_oracle_eval_sigma):
            fn.argtypes = [
                ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                ctypes.c_void_p if fn is L.vfmm_oracle_eval_sigma else ctypes.c_double,
                ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                ctypes.c_void_p, ctypes.c_int,
            ]
            fn.restype = ctypes.c_int
        L.vfmm_oracle_morton.argtypes = [
            ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_float,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
        ]
        L.vfmm_oracle_morton.restype = ctypes.c_int
        _LIBS[native] = L
    return _LIBS[native]


def kernels(r: float, sigma: float):
    """(zeta, g, f, q) at distance r -- PAPER.md Eqs. (4), (6); f = g/(4 pi r^3), q = f'/r."""
    z, g, f, q = (ctypes.c_double() for _ in range(4))
    _lib().vfmm_oracle_kernels(float(r), float(sigma), ctypes.byref(z), ctypes.byref(g),
                               ctypes.byref(f), ctypes.byref(q))
    return z.value, g.value, f.value, q.value


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def direct(pos, gamma, sigma, box_lo, box_len, image_levels=3, scheme=0, targets=None,
           probe_pos=None, probe_gamma=None, nthreads=0, batched=False, native=False):
    """see _direct; sigma may be an array of per-source core radii (Eq. 6's sigma_j)"""
    return _direct(pos, gamma, sigma, box_lo, box_len, image_levels, scheme, targets,
                   probe_pos, probe_gamma, nthreads, batched, native)


def _direct(pos, gamma, sigma, box_lo, box_len, image_levels=3, scheme=0, targets=None,
            probe_pos=None, probe_gamma=None, nthreads=0, batched=False, native=False):
    """Direct periodic-image sum (oracle O1).

    pos, gamma: (3, N) arrays (SoA); values are widened exactly to float64.
    targets: optional int index array into the sources; probe_pos/probe_gamma: (3, T)
    explicit probes (targets != sources).  Returns (vel, dgamma), each (3, T) float64.
    batched=True runs vfmm_oracle_eval_batched (bitwise the same result, one pass over the
    sources per image serves 16 targets: for long sampled-target runs).
    """
    pos = _c(pos, np.float64)
    gamma = _c(gamma, np.float64)
    n = pos.shape[1]
    if probe_pos is not None:
        tp = _c(probe_pos, np.float64)
        tg = _c(probe_gamma, np.float64)
        nt = tp.shape[1]
        tidx = None
    else:
        tidx = _c(np.arange(n) if targets is None else targets, np.int64)
        nt = tidx.shape[0]
        tp = tg = None
    vel = np.zeros((3, nt), np.float64)
    dg = np.zeros((3, nt), np.float64)
    L = _lib(native)
    tail = (float(box_lo), float(box_len), int(image_levels), int(scheme), nt,
            None if tidx is None else tidx.ctypes.data, None if tp is None else tp.ctypes.data,
            None if tg is None else tg.ctypes.data, vel.ctypes.data, dg.ctypes.data,
            int(nthreads))
    if np.ndim(sigma) > 0:  # per-source core radii (plain loop nest)
        sig = _c(np.broadcast_to(np.asarray(sigma, np.float64), (n,)), np.float64)
        rc = L.vfmm_oracle_eval_sigma(n, pos.ctypes.data, gamma.ctypes.data, sig.ctypes.data,
                                      *tail)
    else:
        rc = (L.vfmm_oracle_eval_batched if batched else L.vfmm_oracle_eval)(
            n, pos.ctypes.data, gamma.ctypes.data, float(sigma), *tail)
    if rc != 0:
        raise ValueError(f"vfmm_oracle_eval failed: {rc}")
    return vel, dg


def morton(pos_f32, depth, lo, length):
    """Oracle Morton tree: (keys_sorted u32, perm u32, leaf_start i32[8^depth+1], status)."""
    pos = _c(pos_f32, np.float32)
    n = pos.shape[1]
    keys = np.zeros(n, np.uint32)
    perm = np.zeros(n, np.uint32)
    ls = np.zeros((1 << (3 * depth)) + 1, np.int32)
    rc = _lib().vfmm_oracle_morton(n, pos.ctypes.data, int(depth), float(np.float32(lo)),
                                   float(np.float32(length)), keys.ctypes.data,
                                   perm.ctypes.data, ls.ctypes.data)
    if rc == -1:
        raise ValueError("vfmm_oracle_morton: bad parameters")
    return keys, perm, ls, rc
