"""TEST INFRASTRUCTURE ONLY -- step-by-step float64 oracle of the hybrid treecode's
cell-particle traversal (numpy).  Only tests/ may import it; the CUDA product never does.

PAPER.md:148-152 (section 3.2, "Hybrid treecode-FMM with auto-tuning"): "The traversal is
based on a stack data structure, and allows the interactions in the algorithm to be of
cell-cell or cell-particle type, while at the same time automatically choosing the number of
particles per box at the deepest levels of the tree".  The cell-cell half is the FMM of
``fmm_ref.evaluate``; this module is the cell-particle half, in the paper's terms:

  1. the Morton octree of depth L (same keys as the FMM, ``oracle.morton``);
  2. adaptive leaves ("choosing the number of particles per box"): a non-empty cell of level
     l >= 1 is a leaf when it holds <= n_crit particles or l = L, and its parent is not a leaf
     (reading R22 in DESIGN.md);
  3. the multipole of every cell, Eq. (10) about the cell centre: straight
     from its particles (``fmm_ref.p2m``) -- the definition the FMM's M2M reaches exactly;
  4. per target leaf B, a stack traversal from the near 3^3 root images (reading R5):
     pop cell S; if r_S + r_B < theta |c_B - c_S| (r = half diagonal, reading R22; evaluated
     exactly as 0.75 (w_S + w_B)^2 < theta^2 d^2 in leaf widths) the cell
     interacts with each target of B through its multipole (M2P: Eq. (11)'s local expansion
     at the target point itself, rows n <= 2 of ``fmm_ref.m2l_matrix``'s formula, then Eqs. (12)-(15)'s gradient and
     Hessian at the expansion centre, ``fmm_ref.l2p`` at 0; the cutoff is dropped in the far
     field); else if S is a leaf, particle-particle by Eq. (5) / (8) exactly
     (``fmm_ref.pair_sum``); else push S's non-empty children.  An accepted
     cell holding fewer than (p+1)^2 particles also acts particle-particle (exact and cheaper
     than its multipole: the cell-particle / particle-particle choice, reading R22);
  5. images outside the near 3^3 block by multipole expansions: the root's
     local expansion ``fmm_ref.periodic_far`` evaluated at each particle (L2P about the box
     centre).
Everything is float64.  Pins: tests/test_oracle_pins.py (theta = 0 is the direct sum; M2P of
one cell converges to the cell's direct sum as p grows; theta -> small with high p approaches
the direct sum; the adaptive leaves partition the particles).
"""
from __future__ import annotations

import math

import numpy as np

from . import fmm_ref as F
from . import morton as _morton

_EPS = np.zeros((3, 3, 3))
_EPS[0, 1, 2] = _EPS[1, 2, 0] = _EPS[2, 0, 1] = 1.0
_EPS[0, 2, 1] = _EPS[2, 1, 0] = _EPS[1, 0, 2] = -1.0


def _decode(c: int, l: int):
    return F._m_decode(c, l)


_M2P_CACHE = {}


def _m2p_index(p: int):
    """Rows n <= 2 of Eq. (11)'s M2L, L_n^m = sum_{k,l} (-1)^{n+m} I_{n+k}^{l-m} M_k^l
    (``fmm_ref.m2l_matrix``), as index / sign arrays over I of degree <= p + 2; and the linear
    map of ``fmm_ref.l2p`` at the expansion centre from the 9 coefficients (real, imaginary
    parts) to the gradient and Hessian."""
    if p not in _M2P_CACHE:
        nc = F.ncoef(p)
        idx = np.zeros((9, nc), np.int64)
        sgn = np.zeros((9, nc))
        for n in range(3):
            for m in range(-n, n + 1):
                for k in range(p + 1):
                    for l in range(-k, k + 1):
                        idx[F.kidx(n, m), F.kidx(k, l)] = F.kidx(n + k, l - m)
                        sgn[F.kidx(n, m), F.kidx(k, l)] = (-1) ** ((n + m) & 1)
        # l2p is real-linear in (Re L, Im L): map from the 18 real parts, column by column
        Bg = np.zeros((18, 3))
        Bh = np.zeros((18, 3, 3))
        for j in range(18):
            Lb = np.zeros((3, 9), np.complex128)
            Lb[0, j % 9] = 1.0 if j < 9 else 1.0j
            g_, h_ = F.l2p(Lb, np.zeros((1, 3)), 2)
            Bg[j] = g_[0, 0]  # component 0 carries the basis vector
            Bh[j] = h_[0, 0]
        _M2P_CACHE[p] = (idx, sgn, Bg, Bh)
    return _M2P_CACHE[p]


def m2p(Ms, D, p: int):
    """Cell-particle interactions: multipoles Ms (C, 3, nc) about cell centres c_q evaluated at
    the points c_q + D[:, q] (D: (K, C, 3)), summed over the cells q.  Returns grad (K, 3c, 3a)
    and hess (K, 3c, 3a, 3b) of phi_c (no cutoff in the far field)."""
    idx, sgn, Bg, Bh = _m2p_index(p)
    K, C = D.shape[0], D.shape[1]
    I = F.solid_I(D.reshape(K * C, 3), p + 2).reshape(K, C, -1)
    A = I[:, :, idx] * sgn  # (K, C, 9, nc)
    L2 = np.einsum("kqrj,qcj->kcr", A, Ms)  # (K, 3c, 9): order-2 local expansion at each point
    Lr = np.concatenate([L2.real, L2.imag], axis=-1)  # (K, 3c, 18)
    grad = np.einsum("kcj,ja->kca", Lr, Bg)
    hess = np.einsum("kcj,jab->kcab", Lr, Bh)
    return grad, hess


def adaptive_leaves(leaf_start, L: int, n_crit: int):
    """Step 2: list of (level, cell) leaves, levels >= 1."""
    out = []

    def count(l, c):
        sh = 3 * (L - l)
        return int(leaf_start[(c + 1) << sh] - leaf_start[c << sh])

    stack = [(1, c) for c in range(8)]
    while stack:
        l, c = stack.pop()
        k = count(l, c)
        if k == 0:
            continue
        if l == L or k <= n_crit:
            out.append((l, c))
        else:
            stack.extend((l + 1, 8 * c + ch) for ch in range(8))
    return sorted(out)


def evaluate(pos, gam, sigma, box_lo, box_len, depth, p, theta, n_crit, image_levels=3,
             scheme=0, return_info=False):
    """pos, gam: (3, N) float32 inputs (widened exactly).  Returns (vel, dgam) (3, N) in input
    order [, info dict with the leaves and interaction counts]."""
    pos = np.asarray(pos)
    N = pos.shape[1]
    lo = float(np.float32(box_lo))
    ln = float(np.float32(box_len))
    L = int(depth)
    keys, perm, leaf_start, rc = _morton(np.asarray(pos, np.float32), L, lo, ln)
    if rc != 0:
        raise ValueError("positions outside the box")
    perm = perm.astype(np.int64)
    X = np.asarray(pos, np.float64).T[perm]
    G = np.asarray(gam, np.float64).T[perm]

    def rng(l, c):
        sh = 3 * (L - l)
        return int(leaf_start[c << sh]), int(leaf_start[(c + 1) << sh])

    def center(l, c):
        ix, iy, iz = _decode(c, l)
        w = ln / (1 << l)
        return np.array([lo + (ix + 0.5) * w, lo + (iy + 0.5) * w, lo + (iz + 0.5) * w])

    leaves = adaptive_leaves(leaf_start, L, n_crit)
    leafset = set(leaves)

    def is_leaf(l, c):
        return (l, c) in leafset

    mcache = {}

    def multipole(l, c):  # step 3
        if (l, c) not in mcache:
            s, e = rng(l, c)
            mcache[(l, c)] = F.p2m(X[s:e] - center(l, c), G[s:e], p)
        return mcache[(l, c)]

    # MAC r_S + r_B < theta d with r = (sqrt 3 / 2) w, squared and in leaf widths (exact
    # half-integer centre offsets): 0.75 (w_S + w_B)^2 < theta^2 d^2, theta rounded to float32
    # as the C ABI receives it (so that ties decide the same way on both sides, reading R22)
    th = float(np.float32(theta))
    th2 = th * th
    # an accepted cell with fewer than (p+1)^2 particles interacts particle-particle: exact,
    # and cheaper than its multipole (reading R22)
    n_direct = (p + 1) ** 2

    def cell_lw(l, c):  # centre (leaf widths from the box corner) and width of a cell
        ix, iy, iz = _decode(c, l)
        w = float(1 << (L - l))
        return np.array([(ix + 0.5) * w, (iy + 0.5) * w, (iz + 0.5) * w]), w
    if image_levels > 0:
        images = [(a, b, d) for a in (-1, 0, 1) for b in (-1, 0, 1) for d in (-1, 0, 1)]
    else:
        images = [(0, 0, 0)]
    grad = np.zeros((N, 3, 3))
    hess = np.zeros((N, 3, 3, 3))
    vel = np.zeros((N, 3))
    dg = np.zeros((N, 3))
    n_m2p = 0
    n_pairs = 0
    for (lb, cb) in leaves:  # step 4
        s, e = rng(lb, cb)
        xi, gi = X[s:e], G[s:e]
        cBw, wB = cell_lw(lb, cb)
        stack = [(0, 0, np.array(o, np.float64)) for o in images]
        xs_list, gs_list, acc = [], [], []
        while stack:
            l, c, o = stack.pop()
            sh = o * ln
            cS = center(l, c) + sh
            cSw, wS = cell_lw(l, c)
            dd = cBw - (cSw + o * float(1 << L))
            d2 = dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2]
            s2, e2 = rng(l, c)
            if 0.75 * (wS + wB) ** 2 < th2 * d2 and e2 - s2 >= n_direct:
                acc.append((multipole(l, c), cS))
                n_m2p += e - s
            elif 0.75 * (wS + wB) ** 2 < th2 * d2 or is_leaf(l, c):
                s2, e2 = rng(l, c)
                xs_list.append(X[s2:e2] + sh)
                gs_list.append(G[s2:e2])
            else:
                for ch in range(8):
                    a, b = rng(l + 1, 8 * c + ch)
                    if b > a:
                        stack.append((l + 1, 8 * c + ch, o))
        for q0 in range(0, len(acc), 32):  # the accepted cells, in chunks
            ch = acc[q0:q0 + 32]
            Ms = np.stack([a[0] for a in ch])
            D = xi[:, None, :] - np.stack([a[1] for a in ch])[None, :, :]
            g_, h_ = m2p(Ms, D, p)
            grad[s:e] += g_
            hess[s:e] += h_
        if xs_list:
            xs, gs = np.concatenate(xs_list), np.concatenate(gs_list)
            un, sn = F.pair_sum(xi, gi, xs, gs, sigma, scheme)
            vel[s:e] += un
            dg[s:e] += sn
            n_pairs += (e - s) * len(xs)
    if image_levels >= 2:  # step 5
        M0 = F.p2m(X - center(0, 0), G, p)
        L0 = F.periodic_far(M0, ln, image_levels, p)
        g_, h_ = F.l2p(L0, X - center(0, 0), p)
        grad += g_
        hess += h_
    # u_a = eps_abc d_b phi_c / 4 pi; stretching as in fmm_ref.evaluate (reading R10)
    vel += np.einsum("abc,kcb->ka", _EPS, grad) / F.FOUR_PI
    if scheme == 0:
        dg += np.einsum("abc,kcdb,kd->ka", _EPS, hess, G) / F.FOUR_PI
    else:
        dg += np.einsum("dbc,kcab,kd->ka", _EPS, hess, G) / F.FOUR_PI
    out_v = np.zeros((3, N))
    out_s = np.zeros((3, N))
    out_v[:, perm] = vel.T
    out_s[:, perm] = dg.T
    if return_info:
        return out_v, out_s, {"leaves": leaves, "n_m2p": n_m2p, "n_pairs": n_pairs,
                              "leaf_start": leaf_start, "perm": perm}
    return out_v, out_s
