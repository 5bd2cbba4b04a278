"""Pins of the treecode oracle (oracle/treecode_ref.py) -- the cell-particle half of the
paper's hybrid treecode-FMM -- against what the mathematics fixes:

* theta = 0 never accepts a cell, so the traversal reduces to the direct periodic sum over the
  near 3^3 image block: equal to the C direct-sum oracle O1 (oracle.c) to rounding;
* one cell's multipole evaluated at far points (M2P) converges geometrically in p to the exact
  pair sum of that cell's particles (Eq. 5 / Eq. 8 with g = 1 far from the cores);
* at theta = 0.5 the traversal's error against O1 falls with p (PAPER.md:174's accuracy claim
  is about this convergence), at image_levels 1 and 3 (the 27^3 cube, reading R5);
* the adaptive leaves partition the particles and respect n_crit ("automatically choosing the
  number of particles per box"; reading R22).
"""
import numpy as np
import pytest

import oracle
import synthgen
from oracle import fmm_ref as F
from oracle import treecode_ref as T


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def field():
    return synthgen.clustered(300)


@pytest.mark.parametrize("lam", [0, 1])
def test_theta_zero_is_the_direct_sum(field, lam):
    f = field
    v, s = T.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 4, 4, 0.0, 8,
                      image_levels=lam)
    vr, sr = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, lam, 0)
    assert rel(v, vr) < 1e-12 and rel(s, sr) < 1e-12


def test_m2p_single_cell_converges_to_pair_sum():
    rng = np.random.default_rng(5)
    c = np.array([0.2, -0.1, 0.3])
    w = 0.5
    xs = c + (rng.random((40, 3)) - 0.5) * w
    gs = rng.standard_normal((40, 3))
    # targets at 2.5 .. 4 cell widths from the centre (a MAC ratio of 0.35 .. 0.2)
    d = rng.standard_normal((12, 3))
    d *= (rng.uniform(1.25, 2.0, 12) / np.linalg.norm(d, axis=1))[:, None]
    xt = c + d
    gt = rng.standard_normal((12, 3))
    sigma = 0.01  # g = 1 to double precision at these distances
    for scheme in (0, 1):
        u_ref, s_ref = F.pair_sum(xt, gt, xs, gs, sigma, scheme)
        errs = []
        for p in (2, 5, 8, 12):
            M = F.p2m(xs - c, gs, p)
            g, h = T.m2p(M[None], d[:, None, :], p)
            u = np.einsum("abc,kcb->ka", T._EPS, g) / F.FOUR_PI
            if scheme == 0:
                st = np.einsum("abc,kcdb,kd->ka", T._EPS, h, gt) / F.FOUR_PI
            else:
                st = np.einsum("dbc,kcab,kd->ka", T._EPS, h, gt) / F.FOUR_PI
            errs.append(max(rel(u, u_ref), rel(st, s_ref)))
        assert errs[0] > errs[1] > errs[2] > errs[3], errs
        assert errs[1] < 2e-2 and errs[3] < 1e-6, errs


@pytest.mark.parametrize("lam,bounds", [(1, (3e-5, 1e-6)), (3, (6e-5, 6e-6))])
def test_theta_half_converges_with_p(field, lam, bounds):
    f = field
    vr, sr = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, lam, 0)
    out = []
    for p in (6, 10):
        v, s = T.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 4, p, 0.5, 16,
                          image_levels=lam)
        out.append(max(rel(v, vr), rel(s, sr)))
    assert out[0] < bounds[0] and out[1] < bounds[1] and out[1] < out[0] / 4, out


def test_transpose_scheme_matches_direct(field):
    f = field
    vr, sr = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 1)
    v, s = T.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 4, 10, 0.5, 16,
                      image_levels=1, scheme=1)
    assert rel(v, vr) < 1e-6 and rel(s, sr) < 1e-6


def test_adaptive_leaves_partition(field):
    f = field
    L, ncrit = 4, 16
    keys, perm, leaf_start, rc = oracle.morton(f.pos, L, f.box_lo, f.box_len)
    assert rc == 0
    leaves = T.adaptive_leaves(leaf_start, L, ncrit)
    owner = np.full(f.pos.shape[1], -1)
    for i, (l, c) in enumerate(leaves):
        sh = 3 * (L - l)
        s, e = leaf_start[c << sh], leaf_start[(c + 1) << sh]
        assert e > s
        assert (owner[s:e] == -1).all()
        owner[s:e] = i
        assert l == L or e - s <= ncrit
        if l > 1:  # the parent was split because it held more than n_crit
            pc, sp = c >> 3, 3 * (L - l + 1)
            assert leaf_start[(pc + 1) << sp] - leaf_start[pc << sp] > ncrit
    assert (owner >= 0).all()
    levels = {l for l, _ in leaves}
    assert len(levels) >= 2  # the clustered field gives leaves at several levels
