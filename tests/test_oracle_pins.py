"""Pins for the CPU oracle (oracle/) against things other than itself.

Every check here is fixed by PAPER.md's definitions or by mathematics:
closed forms, printed example values (tests/golden), invariants, special cases,
finite differences, and an independent 30-digit mpmath brute force.  Chosen so
that a dropped term, a wrong sign or index, or a transposed operand in
oracle/oracle.c or oracle/fmm_ref.py fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synthgen
from oracle import fmm_ref as F

mpmath = pytest.importorskip("mpmath")
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _mp_kernels(r, sigma):
    """Independent 30-digit zeta, g, f and q = f'(r)/r (q by numerical differentiation)."""
    mp = mpmath.mp
    mp.dps = 30
    r = mp.mpf(r)
    s = mp.mpf(sigma)

    def g_of(x):
        rho = x / (mp.sqrt(2) * s)
        return mp.erf(rho) - mp.sqrt(4 / mp.pi) * rho * mp.exp(-rho * rho)

    def f_of(x):
        return g_of(x) / (4 * mp.pi * x ** 3)  # gamma x grad(G g), G = 1/(4 pi r) PAPER.md:84

    zeta = (2 * mp.pi * s * s) ** mp.mpf(-1.5) * mp.exp(-r * r / (2 * s * s))
    return zeta, g_of(r), f_of(r), mp.diff(f_of, r) / r


# ---------------------------------------------------------------- scalar kernels

def test_golden_spec_values():
    gold = json.load(open(os.path.join(GOLD, "kernel_values.json")))
    z0, _, _, _ = oracle.kernels(0.0, 1.0)
    assert round(z0, gold["zeta_r0_sigma1"]["digits"] + 1) == pytest.approx(
        gold["zeta_r0_sigma1"]["value"], abs=10 ** -gold["zeta_r0_sigma1"]["digits"])
    z, _, _, _ = oracle.kernels(1.0, 0.5)
    assert z == pytest.approx(gold["zeta_r1_sigma0p5"]["value"], abs=1e-4)
    _, g, _, _ = oracle.kernels(1.0, 1.0)
    assert g == pytest.approx(gold["g_r_eq_sigma"]["value"], abs=1e-4)
    # f at large r reduces to the point vortex 1/(4 pi r^3): G(1)=1/4pi
    _, _, f, _ = oracle.kernels(1.0, 0.05)
    assert f == pytest.approx(gold["greens_r1"]["value"], abs=5e-9)
    assert f == pytest.approx(1.0 / (4 * math.pi), rel=1e-14)


@pytest.mark.parametrize("r,sigma", [(0.0, 1.0), (1e-4, 1.0), (0.1, 1.0), (0.3535, 1.0),
                                     (0.3536, 1.0), (0.5, 1.0), (1.0, 1.0), (2.0, 1.0),
                                     (3.0, 0.7), (5.0, 1.0), (8.0, 1.0), (11.99, 1.0),
                                     (12.01, 1.0), (20.0, 1.0), (1.0, 0.5)])
def test_kernels_vs_mpmath(r, sigma):
    z, g, f, q = oracle.kernels(r, sigma)
    if r == 0.0:
        mp = mpmath.mp
        mp.dps = 30
        z0 = (2 * mp.pi * sigma ** 2) ** mp.mpf(-1.5)
        assert f == pytest.approx(float(z0 / 3), rel=1e-15)        # f(0) = zeta0/3
        assert q == pytest.approx(float(-z0 / (5 * sigma ** 2)), rel=1e-15)
        return
    zm, gm, fm, qm = _mp_kernels(r, sigma)
    assert z == pytest.approx(float(zm), rel=1e-13, abs=1e-30)  # r >= 12 sigma: zeta := 0
    assert f == pytest.approx(float(fm), rel=1e-13)
    assert q == pytest.approx(float(qm), rel=1e-11)
    assert g == pytest.approx(float(gm), rel=1e-13, abs=1e-16)


def test_cutoff_saturation_and_derivative():
    # g' = 4 pi r^2 zeta (Eq. 6 is the radial integral of Eq. 4)
    for r in (0.2, 0.9, 1.7, 3.3):
        h = 1e-6
        gp = (oracle.kernels(r + h, 1.0)[1] - oracle.kernels(r - h, 1.0)[1]) / (2 * h)
        assert gp == pytest.approx(4 * math.pi * r * r * oracle.kernels(r, 1.0)[0], rel=1e-7)
    assert 1.0 - oracle.kernels(8.0, 1.0)[1] < 1e-12
    assert 1.0 - oracle.kernels(5.0, 1.0)[1] == pytest.approx(1.544e-5, rel=1e-3)


# ---------------------------------------------------------------- direct sum

def _direct(pos, gam, sigma, lam, scheme=0, **kw):
    return oracle.direct(np.asarray(pos, np.float64), np.asarray(gam, np.float64), sigma,
                         -math.pi, 2 * math.pi, lam, scheme, **kw)


def test_right_hand_rule_and_sign():
    # gamma = z at origin, target (1,0,0): u = (0, +1/4pi, 0) (physical sign, reading R1)
    pos = np.array([[0.0, 1.0], [0.0, 0.0], [0.0, 0.0]])
    gam = np.array([[0.0, 0.0], [0.0, 0.0], [1.0, 0.0]])
    v, s = _direct(pos, gam, 0.05, 0)
    assert v[:, 1] == pytest.approx([0.0, 1.0 / (4 * math.pi), 0.0], abs=1e-15)
    assert np.all(v[:, 0] == 0.0)  # the target particle has zero strength


def test_single_blob_closed_form_and_curl_of_streamfunction():
    # u(x) = g(r)/(4 pi r^3) gamma x (x - x0); also u = curl psi, psi = gamma erf(rho)/(4 pi r)
    rng = np.random.default_rng(5)
    x0 = np.array([0.1, -0.2, 0.3])
    g0 = np.array([0.3, -0.5, 0.8])
    sigma = 0.4
    probes = x0[:, None] + rng.normal(size=(3, 12)) * 0.5
    v, _ = _direct(x0[:, None], g0[:, None], sigma, 0, probe_pos=probes,
                   probe_gamma=np.zeros_like(probes))
    for t in range(probes.shape[1]):
        d = probes[:, t] - x0
        r = np.linalg.norm(d)
        rho = r / (math.sqrt(2) * sigma)
        g = math.erf(rho) - 2 / math.sqrt(math.pi) * rho * math.exp(-rho * rho)
        assert v[:, t] == pytest.approx(g / (4 * math.pi * r ** 3) * np.cross(g0, d), rel=1e-12)

        def psi(x):
            rr = np.linalg.norm(x - x0)
            return g0 * math.erf(rr / (math.sqrt(2) * sigma)) / (4 * math.pi * rr)

        h = 1e-5
        J = np.zeros((3, 3))  # J[c, b] = d psi_c / d x_b
        for b in range(3):
            e = np.zeros(3)
            e[b] = h
            J[:, b] = (psi(probes[:, t] + e) - psi(probes[:, t] - e)) / (2 * h)
        curl = np.array([J[2, 1] - J[1, 2], J[0, 2] - J[2, 0], J[1, 0] - J[0, 1]])
        assert v[:, t] == pytest.approx(curl, rel=1e-6, abs=1e-9)


@pytest.mark.parametrize("lam", [0, 1])
def test_antisymmetry_two_particles(lam):
    pos = np.array([[0.3, -0.4], [0.1, 0.5], [-0.2, 0.25]])
    gam = np.array([[0.2, 0.2], [-0.1, -0.1], [0.7, 0.7]])
    v, _ = _direct(pos, gam, 0.3, lam)
    assert v[:, 0] == pytest.approx(-v[:, 1], rel=1e-12, abs=1e-15)


def test_zero_net_momentum_equal_strengths():
    rng = np.random.default_rng(7)
    pos = rng.uniform(-math.pi, math.pi, (3, 40))
    gam = np.tile(np.array([[0.3], [-0.2], [0.5]]), (1, 40))
    v, _ = _direct(pos, gam, 0.35, 1)
    scale = np.abs(v).sum()
    assert np.abs(v.sum(axis=1)).max() < 1e-13 * scale


@pytest.mark.parametrize("lam", [1, 2])
def test_single_particle_in_periodic_box_is_at_rest(lam):
    pos = np.array([[0.7], [-1.1], [2.0]])
    gam = np.array([[0.4], [0.9], [-0.3]])
    v, s = _direct(pos, gam, 0.3, lam)
    assert np.abs(v).max() < 1e-14 and np.abs(s).max() < 1e-14


def test_divergence_free_and_stretching_by_finite_differences():
    rng = np.random.default_rng(11)
    pos = rng.uniform(-math.pi, math.pi, (3, 25))
    gam = rng.normal(size=(3, 25))
    sigma = 0.5
    probes = rng.uniform(-2, 2, (3, 4))
    pg = rng.normal(size=(3, 4))
    _, s_cl = _direct(pos, gam, sigma, 1, 0, probe_pos=probes, probe_gamma=pg)
    _, s_tr = _direct(pos, gam, sigma, 1, 1, probe_pos=probes, probe_gamma=pg)
    h = 1e-5
    for t in range(4):
        J = np.zeros((3, 3))  # J[a, b] = d u_a / d x_b
        for b in range(3):
            pp = probes[:, t:t + 1].copy()
            pm = pp.copy()
            pp[b] += h
            pm[b] -= h
            vp, _ = _direct(pos, gam, sigma, 1, probe_pos=pp, probe_gamma=pg[:, t:t + 1])
            vm, _ = _direct(pos, gam, sigma, 1, probe_pos=pm, probe_gamma=pg[:, t:t + 1])
            J[:, b] = (vp[:, 0] - vm[:, 0]) / (2 * h)
        scale = np.abs(J).max()
        assert abs(np.trace(J)) < 1e-7 * scale                     # div u = 0
        assert s_cl[:, t] == pytest.approx(J @ pg[:, t], rel=1e-6, abs=1e-8 * scale)  # (g.grad)u
        assert s_tr[:, t] == pytest.approx(J.T @ pg[:, t], rel=1e-6, abs=1e-8 * scale)


def test_transpose_scheme_sums_to_zero_and_bilinearity():
    rng = np.random.default_rng(13)
    pos = rng.uniform(-math.pi, math.pi, (3, 30))
    gam = rng.normal(size=(3, 30))
    v, s_tr = _direct(pos, gam, 0.4, 1, 1)
    assert np.abs(s_tr.sum(axis=1)).max() < 1e-12 * np.abs(s_tr).sum()
    v2, s2 = _direct(pos, 2.5 * gam, 0.4, 1, 0)
    _, s1 = _direct(pos, gam, 0.4, 1, 0)
    assert v2 == pytest.approx(2.5 * v, rel=1e-13)
    assert s2 == pytest.approx(6.25 * s1, rel=1e-12)


def test_taylor_green_closed_form_image_sum():
    """Lattice TG (c1): u_i = e^{-3 s^2/2} u_TG(x_i), sdot_i = h^3 e^{-3 s^2/2} (w.grad)u_TG,
    up to lattice aliasing e^{-2 pi^2} ~ 2.7e-9 and float32 input rounding; the cube
    surface term vanishes by the TG symmetry."""
    f = synthgen.make("c1")
    tg = np.array([0, 1234, 4095, 2000])
    v, s = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 3, 0, targets=tg)
    x, y, z = (f.pos[i, tg].astype(np.float64) for i in range(3))
    damp = math.exp(-1.5 * f.sigma ** 2)
    h = f.box_len / f.n
    u_tg = np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z),
                     0 * x]) * damp
    s_tg = np.stack([-0.25 * np.sin(2 * y) * np.sin(2 * z), 0.25 * np.sin(2 * x) * np.sin(2 * z),
                     0 * x]) * damp * h ** 3
    assert np.abs(v - u_tg).max() < 2e-6 * np.abs(u_tg).max()
    assert np.abs(s - s_tg).max() < 2e-6 * np.abs(s_tg).max()


def test_tiny_brute_force_mpmath():
    """Independent 30-digit brute force (N=3, 27 images): velocity from Eq. (5), stretching
    as (gamma_i . grad) u by mpmath differentiation of the velocity field (Eq. 8, classical)."""
    mp = mpmath.mp
    mp.dps = 30
    rng = np.random.default_rng(17)
    pos = rng.uniform(-math.pi, math.pi, (3, 3))
    gam = rng.normal(size=(3, 3))
    sigma = 0.9
    L = 2 * mp.pi
    v, s = _direct(pos, gam, sigma, 1)

    def vel_at(xt, exclude=None):
        u = [mp.mpf(0)] * 3
        for j in range(3):
            for nx in (-1, 0, 1):
                for ny in (-1, 0, 1):
                    for nz in (-1, 0, 1):
                        d = [xt[0] - mp.mpf(pos[0, j]) - nx * L, xt[1] - mp.mpf(pos[1, j]) - ny * L,
                             xt[2] - mp.mpf(pos[2, j]) - nz * L]
                        r = mp.sqrt(d[0] ** 2 + d[1] ** 2 + d[2] ** 2)
                        if r == 0:
                            continue
                        rho = r / (mp.sqrt(2) * sigma)
                        g = mp.erf(rho) - mp.sqrt(4 / mp.pi) * rho * mp.exp(-rho ** 2)
                        f = g / (4 * mp.pi * r ** 3)
                        gj = [mp.mpf(gam[k, j]) for k in range(3)]
                        c = [gj[1] * d[2] - gj[2] * d[1], gj[2] * d[0] - gj[0] * d[2],
                             gj[0] * d[1] - gj[1] * d[0]]
                        u = [u[k] + f * c[k] for k in range(3)]
        return u

    for i in range(3):
        xi = [mp.mpf(pos[k, i]) for k in range(3)]
        gi = [mp.mpf(gam[k, i]) for k in range(3)]
        u = vel_at(xi)
        for k in range(3):
            assert float(u[k]) == pytest.approx(v[k, i], rel=1e-12, abs=1e-15)
        # directional derivative along gamma_i (the self term is identically zero, smooth)
        for k in range(3):
            fk = lambda t: vel_at([xi[a] + t * gi[a] for a in range(3)])[k]
            sd = mp.diff(fk, 0)
            assert float(sd) == pytest.approx(s[k, i], rel=1e-9, abs=1e-13)


# ---------------------------------------------------------------- Morton tree

def test_morton_hand_example():
    # depth 1, box [-pi, pi): octant (ix,iy,iz) -> key ix | iy<<1 | iz<<2
    lo, ln = synthgen.BOX_LO, synthgen.BOX_LEN
    pos = np.array([[1.0, -1.0, 1.0, -1.0], [1.0, 1.0, -1.0, -1.0], [-1.0, 1.0, 1.0, -1.0]],
                   np.float32)
    keys, perm, ls, rc = oracle.morton(pos, 1, lo, ln)
    assert rc == 0
    assert list(keys) == [0, 3, 5, 6]
    assert list(perm) == [3, 0, 2, 1]
    assert list(ls) == [0, 1, 1, 1, 2, 2, 3, 4, 4]


def test_morton_depth2_bits_and_stability():
    lo, ln = synthgen.BOX_LO, synthgen.BOX_LEN
    h = float(ln) / 4
    # cell (ix,iy,iz) = (3,1,2): key bits b0: x0=1,y0=1,z0=0 ; b1: x1=1,y1=0,z1=1
    c = np.array([3, 1, 2])
    x = (float(lo) + (c + 0.5) * h).astype(np.float32)
    pos = np.stack([x, x, x], axis=1).astype(np.float32)  # three identical particles
    keys, perm, ls, rc = oracle.morton(pos, 2, lo, ln)
    expect = (1 << 0) | (1 << 1) | (0 << 2) | (1 << 3) | (0 << 4) | (1 << 5)
    assert list(keys) == [expect] * 3 and list(perm) == [0, 1, 2]  # ties keep input order
    assert ls[expect] == 0 and ls[expect + 1] == 3 and ls[-1] == 3


def test_morton_random_vs_python_sort_and_edges():
    rng = np.random.default_rng(21)
    lo, ln = synthgen.BOX_LO, synthgen.BOX_LEN
    pos = rng.uniform(float(lo), float(lo + ln), (3, 5000)).astype(np.float32)
    pos[:, :10] = lo  # exact lower faces
    pos[:, 10:20] = np.nextafter(np.float32(lo + ln), np.float32(0))  # just below upper face
    depth = 3
    keys, perm, ls, rc = oracle.morton(pos, depth, lo, ln)
    assert rc == 0
    inv = np.float32((1 << depth) / float(ln))
    q = np.floor((pos - lo) * inv).astype(np.int64).clip(0, (1 << depth) - 1)
    ref = np.zeros(pos.shape[1], np.int64)
    for b in range(depth):
        for a in range(3):
            ref |= ((q[a] >> b) & 1) << (3 * b + a)
    order = sorted(range(pos.shape[1]), key=lambda i: (ref[i], i))
    assert list(perm) == order and list(keys) == [ref[i] for i in order]
    counts = np.bincount(ref, minlength=8 ** depth)
    assert np.array_equal(np.diff(ls), counts) and ls[0] == 0 and ls[-1] == pos.shape[1]
    assert set(perm.tolist()) == set(range(pos.shape[1]))


def test_morton_flags_out_of_box():
    lo, ln = synthgen.BOX_LO, synthgen.BOX_LEN
    pos = np.zeros((3, 4), np.float32)
    pos[0, 2] = np.float32(lo + ln)  # upper face is outside the half-open box
    assert oracle.morton(pos, 2, lo, ln)[3] == -2
    pos[0, 2] = np.nan
    assert oracle.morton(pos, 2, lo, ln)[3] == -2


def test_lattice_leaves_hold_equal_counts():
    f = synthgen.make("c1")
    keys, perm, ls, rc = oracle.morton(f.pos, 2, f.box_lo, f.box_len)
    assert rc == 0 and np.all(np.diff(ls) == 64)


# ---------------------------------------------------------------- FMM oracle (fmm_ref)

def test_expansion_identities():
    rng = np.random.default_rng(0)
    x = rng.normal(size=3) * 3
    y = rng.normal(size=3) * 0.3
    R = F.solid_R(y[None], 30)[0]
    I = F.solid_I(x[None], 30)[0]
    # addition theorem, Eq. (10): 1/|x-y| = sum conj(R_n^m(y)) I_n^m(x)
    assert np.real((np.conj(R) * I).sum()) == pytest.approx(1 / np.linalg.norm(x - y), rel=1e-14)
    # R_1: z, -(x+iy)/2
    r1 = F.solid_R(np.array([[0.3, -0.7, 1.1]]), 1)[0]
    assert r1[F.kidx(1, 0)] == pytest.approx(1.1)
    assert r1[F.kidx(1, 1)] == pytest.approx(-(0.3 - 0.7j) / 2)
    assert r1[F.kidx(1, -1)] == pytest.approx((0.3 + 0.7j) / 2)
    p = 12
    src = rng.normal(size=(15, 3)) * 0.25
    q = rng.normal(size=(15, 3))
    M = F.p2m(src, q, p)
    xt = np.array([2.0, 1.0, -1.5])
    direct = (q / np.linalg.norm(xt - src, axis=1)[:, None]).sum(0)
    assert np.real(M @ F.solid_I(xt[None], p)[0]) == pytest.approx(direct, rel=1e-7)
    # M2L then L2L vs direct potential; M2M vs P2M about the other centre
    D = np.array([3.0, -2.0, 2.5])
    L = M @ F.m2l_matrix(D, p).T
    z = np.array([0.1, -0.15, 0.2])
    direct = (q / np.linalg.norm(D + z - src, axis=1)[:, None]).sum(0)
    assert np.real(L @ F.solid_R(z[None], p)[0]) == pytest.approx(direct, rel=1e-8)
    d = np.array([0.05, 0.02, -0.04])
    L2 = L @ F.l2l_matrix(d, p).T
    assert np.real(L2 @ F.solid_R((z - d)[None], p)[0]) == pytest.approx(direct, rel=1e-8)
    dm = np.array([0.3, -0.2, 0.1])
    assert M @ F.m2m_matrix(dm, p).T == pytest.approx(F.p2m(src + dm, q, p), abs=1e-12)
    # zero-offset M2M / L2L are the identity
    assert np.allclose(F.m2m_matrix(np.zeros(3), 4), np.eye(25))
    assert np.allclose(F.l2l_matrix(np.zeros(3), 4), np.eye(25))
    # gradient / Hessian stencils vs finite differences of the evaluated local expansion
    g, h = F.l2p(L, z[None], p)
    ev = lambda zz: np.real(L @ F.solid_R(zz[None], p)[0])
    e = 1e-5
    for a in range(3):
        dz = np.zeros(3)
        dz[a] = e
        assert g[0, :, a] == pytest.approx((ev(z + dz) - ev(z - dz)) / (2 * e), rel=1e-7)
        gp, _ = F.l2p(L, (z + dz)[None], p)
        gm, _ = F.l2p(L, (z - dz)[None], p)
        assert h[0, :, a, :] == pytest.approx((gp - gm)[0] / (2 * e), rel=1e-6, abs=1e-9)


def test_periodic_operator_equals_explicit_image_sum():
    """3x supercell rings == explicit M2L from every image box in the cube minus the near 3^3."""
    rng = np.random.default_rng(3)
    p = 6
    src = rng.uniform(-1, 1, (10, 3)) * 0.5
    q = rng.normal(size=(10, 3))
    q -= q.mean(0)
    M0 = F.p2m(src, q, p)
    Lr = F.periodic_far(M0, 2 * math.pi, 2, p)
    Le = np.zeros_like(Lr)
    for a in range(-4, 5):
        for b in range(-4, 5):
            for c in range(-4, 5):
                if max(abs(a), abs(b), abs(c)) > 1:
                    Le += M0 @ F.m2l_matrix(-np.array([a, b, c]) * 2 * math.pi, p).T
    assert Lr == pytest.approx(Le, rel=1e-12, abs=1e-14)


def test_fmm_oracle_converges_to_direct_sum():
    """FMM (fp64) vs direct sum on an isotropic 16^3 field: error decreases with p and is
    at the paper's accuracy level ('4 significant digits' at p = 10)."""
    f = synthgen.isotropic(16)
    tg = synthgen.sample_targets(16 ** 3, 48, n_lattice=16)
    v, s = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 0, targets=tg)
    errs = []
    for p in (2, 4, 6):
        vf, sf = F.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 2, p, 1)
        errs.append((np.linalg.norm(vf[:, tg] - v) / np.linalg.norm(v),
                     np.linalg.norm(sf[:, tg] - s) / np.linalg.norm(s)))
    assert errs[0][0] > errs[1][0] > errs[2][0] and errs[0][1] > errs[1][1] > errs[2][1]
    assert errs[2][0] < 5e-3 and errs[2][1] < 2e-2


def test_fmm_oracle_near_only_depth1_equals_direct():
    """depth 1 in free space (lambda = 0): all 8 octants are mutual neighbours, nothing is
    well separated, so every interaction is P2P and the FMM equals the direct sum."""
    f = synthgen.taylor_green(8)
    vf, sf = F.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 2, 0)
    v, s = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 0, 0)
    assert np.abs(vf - v).max() < 1e-13 * np.abs(v).max()
    assert np.abs(sf - s).max() < 1e-12 * np.abs(s).max()


@pytest.mark.parametrize("lam,scheme", [(0, 0), (1, 1), (2, 0)])
def test_batched_oracle_is_bitwise_the_plain_one(lam, scheme):
    """vfmm_oracle_eval_batched (loop nest reordered for the tests/golden runs) performs the
    same floating-point operations in the same order per target as vfmm_oracle_eval: equal
    bit for bit, including close pairs (series branch), coincident distinct particles (r = 0
    limits), the closed form and the far branch, a ragged last batch, and probe targets."""
    rng = np.random.default_rng(23)
    f = synthgen.jitter(synthgen.make("c1"), 0.75, seed=4)
    pos, gam = f.pos.copy(), f.gamma.copy()
    pos[:, 5] = pos[:, 9]  # a distinct coincident pair
    tg = np.sort(rng.choice(4096, 37, replace=False))
    tg[0], tg[1] = 5, 9
    for native in (False, True):
        a = oracle.direct(pos, gam, f.sigma, f.box_lo, f.box_len, lam, scheme, targets=tg)
        b = oracle.direct(pos, gam, f.sigma, f.box_lo, f.box_len, lam, scheme, targets=tg,
                          batched=True, native=native)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    pp = rng.uniform(-3, 3, (3, 5))
    pg = rng.normal(size=(3, 5))
    a = oracle.direct(pos, gam, f.sigma, f.box_lo, f.box_len, lam, scheme, probe_pos=pp,
                      probe_gamma=pg)
    b = oracle.direct(pos, gam, f.sigma, f.box_lo, f.box_len, lam, scheme, probe_pos=pp,
                      probe_gamma=pg, batched=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.slow
def test_fmm_oracle_supercell_rings_vs_direct_sum_at_27_cubed():
    """fmm_ref.periodic_far at image_levels = 3 (ring k = 0 of 702 boxes and ring k = 1 of 702
    supercells of 27 boxes, PAPER.md:144, :164 '3^3 x 3^3 x 3^3 - 1' images) against the
    direct sum O1 over the same 27^3 cube, on an isotropic 8^3 field where the outer shell
    matters: O1 at lambda = 2 differs from lambda = 3 by > 1e-3, so a wrong or missing ring
    fails.  p = 12, depth 1 (all near-field interactions exact)."""
    f = synthgen.isotropic(8, seed=5)
    v3, s3 = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 3, 0, batched=True)
    v2, s2 = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 2, 0, batched=True)
    shell = np.linalg.norm(v2 - v3) / np.linalg.norm(v3)
    assert shell > 1e-3, shell
    vf, sf = F.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 12, 3)
    eu = np.linalg.norm(vf - v3) / np.linalg.norm(v3)
    es = np.linalg.norm(sf - s3) / np.linalg.norm(s3)
    assert eu < 2e-5 and es < 1e-4, (eu, es)
    # the same FMM at lambda = 2 is far from the lambda = 3 sum (the ring is what matters)
    vf2, _ = F.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 12, 2)
    assert np.linalg.norm(vf2 - v3) / np.linalg.norm(v3) > 1e-3


# ---------------------------------------------------------------- time stepping (NEXT-1)

def test_euler_step_taylor_green_closed_form():
    """One forward-Euler step (PAPER.md:91 Eq. 7, :100 Eq. 8, :107 Eq. 9, :114) of the lattice
    Taylor-Green field: the displacement is dt e^{-3 s^2/2} u_TG(x_i) and the strength change
    dt h^3 e^{-3 s^2/2} (w.grad)u_TG (the closed forms of test_taylor_green_closed_form_image_sum,
    SURVEY App. B), the core grows as sigma^2 + 2 nu dt."""
    from oracle.euler import euler_step

    f = synthgen.make("c1")
    dt, nu = 0.05, 0.01
    x1, g1, s1, u, dg = euler_step(f.pos, f.gamma, f.sigma, nu, dt, f.box_lo, f.box_len, 2)
    x, y, z = (f.pos[i].astype(np.float64) for i in range(3))
    damp = math.exp(-1.5 * f.sigma ** 2)
    h = f.box_len / f.n
    u_tg = np.stack([np.sin(x) * np.cos(y) * np.cos(z), -np.cos(x) * np.sin(y) * np.cos(z),
                     0 * x]) * damp
    s_tg = np.stack([-0.25 * np.sin(2 * y) * np.sin(2 * z), 0.25 * np.sin(2 * x) * np.sin(2 * z),
                     0 * x]) * damp * h ** 3
    disp = x1 - f.pos.astype(np.float64)
    disp -= f.box_len * np.round(disp / f.box_len)  # undo the wrap
    # lambda = 2 instead of 3: the outer shell changes the sum by ~2e-5 relative
    assert np.abs(disp - dt * u_tg).max() < 5e-5 * dt * np.abs(u_tg).max()
    assert np.abs((g1 - f.gamma) - dt * s_tg).max() < 5e-5 * dt * np.abs(s_tg).max()
    assert s1 == pytest.approx(math.sqrt(f.sigma ** 2 + 2 * nu * dt), rel=1e-15)
    assert np.all(x1 >= f.box_lo) and np.all(x1 < f.box_lo + f.box_len)


def test_euler_step_lone_particle_and_zero_dt():
    """A lone particle in the periodic box is at rest with constant strength (its images
    cancel); dt = 0 is the identity; free space: no wrap."""
    from oracle.euler import euler_step

    pos = np.array([[0.7], [-1.1], [2.0]])
    gam = np.array([[0.4], [0.9], [-0.3]])
    x1, g1, s1, _, _ = euler_step(pos, gam, 0.3, 0.02, 0.1, -math.pi, 2 * math.pi, 2)
    assert np.abs(x1 - pos).max() < 1e-14 and np.abs(g1 - gam).max() < 1e-14
    assert s1 == pytest.approx(math.sqrt(0.09 + 0.004))
    rng = np.random.default_rng(3)
    p = rng.uniform(-3, 3, (3, 20))
    g = rng.normal(size=(3, 20))
    x1, g1, s1, _, _ = euler_step(p, g, 0.4, 0.0, 0.0, -math.pi, 2 * math.pi, 1)
    assert np.abs(x1 - p).max() < 1e-15 and np.array_equal(g1, g) and s1 == 0.4
    # free space, two particles: the step moves each by dt u (antisymmetric pair, Eq. 7)
    p2 = np.array([[0.3, -0.4], [0.1, 0.5], [-0.2, 0.25]])
    g2 = np.array([[0.2, 0.2], [-0.1, -0.1], [0.7, 0.7]])
    x1, _, _, u, _ = euler_step(p2, g2, 0.3, 0.0, 0.2, -math.pi, 2 * math.pi, 0)
    assert np.allclose(x1 - p2, 0.2 * u, rtol=0, atol=1e-15)
    assert np.allclose(u[:, 0], -u[:, 1], rtol=1e-12)


# ---------------------------------------------------------------- RBF reinitialization (NEXT-2)

def test_rbf_oracle_fourier_mode_closed_form():
    """On the cell-centre lattice with sigma = h a Fourier mode is an eigenvector
    of the Gaussian sum (Eq. 3): sum_j h^3 sin(k.x_j) zeta(x_i - x_j) = e^{-|k|^2 s^2/2} sin(k.x_i)
    up to lattice aliasing, here e^{-|k - (2 pi/h) e_x|^2 s^2 / 2} = 3e-8 (Poisson summation;
    16^3, k = (1, 1, 0)).  So the RBF solve of omega = sin(k.x) is
    gamma = h^3 e^{|k|^2 s^2/2} sin(k.x)."""
    from oracle import rbf

    n = 16
    L = 2 * math.pi
    h = L / n
    c = -math.pi + h * (np.arange(n) + 0.5)  # exact float64 lattice (Poisson summation)
    zz, yy, xx = np.meshgrid(c, c, c, indexing="ij")
    x = np.stack([xx.ravel(), yy.ravel(), zz.ravel()])
    s = h
    f = synthgen.Field(x, x, s, -math.pi, L, n, "lattice")
    k = np.array([1.0, 1.0, 0.0])
    mode = np.sin(k @ x)
    w = np.stack([mode, 0.5 * mode, -mode]) * h ** 3
    om = rbf.gaussian_sum(x, x, w, s, f.box_len)
    damp = math.exp(-0.5 * (k @ k) * s * s)
    assert np.abs(om - damp * w / h ** 3).max() < 2e-7 * np.abs(w / h ** 3).max()
    A = rbf.rbf_matrix(x, s, f.box_len)
    g2 = np.linalg.solve(A, mode)
    assert np.abs(g2 - h ** 3 * mode / damp).max() < 5e-6 * np.abs(h ** 3 * mode / damp).max()
    g, _ = rbf.reinit(x, w, s, x, s, f.box_len)
    assert np.abs(g - w).max() < 1e-9 * np.abs(w).max()   # the same particles back


def test_rbf_oracle_single_particle_and_partition_of_unity():
    """A particle already on a lattice point with the new core size is its own interpolant;
    the lattice quadrature of one Gaussian sums to 1 (Eq. 4 integrates to 1)."""
    from oracle import rbf

    f = synthgen.taylor_green(8)
    x = f.pos.astype(np.float64)
    h = f.box_len / 8
    p = 77
    g_old = np.array([[0.3], [-0.2], [0.9]])
    g, _ = rbf.reinit(x[:, p:p + 1], g_old, f.sigma, x, f.sigma, f.box_len)
    want = np.zeros_like(g)
    want[:, p] = g_old[:, 0]
    assert np.abs(g - want).max() < 1e-9
    one = rbf.gaussian_sum(np.array([[0.123], [-0.4], [1.0]]), x, np.ones_like(x) * h ** 3,
                           f.sigma, f.box_len)
    assert one == pytest.approx(np.ones((3, 1)), rel=1e-8)


# ---------------------------------------------------------------- per-particle core radius (NEXT-4)

def test_per_source_sigma_oracle():
    """Eq. (6) as written carries the source's sigma_j: a uniform sigma array is
    the scalar sum bit for bit; with different sigma_j each source contributes its own closed
    form g(r/sigma_j) gamma_j x d / (4 pi r^3); the field stays divergence-free and the
    stretching stays (gamma_i . grad) u by finite differences."""
    f = synthgen.jitter(synthgen.make("c1"))
    tg = np.arange(0, 4096, 97)
    a = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 0, targets=tg)
    b = oracle.direct(f.pos, f.gamma, np.full(4096, f.sigma), f.box_lo, f.box_len, 1, 0,
                      targets=tg)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    rng = np.random.default_rng(8)
    xs = rng.uniform(-1, 1, (3, 3))
    gs = rng.normal(size=(3, 3))
    sig = np.array([0.2, 0.45, 0.8])
    probes = rng.uniform(-1.5, 1.5, (3, 6))
    v, _ = _direct(xs, gs, sig, 0, probe_pos=probes, probe_gamma=np.zeros_like(probes))
    for t in range(6):
        want = np.zeros(3)
        for j in range(3):
            d = probes[:, t] - xs[:, j]
            r = np.linalg.norm(d)
            rho = r / (math.sqrt(2) * sig[j])
            g = math.erf(rho) - 2 / math.sqrt(math.pi) * rho * math.exp(-rho * rho)
            want += g / (4 * math.pi * r ** 3) * np.cross(gs[:, j], d)
        assert v[:, t] == pytest.approx(want, rel=1e-12)
    pg = rng.normal(size=(3, 2))
    _, s_cl = _direct(xs, gs, sig, 0, 0, probe_pos=probes[:, :2], probe_gamma=pg)
    h = 1e-5
    for t in range(2):
        J = np.zeros((3, 3))
        for bb in range(3):
            pp = probes[:, t:t + 1].copy()
            pm = pp.copy()
            pp[bb] += h
            pm[bb] -= h
            vp, _ = _direct(xs, gs, sig, 0, probe_pos=pp, probe_gamma=pg[:, t:t + 1])
            vm, _ = _direct(xs, gs, sig, 0, probe_pos=pm, probe_gamma=pg[:, t:t + 1])
            J[:, bb] = (vp[:, 0] - vm[:, 0]) / (2 * h)
        sc = np.abs(J).max()
        assert abs(np.trace(J)) < 1e-7 * sc
        assert s_cl[:, t] == pytest.approx(J @ pg[:, t], rel=1e-6, abs=1e-8 * sc)
