"""TEST INFRASTRUCTURE ONLY -- step-by-step float64 FMM oracle (numpy).

Follows the paper's FMM for the vortex kernels, section 3.1:
  * Eq. (10): multipole expansion, M_j = rho^n Y_n^{-m}  -> ``p2m``
  * Eq. (11): local expansion,    L_j = rho^{-n-1} Y_n^{-m}
  * operators of Cheng et al.: ``m2m``, ``m2l``, ``l2l``
  * Eqs. (12)-(13): far velocity {sum gamma_j M_j} x grad S_i
    -> u_far = (1/4pi) curl(phi), phi_c = sum_j gamma_{j,c}/|x - x_j|       ``l2p``
  * Eqs. (14)-(15) (garbled; reading R10): far stretching
    (gamma_i . grad)(curl phi)/4pi from the Hessian of the local expansions ``l2p``
  * far field drops the cutoff g (g ~ 1)
  * near field "by solving Eq. (5) exactly" -> ``p2p``; periodic images
    "via multipole expansions" -> ``periodic_far`` (3x supercell rings, reading R5)
Uniform octree of depth L, ws = 1 (27 near leaves, 189-cell interaction lists;
reading R9), expansion order p = highest degree (reading R6).

Solid harmonics, complex, for m >= 0:
  R_n^m(x) = r^n P_n^m(cos t) e^{i m phi} / (n+m)!        (P_n^m WITH Condon-Shortley phase)
  I_n^m(x) = (n-m)! P_n^m(cos t) e^{i m phi} / r^{n+1}
  R_n^{-m} = (-1)^m conj(R_n^m),  I_n^{-m} = (-1)^m conj(I_n^m)
so that 1/|x - y| = sum_{n,m} conj(R_n^m(y)) I_n^m(x), |y| < |x|  (Eq. 10 with
Y_n^m normalised as in Cheng et al.).  Evaluated here straight from scipy's
associated Legendre functions -- no recurrences shared with the CUDA side.

Coefficients are complex arrays indexed k(n, m) = n*n + n + m, |m| <= n <= p.
Everything is float64/complex128.  No blocking or fusion beyond matrix products.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erf, lpmv

from . import morton as _morton

FOUR_PI = 4.0 * math.pi


def ncoef(p: int) -> int:
    return (p + 1) * (p + 1)


def kidx(n: int, m: int) -> int:
    return n * n + n + m


# ---------------------------------------------------------------------------
# solid harmonics
# ---------------------------------------------------------------------------

def _sph(x):
    x = np.atleast_2d(np.asarray(x, np.float64))
    r = np.sqrt((x * x).sum(axis=1))
    with np.errstate(invalid="ignore", divide="ignore"):
        ct = np.where(r > 0, x[:, 2] / np.where(r > 0, r, 1.0), 1.0)
    ct = np.clip(ct, -1.0, 1.0)
    ph = np.arctan2(x[:, 1], x[:, 0])
    return r, ct, ph


def solid_R(x, p: int):
    """Regular solid harmonics R_n^m(x), all |m| <= n <= p; shape (K, (p+1)^2)."""
    r, ct, ph = _sph(x)
    out = np.zeros((r.shape[0], ncoef(p)), np.complex128)
    for n in range(p + 1):
        rn = r ** n
        for m in range(0, n + 1):
            v = rn * lpmv(m, n, ct) * np.exp(1j * m * ph) / math.factorial(n + m)
            out[:, kidx(n, m)] = v
            if m > 0:
                out[:, kidx(n, -m)] = (-1) ** m * np.conj(v)
    return out


def solid_I(x, p: int):
    """Irregular solid harmonics I_n^m(x), all |m| <= n <= p; shape (K, (p+1)^2)."""
    r, ct, ph = _sph(x)
    out = np.zeros((r.shape[0], ncoef(p)), np.complex128)
    for n in range(p + 1):
        rn = r ** (-(n + 1))
        for m in range(0, n + 1):
            v = math.factorial(n - m) * lpmv(m, n, ct) * np.exp(1j * m * ph) * rn
            out[:, kidx(n, m)] = v
            if m > 0:
                out[:, kidx(n, -m)] = (-1) ** m * np.conj(v)
    return out


# ---------------------------------------------------------------------------
# translation operators as (nc x nc) matrices acting on coefficient vectors
# ---------------------------------------------------------------------------

def m2m_matrix(d, p: int):
    """Multipole about c' -> multipole about c, d = c' - c:
    M_n^m(c) = sum_{k,l} conj(R_k^l(d)) M_{n-k}^{m-l}(c')."""
    R = solid_R(np.asarray(d, np.float64)[None, :], p)[0]
    A = np.zeros((ncoef(p), ncoef(p)), np.complex128)
    for n in range(p + 1):
        for m in range(-n, n + 1):
            for k in range(n + 1):
                for l in range(-k, k + 1):
                    nn, mm = n - k, m - l
                    if abs(mm) <= nn:
                        A[kidx(n, m), kidx(nn, mm)] += np.conj(R[kidx(k, l)])
    return A


def m2l_matrix(D, p: int):
    """Multipole about c_s -> local about c_t, D = c_t - c_s:
    L_n^m = sum_{k,l} (-1)^{n+m} I_{n+k}^{l-m}(D) M_k^l."""
    I = solid_I(np.asarray(D, np.float64)[None, :], 2 * p)[0]
    A = np.zeros((ncoef(p), ncoef(p)), np.complex128)
    for n in range(p + 1):
        for m in range(-n, n + 1):
            s = (-1) ** ((n + m) & 1)
            for k in range(p + 1):
                for l in range(-k, k + 1):
                    A[kidx(n, m), kidx(k, l)] = s * I[kidx(n + k, l - m)]
    return A


def l2l_matrix(d, p: int):
    """Local about c -> local about c', d = c' - c:
    L_n^m(c') = sum_{k>=n, l} L_k^l(c) R_{k-n}^{l-m}(d)."""
    R = solid_R(np.asarray(d, np.float64)[None, :], p)[0]
    A = np.zeros((ncoef(p), ncoef(p)), np.complex128)
    for n in range(p + 1):
        for m in range(-n, n + 1):
            for k in range(n, p + 1):
                for l in range(-k, k + 1):
                    j, s = k - n, l - m
                    if abs(s) <= j:
                        A[kidx(n, m), kidx(k, l)] += R[kidx(j, s)]
    return A


def p2m(rel, gam, p: int):
    """Eq. (10): M_n^m[c] = sum_j gamma_{j,c} conj(R_n^m(x_j - center)); rel (K,3), gam (K,3)."""
    R = np.conj(solid_R(rel, p))  # (K, nc)
    return gam.T.astype(np.complex128) @ R  # (3, nc)


def deriv_stencil(V, axis: int, p: int):
    """Given V[n,m] = R_n^m(z) (or any array obeying the same rules), return W with
    W[n,m] = d/dx_axis R_n^m:
      d_z R_n^m = R_{n-1}^m
      d_x R_n^m = -1/2 R_{n-1}^{m-1} + 1/2 R_{n-1}^{m+1}
      d_y R_n^m = -i/2 R_{n-1}^{m-1} - i/2 R_{n-1}^{m+1}
    (from R_n^m(x+y) = sum R_k^l(y) R_{n-k}^{m-l}(x) at first order in y)."""
    W = np.zeros_like(V)
    for n in range(1, p + 1):
        for m in range(-n, n + 1):
            acc = 0
            if axis == 2:
                if abs(m) <= n - 1:
                    acc = V[..., kidx(n - 1, m)]
            else:
                a = V[..., kidx(n - 1, m - 1)] if abs(m - 1) <= n - 1 else 0
                b = V[..., kidx(n - 1, m + 1)] if abs(m + 1) <= n - 1 else 0
                acc = (-0.5 * a + 0.5 * b) if axis == 0 else (-0.5j * a - 0.5j * b)
            W[..., kidx(n, m)] = acc
    return W


def l2p(L, rel, p: int):
    """Gradient (3 comps x 3) and Hessian (3 comps x 3 x 3) of phi_c(x) = sum L_c[n,m] R_n^m(x - c).
    L: (3, nc) complex; rel: (K,3).  Returns grad (K,3c,3a) and hess (K,3c,3a,3b), real."""
    V = solid_R(rel, p)  # (K, nc)
    G = [deriv_stencil(V, a, p) for a in range(3)]
    H = [[deriv_stencil(G[b], a, p) for b in range(3)] for a in range(3)]
    grad = np.stack([np.real(G[a] @ L.T) for a in range(3)], axis=-1)  # (K, 3c, 3a)
    hess = np.stack([np.stack([np.real(H[a][b] @ L.T) for b in range(3)], axis=-1)
                     for a in range(3)], axis=-2)  # (K, 3c, 3a, 3b)
    return grad, hess


# ---------------------------------------------------------------------------
# exact near-field kernels (Eqs. 4-6, 8) -- vectorised float64
# ---------------------------------------------------------------------------

def kernel_fq(r, sigma):
    """f(r) = g/(4 pi r^3), q(r) = (zeta - 3f)/r^2, with the rho<0.25 series and r=0 limits."""
    r = np.asarray(r, np.float64)
    zeta0 = (2.0 * math.pi * sigma * sigma) ** -1.5
    rho2 = r * r / (2.0 * sigma * sigma)
    rho = np.sqrt(rho2)
    f = np.empty_like(r)
    q = np.empty_like(r)
    small = rho < 0.25
    big = ~small
    if small.any():
        s = rho2[small]
        sf = np.zeros_like(s)
        sq = np.zeros_like(s)
        term = np.ones_like(s)
        for k in range(8):
            sf += term / (2 * k + 3)
            term = term * (-s) / (k + 1)
        term = -np.ones_like(s)
        for k in range(1, 9):
            sq += term / (2 * k + 3)
            term = term * (-s) / k
        f[small] = zeta0 * sf
        q[small] = zeta0 / (sigma * sigma) * sq
    if big.any():
        rb, pb = r[big], rho[big]
        e = np.exp(-rho2[big])
        g = erf(pb) - 2.0 / math.sqrt(math.pi) * pb * e
        fb = g / (FOUR_PI * rb ** 3)
        f[big] = fb
        q[big] = (zeta0 * e - 3.0 * fb) / (rb * rb)
    return f, q


def pair_sum(xi, gi, xs, gs, sigma, scheme=0):
    """Exact velocity/stretching at targets xi (T,3) with strengths gi from sources xs,gs (S,3)."""
    d = xi[:, None, :] - xs[None, :, :]  # (T,S,3)
    r = np.sqrt((d * d).sum(-1))
    f, q = kernel_fq(r, sigma)
    c = np.cross(np.broadcast_to(gs[None, :, :], d.shape), d)  # gamma_j x d
    u = (f[..., None] * c).sum(1)
    if scheme == 0:
        gd = (gi[:, None, :] * d).sum(-1)
        s = (f[..., None] * np.cross(np.broadcast_to(gs[None], d.shape),
                                     np.broadcast_to(gi[:, None], d.shape))).sum(1)
        s += ((q * gd)[..., None] * c).sum(1)
    else:
        gc = (gi[:, None, :] * c).sum(-1)
        s = (f[..., None] * np.cross(np.broadcast_to(gi[:, None], d.shape),
                                     np.broadcast_to(gs[None], d.shape))).sum(1)
        s += ((q * gc)[..., None] * d).sum(1)
    return u, s


# ---------------------------------------------------------------------------
# the FMM, step by step
# ---------------------------------------------------------------------------

def _m_decode(c: int, l: int):
    ix = iy = iz = 0
    for b in range(l):
        ix |= ((c >> (3 * b)) & 1) << b
        iy |= ((c >> (3 * b + 1)) & 1) << b
        iz |= ((c >> (3 * b + 2)) & 1) << b
    return ix, iy, iz


def _m_encode(ix: int, iy: int, iz: int, l: int) -> int:
    c = 0
    for b in range(l):
        c |= ((ix >> b) & 1) << (3 * b)
        c |= ((iy >> b) & 1) << (3 * b + 1)
        c |= ((iz >> b) & 1) << (3 * b + 2)
    return c


def periodic_far(M0, box_len: float, image_levels: int, p: int):
    """L0 contribution of all images outside the near 3^3 block (reading R5):
    ring k (k = 0..levels-2): supercells of width w_k = 3^k len at offsets n w_k,
    n in {-4..4}^3 minus {-1..1}^3; supercell k+1 = M2M of the 27 supercells k."""
    L0 = np.zeros_like(M0)
    Mk = M0.copy()
    ring = [(a, b, c) for a in range(-4, 5) for b in range(-4, 5) for c in range(-4, 5)
            if max(abs(a), abs(b), abs(c)) > 1]
    near = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)]
    for k in range(0, image_levels - 1):
        w = box_len * 3.0 ** k
        for n in ring:
            T = m2l_matrix(-np.array(n, np.float64) * w, p)
            L0 += Mk @ T.T
        Mn = np.zeros_like(Mk)
        for d in near:
            A = m2m_matrix(np.array(d, np.float64) * w, p)
            Mn += Mk @ A.T
        Mk = Mn
    return L0


def evaluate(pos, gam, sigma, box_lo, box_len, depth, p, image_levels=3, scheme=0,
             return_stages=False):
    """Step-by-step FMM in float64.  pos, gam: (3,N) (float32 inputs widened exactly).
    Returns (vel (3,N), dgam (3,N)) in input order [, stages dict]."""
    pos = np.asarray(pos)
    N = pos.shape[1]
    lo = float(np.float32(box_lo))
    ln = float(np.float32(box_len))
    L = int(depth)
    periodic = image_levels > 0
    keys, perm, leaf_start, rc = _morton(np.asarray(pos, np.float32), L, lo, ln)
    if rc != 0:
        raise ValueError("positions outside the box")
    X = np.asarray(pos, np.float64).T[perm.astype(np.int64)]  # sorted (N,3)
    Gm = np.asarray(gam, np.float64).T[perm.astype(np.int64)]
    nleaf = 1 << (3 * L)
    side = 1 << L
    a = ln / side
    nc = ncoef(p)

    def center(c, l):
        ix, iy, iz = _m_decode(c, l)
        w = ln / (1 << l)
        return np.array([lo + (ix + 0.5) * w, lo + (iy + 0.5) * w, lo + (iz + 0.5) * w])

    # P2M at leaves (Eq. 10)
    M = [None] * (L + 1)
    M[L] = np.zeros((nleaf, 3, nc), np.complex128)
    for c in range(nleaf):
        s, e = leaf_start[c], leaf_start[c + 1]
        if e > s:
            M[L][c] = p2m(X[s:e] - center(c, L), Gm[s:e], p)
    # M2M upward
    for l in range(L - 1, -1, -1):
        M[l] = np.zeros((1 << (3 * l), 3, nc), np.complex128)
        w = ln / (1 << (l + 1))
        for ch in range(8):
            d = np.array([((ch >> 0) & 1) - 0.5, ((ch >> 1) & 1) - 0.5, ((ch >> 2) & 1) - 0.5]) * w
            A = m2m_matrix(d, p)
            M[l] += M[l + 1][ch::8] @ A.T
    # local expansions
    Lx = [np.zeros((1 << (3 * l), 3, nc), np.complex128) for l in range(L + 1)]
    if periodic and image_levels >= 2:
        Lx[0][0] = periodic_far(M[0][0], ln, image_levels, p)
    # M2L, levels 1..L (ws = 1, periodic wrap of source cells)
    cache = {}
    for l in range(1, L + 1):
        n_l = 1 << l
        w = ln / n_l
        groups = {}
        for t in range(1 << (3 * l)):
            tx, ty, tz = _m_decode(t, l)
            px, py, pz = tx >> 1, ty >> 1, tz >> 1
            for sx in range(2 * px - 2, 2 * px + 4):
                for sy in range(2 * py - 2, 2 * py + 4):
                    for sz in range(2 * pz - 2, 2 * pz + 4):
                        o = (sx - tx, sy - ty, sz - tz)
                        if max(abs(o[0]), abs(o[1]), abs(o[2])) <= 1:
                            continue
                        if not periodic and not (0 <= sx < n_l and 0 <= sy < n_l and 0 <= sz < n_l):
                            continue
                        s = _m_encode(sx % n_l, sy % n_l, sz % n_l, l)
                        groups.setdefault(o, []).append((t, s))
        for o, pairs in groups.items():
            key = (o, l)
            if key not in cache:
                cache[key] = m2l_matrix(-np.array(o, np.float64) * w, p)
            T = cache[key]
            tt = np.array([q[0] for q in pairs])
            ss = np.array([q[1] for q in pairs])
            np.add.at(Lx[l], tt, M[l][ss] @ T.T)
    # L2L downward
    for l in range(0, L):
        w = ln / (1 << (l + 1))
        for ch in range(8):
            d = np.array([((ch >> 0) & 1) - 0.5, ((ch >> 1) & 1) - 0.5, ((ch >> 2) & 1) - 0.5]) * w
            A = l2l_matrix(d, p)
            Lx[l + 1][ch::8] += Lx[l] @ A.T
    # L2P (far field, g = 1) and P2P (near field, exact) per leaf
    vel = np.zeros((N, 3))
    dg = np.zeros((N, 3))
    eps = np.zeros((3, 3, 3))
    eps[0, 1, 2] = eps[1, 2, 0] = eps[2, 0, 1] = 1.0
    eps[0, 2, 1] = eps[2, 1, 0] = eps[1, 0, 2] = -1.0
    for c in range(nleaf):
        s, e = leaf_start[c], leaf_start[c + 1]
        if e == s:
            continue
        xi, gi = X[s:e], Gm[s:e]
        grad, hess = l2p(Lx[L][c], xi - center(c, L), p)  # (K,3c,3a), (K,3c,3a,3b)
        # u_a = eps_abc d_b phi_c / 4pi
        uf = np.einsum("abc,kcb->ka", eps, grad) / FOUR_PI
        if scheme == 0:
            sf = np.einsum("abc,kcdb,kd->ka", eps, hess, gi) / FOUR_PI  # eps_abc g_d d_d d_b phi_c
        else:
            sf = np.einsum("dbc,kcab,kd->ka", eps, hess, gi) / FOUR_PI  # eps_dbc g_d d_a d_b phi_c
        tx, ty, tz = _m_decode(c, L)
        xs_list, gs_list = [], []
        for ox in (-1, 0, 1):
            for oy in (-1, 0, 1):
                for oz in (-1, 0, 1):
                    nx, ny, nz = tx + ox, ty + oy, tz + oz
                    if not periodic and not (0 <= nx < side and 0 <= ny < side and 0 <= nz < side):
                        continue
                    sc = _m_encode(nx % side, ny % side, nz % side, L)
                    shift = np.array([(nx - nx % side), (ny - ny % side), (nz - nz % side)],
                                     np.float64) / side * ln
                    s2, e2 = leaf_start[sc], leaf_start[sc + 1]
                    if e2 > s2:
                        xs_list.append(X[s2:e2] + shift)
                        gs_list.append(Gm[s2:e2])
        un, sn = pair_sum(xi, gi, np.concatenate(xs_list), np.concatenate(gs_list), sigma, scheme)
        vel[s:e] = uf + un
        dg[s:e] = sf + sn
    out_v = np.zeros((3, N))
    out_s = np.zeros((3, N))
    out_v[:, perm.astype(np.int64)] = vel.T
    out_s[:, perm.astype(np.int64)] = dg.T
    if return_stages:
        return out_v, out_s, {"M": M, "L": Lx, "perm": perm, "leaf_start": leaf_start,
                              "keys": keys}
    return out_v, out_s
