"""Seeded synthetic input generators (test/bench plumbing; none of the method's arithmetic).

Shared by the oracle-side tests and the CUDA-side tests/bench: it only builds the
particle fields the paper's runs use (section 4.2, :183-191):

* particles at the centres of an n^3 lattice in the box [lo, lo+len)^3 (PAPER.md:191,
  "placed at the center of this box"), x fastest, h = len/n, sigma = h (overlap 1, :191);
* strengths gamma_j = h^3 omega(x_j) -- the RBF solver's initial guess;
* omega from Taylor-Green (config c1) or from a solenoidal random-phase field with
  E(k) ~ k^4 exp(-2k^2/k_p^2), k_p = 4 (Rogallo), normalised so the
  large-eddy turnover time T = L/u' = 2; omega is the exact spectral curl
  evaluated at cell centres (reading R15, instead of the paper's 4th-order differences);
* c5 stand-in: a von Karman-Pao spectrum with more small-scale content (reading R14);
* robustness fields (not timed): jittered lattices, clustered random points (non-uniform
  leaves: empty and overfull), dense leaves, distinct coincident particles.

Everything is float32 on output (the GPU path's precision); the box is
lo = float32(-pi), len = float32(2 pi) (reading R8).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

BOX_LO = np.float32(-math.pi)
BOX_LEN = np.float32(2.0 * math.pi)


@dataclass
class Field:
    pos: np.ndarray      # (3, N) float32, SoA
    gamma: np.ndarray    # (3, N) float32, SoA
    sigma: float         # float32 value
    box_lo: float
    box_len: float
    n: int               # lattice points per axis
    name: str


def lattice(n: int):
    """Cell-centre lattice, x fastest: index = kx + n (ky + n kz).  Returns (3, n^3) float32."""
    lo = float(BOX_LO)
    h = float(BOX_LEN) / n
    k = np.arange(n, dtype=np.float64)
    c = lo + (k + 0.5) * h
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    pos = np.stack([x.ravel(), y.ravel(), z.ravel()]).astype(np.float32)
    hi = np.float32(BOX_LO + BOX_LEN)
    pos = np.where(pos >= hi, np.nextafter(hi, np.float32(-np.inf)), pos)
    return pos


def sigma_for(n: int, overlap: float = 1.0) -> float:
    """sigma = h / overlap, h = len/n (overlap h/sigma)."""
    return float(np.float32(float(BOX_LEN) / n / overlap))


def taylor_green(n: int) -> Field:
    """u_TG = (sin x cos y cos z, -cos x sin y cos z, 0);
    omega_TG = (-cos x sin y sin z, -sin x cos y sin z, 2 sin x sin y cos z)."""
    pos = lattice(n)
    x, y, z = (pos[i].astype(np.float64) for i in range(3))
    h = float(BOX_LEN) / n
    om = np.stack([-np.cos(x) * np.sin(y) * np.sin(z),
                   -np.sin(x) * np.cos(y) * np.sin(z),
                   2.0 * np.sin(x) * np.sin(y) * np.cos(z)])
    gam = (om * h ** 3).astype(np.float32)
    return Field(pos, gam, sigma_for(n), float(BOX_LO), float(BOX_LEN), n, f"taylor_green_{n}")


def _spectrum(k, kind: str, kp: float):
    if kind == "pp":  # PAPER.md:185, E ~ k^4 exp(-2k^2/kp^2)
        return k ** 4 * np.exp(-2.0 * k ** 2 / kp ** 2)
    if kind == "vkp":  # von Karman-Pao stand-in for the Re_lambda=100 reinitialized field
        ke, kd = 4.0, None
        return (k / ke) ** 4 * (1.0 + (k / ke) ** 2) ** (-17.0 / 6.0)
    raise ValueError(kind)


def isotropic(n: int, seed: int = 11102921, kind: str = "pp", kp: float = 4.0,
              T: float = 2.0) -> Field:
    """Solenoidal random-phase isotropic field (Rogallo 1981 construction),
    zero mean, k = 0 and Nyquist planes zeroed, normalised to T = L/u' = 2."""
    rng = np.random.default_rng(seed)
    k1 = np.fft.fftfreq(n, 1.0 / n)
    kr = np.fft.rfftfreq(n, 1.0 / n)
    KZ, KY, KX = np.meshgrid(k1, k1, kr, indexing="ij")
    kk = np.sqrt(KX ** 2 + KY ** 2 + KZ ** 2)
    shape = kk.shape
    th1 = rng.uniform(0, 2 * np.pi, shape)
    th2 = rng.uniform(0, 2 * np.pi, shape)
    phi = rng.uniform(0, 2 * np.pi, shape)
    ksafe = np.where(kk > 0, kk, 1.0)
    E = _spectrum(ksafe, kind, kp)
    if kind == "vkp":
        E = E * np.exp(-2.0 * (ksafe / (n / 6.0)) ** 2)
    amp = np.sqrt(E / (4.0 * np.pi * ksafe ** 2))
    alpha = amp * np.exp(1j * th1) * np.cos(phi)
    beta = amp * np.exp(1j * th2) * np.sin(phi)
    # Rogallo basis: e1 = k x z / |k x z| (or x if k || z), e2 = k x e1 / |k|
    kxy = np.sqrt(KX ** 2 + KY ** 2)
    par = kxy == 0
    e1 = np.stack([np.where(par, 1.0, KY / np.where(par, 1, kxy)),
                   np.where(par, 0.0, -KX / np.where(par, 1, kxy)),
                   np.zeros(shape)])
    kvec = np.stack([KX, KY, KZ])
    e2 = np.cross(kvec, e1, axis=0) / ksafe
    uh = alpha * e1 + beta * e2
    nyq = n // 2
    mask = (kk == 0) | (np.abs(KX) == nyq) | (np.abs(KY) == nyq) | (np.abs(KZ) == nyq)
    uh[:, mask] = 0.0
    h = float(BOX_LEN) / n
    # values at cell centres x = lo + h (j + 1/2): phase e^{i k (h/2)} relative to x_j = lo + h j
    shift = np.exp(1j * (KX + KY + KZ) * (h / 2.0) * (2.0 * np.pi / float(BOX_LEN)))
    uh = uh * shift
    # normalise: u' = sqrt(<|u|^2>/3), L = sqrt(2 pi)/kp for the pp spectrum; T = L/u'
    u = np.stack([np.fft.irfftn(uh[i], s=(n, n, n), axes=(0, 1, 2)) for i in range(3)])
    up = math.sqrt(float((u ** 2).sum(0).mean()) / 3.0)
    Lint = math.sqrt(2.0 * math.pi) / kp
    scale = (Lint / T) / up if up > 0 else 1.0
    uh *= scale
    # omega_hat = i k x u_hat (exact spectral curl; reading R15)
    kx, ky, kz = KX, KY, KZ
    wh = np.stack([1j * (ky * uh[2] - kz * uh[1]),
                   1j * (kz * uh[0] - kx * uh[2]),
                   1j * (kx * uh[1] - ky * uh[0])])
    # irfftn returns [z, y, x] indexed arrays -> ravel gives x fastest
    om = np.stack([np.fft.irfftn(wh[i], s=(n, n, n), axes=(0, 1, 2)).ravel() for i in range(3)])
    pos = lattice(n)
    gam = (om * h ** 3).astype(np.float32)
    return Field(pos, gam, sigma_for(n), float(BOX_LO), float(BOX_LEN), n,
                 f"isotropic_{kind}_{n}_s{seed}")


def jitter(f: Field, frac: float = 0.75, seed: int = 2) -> Field:
    """Move each particle uniformly by +-frac*h per axis and re-wrap into [lo, lo+len).
    frac > 0.5 moves particles across lattice cells (and leaf faces), so leaves hold unequal
    counts, some leaves can be empty, and pairs come arbitrarily close."""
    rng = np.random.default_rng(seed)
    h = f.box_len / f.n
    p = f.pos.astype(np.float64) + rng.uniform(-frac * h, frac * h, f.pos.shape)
    lo, ln = float(BOX_LO), float(BOX_LEN)
    p = lo + np.mod(p - lo, ln)
    p32 = p.astype(np.float32)
    hi = np.float32(BOX_LO + BOX_LEN)
    p32 = np.where(p32 >= hi, np.float32(BOX_LO), p32)
    p32 = np.where(p32 < BOX_LO, np.float32(BOX_LO), p32)
    return Field(p32, f.gamma.copy(), f.sigma, f.box_lo, f.box_len, f.n, f.name + "_jit")


# Configurations of BASELINE.json; depth gives 64 particles per leaf.
CONFIGS = {
    "c1": dict(n=16, field="tg", p=4, depth=2),
    "c2": dict(n=64, field="pp", p=6, depth=4, seed=11102921),
    "c3": dict(n=128, field="pp", p=10, depth=5, seed=11102921),
    "c4": dict(n=256, field="pp", p=10, depth=6, seed=11102921),
    "c5": dict(n=256, field="vkp", p=10, depth=6, seed=11102922),
}


def make(name: str, **over) -> Field:
    c = dict(CONFIGS[name])
    c.update(over)
    if c["field"] == "tg":
        return taylor_green(c["n"])
    return isotropic(c["n"], seed=c.get("seed", 11102921), kind=c["field"])


def sample_targets(n_total: int, count: int, seed: int = 3, n_lattice: int | None = None,
                   leaf: int = 4):
    """Seeded stratified target sample: 25% near box faces, 25% on leaf
    boundaries, 50% uniform.  Returns sorted unique int64 indices."""
    rng = np.random.default_rng(seed)
    if n_lattice is None or count >= n_total:
        return np.sort(rng.choice(n_total, size=min(count, n_total), replace=False)).astype(np.int64)
    n = n_lattice
    out = set()
    q = count // 4
    while len(out) < q:  # near a face: some coordinate in {0, n-1}
        k = rng.integers(0, n, 3)
        k[rng.integers(0, 3)] = rng.choice([0, n - 1])
        out.add(int(k[0] + n * (k[1] + n * k[2])))
    while len(out) < 2 * q:  # leaf boundary: coordinate = 0 or leaf-1 mod leaf
        k = rng.integers(0, n, 3)
        a = rng.integers(0, 3)
        k[a] = (k[a] // leaf) * leaf + rng.choice([0, leaf - 1])
        out.add(int(k[0] + n * (k[1] + n * k[2])))
    while len(out) < count:
        out.add(int(rng.integers(0, n_total)))
    return np.array(sorted(out), np.int64)


def clustered(n: int, n_clusters: int = 12, spread: float = 0.25, seed: int = 31,
              sigma: float = 0.05, strength: float = 1e-3) -> Field:
    """n random points in Gaussian clusters (std `spread`, wrapped into the box) around
    uniform random centres, plus normal strengths: strongly non-uniform leaf occupancy (many
    empty leaves, some with hundreds of particles) for robustness tests."""
    rng = np.random.default_rng(seed)
    lo, ln = float(BOX_LO), float(BOX_LEN)
    centres = rng.uniform(lo, lo + ln, (3, n_clusters))
    which = rng.integers(0, n_clusters, n)
    p = centres[:, which] + rng.normal(0.0, spread, (3, n))
    p = lo + np.mod(p - lo, ln)
    p32 = p.astype(np.float32)
    hi = np.float32(BOX_LO + BOX_LEN)
    p32 = np.where(p32 >= hi, np.float32(BOX_LO), p32)
    p32 = np.where(p32 < BOX_LO, np.float32(BOX_LO), p32)
    gam = (rng.normal(size=(3, n)) * strength).astype(np.float32)
    return Field(p32, gam, float(np.float32(sigma)), float(BOX_LO), float(BOX_LEN), 0,
                 f"clustered{n}_s{seed}")


def with_coincident(f: Field, count: int = 16, seed: int = 41) -> Field:
    """Copy of f in which `count` particles are moved exactly onto other particles' positions
    (distinct coincident pairs: the r -> 0 limits of Eqs. 5 and 8, reading R7)."""
    rng = np.random.default_rng(seed)
    n = f.pos.shape[1]
    idx = rng.choice(n, 2 * count, replace=False)
    pos = f.pos.copy()
    pos[:, idx[:count]] = pos[:, idx[count:]]
    return Field(pos, f.gamma.copy(), f.sigma, f.box_lo, f.box_len, f.n, f.name + "_coinc")
