"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

* tree: Morton keys, stable sort and leaf ranges bit-exact vs oracle.morton
* DIRECT mode vs the direct-sum oracle O1 (FP32 kernel arithmetic vs float64)
* NEAR_ONLY / FAR_ONLY structure; NEAR_ONLY at depth 1 free space == O1
* FMM vs the float64 step-by-step FMM oracle (same algorithm: FP32 rounding only),
  including per-stage multipole / local expansions
* FMM vs O1 at the frozen per-p tolerances (tests/tolerances.py), p sweep decreasing
* edge cases: ragged N, single particle, empty leaves, free space, jittered, bad input
* full size (256^3, the bench configuration) on sampled targets
"""
import math

import numpy as np
import pytest

import oracle
import synthgen
from oracle import fmm_ref as F
import tolerances as TOL  # tests/tolerances.py

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1110_2921_b200 as vf  # noqa: E402

DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def run(field, **kw):
    ev = vf.Evaluator(sigma=field.sigma, box_lo=field.box_lo, box_len=field.box_len, **kw)
    pos = torch.from_numpy(np.ascontiguousarray(field.pos)).to(DEV)
    gam = torch.from_numpy(np.ascontiguousarray(field.gamma)).to(DEV)
    v, s = ev.evaluate(pos, gam)
    ev.sync_status()
    torch.cuda.synchronize()
    return v.cpu().numpy().astype(np.float64), s.cpu().numpy().astype(np.float64), ev


def random_field(n, seed=0, sigma=0.3):
    rng = np.random.default_rng(seed)
    lo, ln = synthgen.BOX_LO, synthgen.BOX_LEN
    pos = rng.uniform(float(lo), float(lo + ln), (3, n)).astype(np.float32)
    pos = np.minimum(pos, np.nextafter(np.float32(lo + ln), np.float32(0)))
    gam = rng.normal(size=(3, n)).astype(np.float32) * 1e-3
    return synthgen.Field(pos, gam, sigma, float(lo), float(ln), 0, f"random{n}")


# ------------------------------------------------------------------ tree (bit-exact)

@pytest.mark.parametrize("case", ["c1", "c2", "c1j", "rand", "ragged"])
def test_tree_bit_exact(case):
    if case == "c1":
        f, depth = synthgen.make("c1"), 2
    elif case == "c2":
        f, depth = synthgen.make("c2"), 4
    elif case == "c1j":
        f, depth = synthgen.jitter(synthgen.make("c1")), 3
    elif case == "rand":
        f, depth = random_field(100000, 1), 5
    else:
        f, depth = random_field(12345, 2), 3
    _, _, ev = run(f, p=2, depth=depth, image_levels=1, mode=vf.MODE_NEAR_ONLY)
    keys, perm, ls = ev.debug_tree(depth)
    k_o, p_o, ls_o, rc = oracle.morton(f.pos, depth, f.box_lo, f.box_len)
    assert rc == 0
    assert np.array_equal(keys, k_o)
    assert np.array_equal(perm, p_o)
    assert np.array_equal(ls, ls_o)
    ev.close()


def test_bad_input_is_flagged():
    f = random_field(1000, 3)
    f.pos[1, 17] = np.float32(f.box_lo + f.box_len)  # upper face is outside [lo, lo+len)
    ev = vf.Evaluator(sigma=f.sigma, p=2, depth=2, image_levels=1)
    pos = torch.from_numpy(f.pos).to(DEV)
    gam = torch.from_numpy(f.gamma).to(DEV)
    ev.evaluate(pos, gam)
    with pytest.raises(vf.VfmmError) as e:
        ev.sync_status()
    assert e.value.status == vf.VFMM_EDOMAIN
    ev.sync_status()  # sticky flag was cleared
    with pytest.raises(vf.VfmmError):
        ev.evaluate_into(pos, gam, pos, gam)  # outputs aliasing inputs
    ev.close()


# ------------------------------------------------------------------ DIRECT / NEAR vs O1

@pytest.mark.parametrize("lam,scheme", [(0, 0), (1, 0), (1, 1), (3, 0)])
def test_direct_mode_vs_oracle(lam, scheme):
    f = synthgen.make("c1") if lam != 0 else random_field(3000, 4)
    v, s, ev = run(f, p=2, image_levels=lam, scheme=scheme, mode=vf.MODE_DIRECT)
    tg = synthgen.sample_targets(f.pos.shape[1], 64, n_lattice=f.n or None)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, lam, scheme, targets=tg)
    assert rel(v[:, tg], vo) < TOL.DIRECT_VS_ORACLE[0]
    assert rel(s[:, tg], so) < TOL.DIRECT_VS_ORACLE[1]
    ev.close()


@pytest.mark.parametrize("scheme,p2p", [(0, "sj"), (0, "cross"), (1, "cross")])
def test_near_only_depth1_free_space_equals_direct(scheme, p2p, monkeypatch):
    """Depth 1, free space: all octants are neighbours, so P2P alone is the whole sum.
    Classical scheme in both P2P accumulations (VFMM_P2P=cross: per-pair gamma_j x d; default /
    VFMM_P2P=sj: staged gamma_j x x_j, looser FP32 rounding bound).  The jittered lattice
    (+-0.75 h) has unequal leaves and close pairs; 16 distinct coincident pairs exercise the
    r -> 0 limits (reading R7)."""
    monkeypatch.setenv("VFMM_P2P", p2p)
    f = synthgen.with_coincident(synthgen.jitter(synthgen.taylor_green(12), seed=5))
    v, s, ev = run(f, p=2, depth=1, image_levels=0, scheme=scheme, mode=vf.MODE_NEAR_ONLY)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 0, scheme)
    tol = TOL.NEAR_VS_ORACLE_SJ if (scheme == 0 and p2p == "sj") else TOL.NEAR_VS_ORACLE
    assert rel(v, vo) < tol[0] and rel(s, so) < tol[1], (rel(v, vo), rel(s, so))
    ev.close()


@pytest.mark.parametrize("scheme", [0, 1])
def test_near_only_dense_leaves_multiwindow_equals_direct(scheme, monkeypatch):
    """Dense leaves: 20000 clustered points at depth 1 (thousands per leaf) -- the P2P kernel
    stages the 64-leaf region in several shared-memory windows (> 4352 sources) and loops over
    many 64-target chunks per warp.  Free space, so NEAR_ONLY is the whole direct sum.  Per-pair
    cross products (VFMM_P2P=cross): at depth 1 the staged form's lever arm is the whole box."""
    monkeypatch.setenv("VFMM_P2P", "cross")
    f = synthgen.with_coincident(synthgen.clustered(20000, seed=33, sigma=0.2), count=8)
    v, s, ev = run(f, p=2, depth=1, image_levels=0, scheme=scheme, mode=vf.MODE_NEAR_ONLY)
    keys, perm, ls = ev.debug_tree(1)
    assert np.diff(ls).max() > 2 * 4352 // 8  # several windows per region
    tg = np.arange(0, 20000, 61)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 0, scheme, targets=tg,
                           batched=True)
    tu, ts = TOL.NEAR_VS_ORACLE_DENSE
    assert rel(v[:, tg], vo) < tu and rel(s[:, tg], so) < ts, (rel(v[:, tg], vo), rel(s[:, tg], so))
    ev.close()


def test_dense_leaves_fmm_vs_direct():
    """64^3 lattice at depth 3 (512 particles per leaf; 64 x 512 staged sources per region in
    8 windows), p = 8, one image level, against O1 on stratified targets."""
    f = synthgen.isotropic(64, seed=15)
    v, s, ev = run(f, p=8, depth=3, image_levels=1)
    tg = synthgen.sample_targets(64 ** 3, 32, n_lattice=64, leaf=8)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 0, targets=tg,
                           batched=True)
    tu, ts = TOL.FMM_VS_DIRECT[8]
    assert rel(v[:, tg], vo) < tu and rel(s[:, tg], so) < ts, (rel(v[:, tg], vo), rel(s[:, tg], so))
    ev.close()


def test_clustered_field_vs_direct():
    """Non-uniform leaves (SURVEY 8(d) robustness fields): 20000 points in 12 Gaussian clusters
    at depth 3 -- 318 of 512 leaves empty, up to 1105 particles in one leaf -- with coincident
    pairs, p = 10, one image level.  The fp64 FMM oracle's own error here is 4.0e-6 / 3.8e-6."""
    f = synthgen.with_coincident(synthgen.clustered(20000), count=8)
    v, s, ev = run(f, p=10, depth=3, image_levels=1)
    tg = np.arange(0, 20000, 97)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 0, targets=tg,
                           batched=True)
    eu, es = rel(v[:, tg], vo), rel(s[:, tg], so)
    print(f"clustered p=10: u {eu:.2e} sdot {es:.2e}")
    tu, ts = TOL.FMM_VS_DIRECT[10]
    assert eu < tu and es < ts, (eu, es)
    ev.close()


def test_north_star_accuracy_p13_27cubed_vs_direct():
    """north_star: u within 1e-5 of the direct sum (and sdot within 3e-5) at the benched image
    count.  With the uniform ws = 1 tree that takes p = 13 ((p+1)^2 = 196: the tcgen05 M2L with
    two 128-row output tiles); isotropic 32^3, depth 3, 27^3 images, against O1."""
    f = synthgen.isotropic(32, seed=12)
    tg = synthgen.sample_targets(32 ** 3, 48, n_lattice=32)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 3, 0, targets=tg,
                           batched=True)
    v, s, ev = run(f, p=13, depth=3, image_levels=3)
    eu, es = rel(v[:, tg], vo), rel(s[:, tg], so)
    print(f"iso32 lambda=3 p=13 (tc f16, 2 row tiles): u {eu:.2e} sdot {es:.2e}")
    tu, ts = TOL.FMM_VS_DIRECT[13]
    assert eu < tu and es < ts, (eu, es)
    ev.close()


def test_periodic_27cubed_images_vs_direct():
    """The benched image count (27^3 boxes, image_levels = 3) against O1
    over the same cube, isotropic 32^3, p = 10, depth 3.  On this field O1 at lambda = 2 differs
    from lambda = 3 by 7.2e-4 (u), so a wrong or missing outer supercell ring fails."""
    f = synthgen.isotropic(32, seed=12)
    tg = synthgen.sample_targets(32 ** 3, 48, n_lattice=32)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 3, 0, targets=tg,
                           batched=True)
    for engine in ("f16", "simt"):
        import os
        os.environ["VFMM_M2L"] = engine
        try:
            v, s, ev = run(f, p=10, depth=3, image_levels=3)
        finally:
            os.environ.pop("VFMM_M2L", None)
        eu, es = rel(v[:, tg], vo), rel(s[:, tg], so)
        print(f"iso32 lambda=3 p=10 {engine}: u {eu:.2e} sdot {es:.2e}")
        tu, ts = TOL.FMM_VS_DIRECT[10]
        assert eu < tu and es < ts, (engine, eu, es)
        ev.close()


def test_m2m_split_levels_per_stage_depth5():
    """Depth 5: the level-4 M2M (4096 parents, < 2 tiles per SM) runs as the deterministic
    8-way child split + ordered sum.  Per-stage check of every level's multipoles against the
    fp64 M2M operators (oracle.fmm_ref.m2m_matrix) applied to the GPU's own child level."""
    f = synthgen.isotropic(32, seed=6)
    p, depth = 6, 5
    v, s, ev = run(f, p=p, depth=depth, image_levels=1, mode=vf.MODE_FAR_ONLY)
    for l in range(depth - 1, -1, -1):
        child = _unpack(ev.debug_expansions(0, l + 1), p, (f.box_len / (1 << (l + 1))) ** np.arange(p + 1.0))
        got = _unpack(ev.debug_expansions(0, l), p, (f.box_len / (1 << l)) ** np.arange(p + 1.0))
        want = np.zeros_like(got)
        mag = np.zeros(got.shape)  # sum of |terms|: FP32 rounding scale under cancellation
        w = f.box_len / (1 << (l + 1))
        for ch in range(8):
            d = np.array([(ch & 1) - 0.5, ((ch >> 1) & 1) - 0.5, ((ch >> 2) & 1) - 0.5]) * w
            t = child[ch::8] @ F.m2m_matrix(d, p).T
            want += t
            mag += np.abs(t)
        err = np.linalg.norm(got - want) / np.linalg.norm(mag)
        assert err < 1e-6, (l, err)
    ev.close()


def _unpack(P, p, scale_n):
    """packed real [cell][comp][(p+1)^2] -> complex [cell][comp][(n,m) full], times scale_n[n]
    (negative m from the real-source symmetry C_n^{-m} = (-1)^m conj(C_n^m))."""
    out = np.zeros(P.shape[:2] + ((p + 1) ** 2,), np.complex128)
    P = P.astype(np.float64)
    for n in range(p + 1):
        out[..., F.kidx(n, 0)] = P[..., n * n] * scale_n[n]
        for m in range(1, n + 1):
            c = (P[..., n * n + 2 * m - 1] + 1j * P[..., n * n + 2 * m]) * scale_n[n]
            out[..., F.kidx(n, m)] = c
            out[..., F.kidx(n, -m)] = (-1) ** m * np.conj(c)
    return out


def test_near_plus_far_equals_fmm():
    f = synthgen.isotropic(16, seed=7)
    v, s, ev = run(f, p=6, depth=2, image_levels=3)
    vn, sn, _ = run(f, p=6, depth=2, image_levels=3, mode=vf.MODE_NEAR_ONLY)
    vf_, sf_, _ = run(f, p=6, depth=2, image_levels=3, mode=vf.MODE_FAR_ONLY)
    assert np.abs(vn + vf_ - v).max() <= 1e-6 * np.abs(v).max()
    assert np.abs(sn + sf_ - s).max() <= 1e-6 * np.abs(s).max()
    ev.close()


# ------------------------------------------------------------------ FMM vs fp64 FMM oracle

def _fmm_oracle(f, depth, p, lam, scheme=0):
    return F.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, depth, p, lam, scheme,
                      return_stages=True)


@pytest.mark.parametrize("name,depth,p,lam,scheme", [
    ("c1", 2, 4, 3, 0),
    ("iso16", 2, 6, 2, 0),
    ("iso16", 2, 6, 2, 1),
    ("iso16", 3, 3, 0, 0),
    ("c1j", 2, 5, 1, 0),
    ("iso16", 2, 10, 2, 0),  # compile-time p = 10 kernels, tcgen05 f16 M2L
    ("c1", 2, 12, 1, 0),     # (p+1)^2 = 169 > 128: two row tiles, runtime-p P2M / L2P kernels
    ("c1", 2, 16, 1, 0),     # VFMM_PMAX: (p+1)^2 = 289 > 256: SIMT M2L, three 128-row tiles
])
@pytest.mark.parametrize("split", ["6", "full"])
def test_fmm_vs_fmm_oracle(name, depth, p, lam, scheme, split, monkeypatch):
    """Every stage against the float64 step-by-step FMM oracle.  With the order-split M2L
    (VFMM_M2L_SPLIT = 6, the default: terms of local and multipole degree >= 6 run hi x hi
    alone) the local expansions are compared at the FP32 bound on the rows of
    degree < 6 and at 5e-2 on every row: a high-degree row is a sum of operator terms that
    cancel by orders of magnitude, so hi x hi rounding (2^-11 per term) leaves up to ~1e-2 of
    the row, which reaches u and dgamma/dt below 1e-7 (test_m2l_order_split); "full" checks
    every row at the FP32 bound."""
    monkeypatch.setenv("VFMM_M2L_SPLIT", split)
    f = {"c1": lambda: synthgen.make("c1"), "iso16": lambda: synthgen.isotropic(16, seed=9),
         "c1j": lambda: synthgen.jitter(synthgen.make("c1"))}[name]()
    v, s, ev = run(f, p=p, depth=depth, image_levels=lam, scheme=scheme)
    vo, so, st = _fmm_oracle(f, depth, p, lam, scheme)
    assert rel(v, vo) < TOL.FMM_VS_FMM_ORACLE[0], rel(v, vo)
    assert rel(s, so) < TOL.FMM_VS_FMM_ORACLE[1], rel(s, so)
    # per-stage: leaf multipoles, and local expansions at every level (scaled, packed)
    a = f.box_len / (1 << depth)
    for l in range(depth + 1):
        al = f.box_len / (1 << l)
        for kind, C, scale in ((0, st["M"][l], al ** -np.arange(p + 1.0)),
                               (1, st["L"][l], al ** (np.arange(p + 1.0) + 1))):
            got = ev.debug_expansions(kind, l)
            want = _pack(C, p, scale)
            if kind == 1:  # L_0^0 is a constant potential: no effect on u or dgamma, and the
                got = got[..., 1:]  # periodic sum amplifies FP32 noise in sum(gamma) into it
                want = want[..., 1:]
            if np.abs(want).max() == 0:
                continue
            # FP32 sums over up to 8^L particles with cancellation (root multipole ~ 0); at
            # p = 16 the scaled M2L operators span ~(2p)! in magnitude and the high-order local
            # coefficients of the coarse levels keep ~1e-4, while u and dgamma
            # above still meet FMM_VS_FMM_ORACLE
            tol = 5e-5 if p <= 12 else 5e-4
            if kind == 1 and split != "full":
                low = min(36, got.shape[-1] + 1) - 1  # packed rows of degree < 6, minus L_0^0
                assert rel(got[..., :low], want[..., :low]) < tol, (kind, l, "deg<6")
                tol = max(tol, 5e-2)
            assert rel(got, want) < tol, (kind, l, rel(got, want))
    ev.close()


def _pack(C, p, scale_n):
    """complex coefficients [cell][comp][(n,m) full] -> packed real, times scale_n[n]."""
    out = np.zeros(C.shape[:2] + ((p + 1) ** 2,))
    for n in range(p + 1):
        out[..., n * n] = C[..., F.kidx(n, 0)].real * scale_n[n]
        for m in range(1, n + 1):
            out[..., n * n + 2 * m - 1] = C[..., F.kidx(n, m)].real * scale_n[n]
            out[..., n * n + 2 * m] = C[..., F.kidx(n, m)].imag * scale_n[n]
    return out


# ------------------------------------------------------------------ FMM vs direct sum

def test_auto_depth_matches_explicit():
    """depth = 0 picks the depth from N (~64 particles per leaf): same result as asking for it."""
    f = synthgen.isotropic(32, seed=4)
    v0, s0, ev0 = run(f, p=6, depth=0, image_levels=1)
    st = ev0.stats()
    L = st["depth_used"]
    assert L == 3  # 32^3 / 64 = 8^3 leaves
    v1, s1, ev1 = run(f, p=6, depth=L, image_levels=1)
    assert np.array_equal(v0, v1) and np.array_equal(s0, s1)
    ev0.close()
    ev1.close()


def test_coresident_mode_matches_sequential(monkeypatch):
    """VFMM_CORES=1: P2P on the caller's stream concurrently with the far-field chain on a
    high-priority stream, both in their lean variants (one block of each per SM): the same
    result as the sequential pipeline up to the P2P's FP32 summation order (its staging windows
    are smaller), the tensor-core M2L bitwise unchanged."""
    f = synthgen.isotropic(32, seed=14)
    monkeypatch.setenv("VFMM_P2P", "cross")  # the lean P2P variant has the per-pair form only
    v0, s0, ev0 = run(f, p=10, depth=3, image_levels=3)
    L0 = ev0.debug_expansions(1, 3)
    monkeypatch.setenv("VFMM_CORES", "1")
    v1, s1, ev1 = run(f, p=10, depth=3, image_levels=3)
    L1 = ev1.debug_expansions(1, 3)
    assert np.array_equal(L0, L1)
    assert rel(v1, v0) < 1e-6 and rel(s1, s0) < 1e-6, (rel(v1, v0), rel(s1, s0))
    ev0.close()
    ev1.close()


def test_tuned_depth_is_timed_and_consistent():
    """depth = -1: the first evaluate of a new N times the auto depth and its neighbours and
    keeps the fastest ("automatically choosing the number of particles per box");
    the result equals an explicit evaluation at the chosen depth, and the choice is cached."""
    f = synthgen.isotropic(64, seed=4)
    v0, s0, ev0 = run(f, p=6, depth=-1, image_levels=2)
    L = ev0.stats()["depth_used"]
    assert L in (3, 4, 5)
    v1, s1, ev1 = run(f, p=6, depth=L, image_levels=2)
    assert np.array_equal(v0, v1) and np.array_equal(s0, s1)
    pos = torch.from_numpy(f.pos).to(DEV)
    gam = torch.from_numpy(f.gamma).to(DEV)
    ev0.evaluate(pos, gam)
    assert ev0.stats()["depth_used"] == L
    print(f"tuned depth for 64^3 at p = 6: {L}")
    ev0.close()
    ev1.close()


@pytest.mark.parametrize("engine", ["f16", "simt"])
def test_evaluation_is_deterministic(engine, monkeypatch):
    """No atomics on the value path (op splits reduce partials in a fixed order): two
    evaluations of the same input are bitwise identical."""
    monkeypatch.setenv("VFMM_M2L", engine)
    f = synthgen.isotropic(16, seed=3)
    v0, s0, ev = run(f, p=6, depth=3, image_levels=2)
    v1, s1, ev1 = run(f, p=6, depth=3, image_levels=2)
    assert np.array_equal(v0, v1) and np.array_equal(s0, s1)
    ev.close()
    ev1.close()


def test_evaluates_on_different_streams_are_ordered():
    """one context's workspace serves every evaluate, so an evaluate on a new stream
    waits for the previous one (its end event).  Back-to-back evaluations of two different
    fields on two streams, without host synchronization in between, give each field's own
    single-stream result."""
    fa = synthgen.isotropic(32, seed=41)
    fb = synthgen.isotropic(32, seed=42)
    va, _, ev = run(fa, p=6, depth=3, image_levels=2)
    vb, _, ev_b = run(fb, p=6, depth=3, image_levels=2)
    ev_b.close()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    pa, ga = (torch.from_numpy(x).to(DEV) for x in (fa.pos, fa.gamma))
    pb, gb = (torch.from_numpy(x).to(DEV) for x in (fb.pos, fb.gamma))
    torch.cuda.synchronize()
    outs = []
    for k in range(3):
        with torch.cuda.stream(s1):
            v1, _ = ev.evaluate(pa, ga, stream=s1)
        with torch.cuda.stream(s2):
            v2, _ = ev.evaluate(pb, gb, stream=s2)
        outs.append((v1, v2))
    torch.cuda.synchronize()
    for v1, v2 in outs:
        assert np.array_equal(v1.cpu().numpy().astype(np.float64), va)
        assert np.array_equal(v2.cpu().numpy().astype(np.float64), vb)
    ev.close()


@pytest.mark.parametrize("mode", ["fmm", "direct"])
def test_host_buffers_match_device_buffers(mode):
    """vfmm_evaluate_host (pageable host in/out; the strengths' copy overlaps the tree build on
    a second stream) gives bitwise the device-buffer result, repeatedly."""
    f = synthgen.isotropic(16, seed=8)
    m = vf.MODE_FMM if mode == "fmm" else vf.MODE_DIRECT
    v0, s0, ev = run(f, p=6, depth=2, image_levels=2, mode=m)
    for _ in range(2):
        vh, sh = ev.evaluate_host(f.pos, f.gamma)
        assert np.array_equal(vh.astype(np.float64), v0) and np.array_equal(sh.astype(np.float64), s0)
    ev.close()


def test_c_example_matches_python_binding():
    """examples/vfmm_c_example.c drives the C ABI from plain C (vfmm_evaluate_host); its output
    matches the Python binding on the same lattice field (inputs rebuilt in float32)."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "examples", "vfmm_c_example")
    lib = os.path.join(root, "paper_1110_2921_b200", "lib")
    if not os.path.exists(exe):
        subprocess.check_call(["gcc", "-O2", "-I", os.path.join(root, "include"), exe + ".c",
                               "-L", lib, "-lvfmm", f"-Wl,-rpath,{lib}", "-lm", "-o", exe])
    out = subprocess.run([exe, "16"], capture_output=True, text=True, check=True).stdout.split("\n")
    n, p, depth = (int(t) for t in out[0].split()[:3])
    assert (n, p, depth) == (16, 6, 2)
    c_rows = np.array([[float(t) for t in out[k].split()] for k in (1, 2)])
    lo, ln = np.float32(synthgen.BOX_LO), np.float32(synthgen.BOX_LEN)
    h = ln / np.float32(n)
    i = np.arange(n ** 3)
    x = lo + h * ((i % n).astype(np.float32) + np.float32(0.5))
    y = lo + h * (((i // n) % n).astype(np.float32) + np.float32(0.5))
    z = lo + h * ((i // (n * n)).astype(np.float32) + np.float32(0.5))
    v3 = h * h * h
    g = np.stack([-np.cos(x) * np.sin(y) * np.sin(z) * v3, -np.sin(x) * np.cos(y) * np.sin(z) * v3,
                  np.float32(2) * np.sin(x) * np.sin(y) * np.cos(z) * v3]).astype(np.float32)
    pos = np.stack([x, y, z]).astype(np.float32)
    ev = vf.Evaluator(p=6, depth=2, image_levels=3, sigma=float(h), box_lo=float(lo),
                      box_len=float(ln))
    v, s = ev.evaluate_host(pos, g)
    py_rows = np.array([np.concatenate([v[:, k], s[:, k]]) for k in (0, n ** 3 - 1)])
    assert np.allclose(c_rows, py_rows, rtol=1e-4, atol=1e-6 * np.abs(py_rows).max()), (c_rows, py_rows)
    ev.close()


def test_c1_fmm_vs_direct_oracle():
    f = synthgen.make("c1")
    v, s, ev = run(f, p=4, depth=2, image_levels=3)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 3, 0)
    tu, ts = TOL.FMM_VS_DIRECT[4]
    assert rel(v, vo) < tu and rel(s, so) < ts
    ev.close()


def test_p_sweep_error_decreases():
    f = synthgen.isotropic(32, seed=12)
    tg = synthgen.sample_targets(32 ** 3, 48, n_lattice=32)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 0, targets=tg)
    errs = []
    for p in (4, 6, 8, 10):
        v, s, ev = run(f, p=p, depth=3, image_levels=1)
        errs.append((rel(v[:, tg], vo), rel(s[:, tg], so)))
        tu, ts = TOL.FMM_VS_DIRECT[p]
        assert errs[-1][0] < tu and errs[-1][1] < ts, (p, errs[-1])
        ev.close()
    for a, b in zip(errs, errs[1:]):
        assert b[0] < a[0] and b[1] < a[1], errs


# ------------------------------------------------------------------ edge cases

def test_single_particle_periodic_is_at_rest():
    f = random_field(1, 5)
    v, s, ev = run(f, p=6, depth=2, image_levels=3)
    # a lone particle feels no velocity from its own images (cube symmetry); FMM to tolerance
    assert np.abs(v).max() < 1e-6 * abs(f.gamma).max() / f.sigma ** 2
    ev.close()


def test_ragged_random_points_vs_direct():
    f = random_field(5003, 6, sigma=0.2)
    tg = np.arange(0, 5003, 97)
    v, s, ev = run(f, p=8, depth=3, image_levels=1)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 0, targets=tg)
    tu, ts = TOL.FMM_VS_DIRECT[8]
    assert rel(v[:, tg], vo) < tu and rel(s[:, tg], so) < ts
    ev.close()


def test_zero_strengths_give_zero():
    f = synthgen.make("c1")
    f.gamma[:] = 0
    v, s, ev = run(f, p=4, depth=2, image_levels=3)
    assert np.all(v == 0) and np.all(s == 0)
    ev.close()


# ------------------------------------------------------------------ full size (bench config)

@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_c4_full_size_sampled_targets(cfg):
    """256^3 (the bench workload c4, and the intermittent Re_lambda = 100 field c5; p = 10,
    depth 6): lambda = 1 so the oracle finishes in seconds per target; the lambda = 3
    far-image operator is covered at c1/c2 sizes."""
    f = synthgen.make(cfg)
    v, s, ev = run(f, p=10, depth=6, image_levels=1)
    tg = synthgen.sample_targets(f.pos.shape[1], 8, n_lattice=f.n)
    vo, so = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 0, targets=tg)
    tu, ts = TOL.FMM_VS_DIRECT[10]
    assert rel(v[:, tg], vo) < tu and rel(s[:, tg], so) < ts, (rel(v[:, tg], vo), rel(s[:, tg], so))
    ev.close()


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_bench_config_vs_golden_o1_27cubed(cfg):
    """Exactly the benched configuration (bench.py: p = 10, depth 6, image_levels = 3 = the
    paper's 27^3 boxes, default tensor-core M2L engine) against O1 reference values for 16
    stratified targets computed once by scripts/make_golden.py (oracle/ only) and stored in
    tests/golden/<cfg>_lam3_s0_o1.json."""
    import hashlib
    import json
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", f"{cfg}_lam3_s0_o1.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet (scripts/make_golden.py {cfg})")
    g = json.load(open(path))
    f = synthgen.make(cfg)
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(f.pos, np.float32).tobytes())
    h.update(np.ascontiguousarray(f.gamma, np.float32).tobytes())
    assert h.hexdigest() == g["field_sha256"], "generator output differs from the golden field"
    v, s, ev = run(f, p=10, depth=6, image_levels=3)
    tg = np.array(g["targets"], np.int64)
    vo, so = np.array(g["vel"]), np.array(g["dgamma"])
    eu, es = rel(v[:, tg], vo), rel(s[:, tg], so)
    print(f"{cfg} bench config vs O1 (27^3 images): u {eu:.3e} sdot {es:.3e}")
    tu, ts = TOL.FMM_VS_DIRECT[10]
    assert eu < tu and es < ts, (eu, es)
    ev.close()


# ------------------------------------------------------------------ tensor-core M2L (tcgen05)

_FP64_STAGES = {}


@pytest.mark.parametrize("engine", ["simt", "f16", "tf32"])
@pytest.mark.parametrize("n,depth,p,lam", [(32, 3, 10, 1), (32, 3, 6, 3), (64, 4, 8, 1),
                                           (16, 2, 13, 2), (16, 2, 15, 1),
                                           pytest.param(64, 5, 10, 3, marks=pytest.mark.slow)])
def test_m2l_engines_vs_fp64_fmm_oracle(n, depth, p, lam, engine, monkeypatch):
    if depth == 5 and engine != "f16":
        pytest.skip("depth 5 (fp64 oracle ~4 min): the default engine only; SIMT and 3xTF32 "
                    "measured in profiles/r2 (scripts/m2l_tc_accuracy.py)")
    """Every M2L engine -- SIMT FP32, tcgen05 scaled 3xFP16 (default), tcgen05 3xTF32 -- against
    the float64 step-by-step FMM oracle running the same algorithm: the local expansions of
    every level and the velocity / stretching differ by FP32 rounding only.  The tensor core
    accumulates with truncation; chains are cut after every (offset, K chunk) and summed in
    FP32 registers (DESIGN.md "tcgen05 M2L accuracy")."""
    f = synthgen.isotropic(n, seed=21)
    monkeypatch.setenv("VFMM_M2L", engine)
    monkeypatch.setenv("VFMM_M2L_SPLIT", "full")  # the engine's arithmetic on every term
    v, s, ev = run(f, p=p, depth=depth, image_levels=lam)
    key = (n, depth, p, lam)
    if key not in _FP64_STAGES:  # one fp64 oracle run serves the three engines
        _FP64_STAGES[key] = F.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, depth, p,
                                       lam, return_stages=True)
    vo, so, st = _FP64_STAGES[key]
    line = [f"{engine} n={n} L={depth} p={p} lam={lam}: u {rel(v, vo):.2e} sdot {rel(s, so):.2e}"]
    for l in range(1, depth + 1):
        al = f.box_len / (1 << l)
        got = ev.debug_expansions(1, l)[..., 1:]
        want = _pack(st["L"][l], p, al ** (np.arange(p + 1.0) + 1))[..., 1:]
        line.append(f"L{l} {rel(got, want):.2e}")
        # the finest levels at p = 10 carry ~1.3e-5 of FP32 rounding in EVERY engine (SIMT
        # included: 64^3, depth 5 -- 8 particles per leaf), none of which reaches u or sdot
        assert rel(got, want) < (5e-6 if l < 4 else 2e-5), (l, rel(got, want))
    print(" ".join(line))
    assert rel(v, vo) < 3e-6 and rel(s, so) < 3e-6, (rel(v, vo), rel(s, so))
    ev.close()


@pytest.mark.parametrize("engine", ["tf32", "f16"])
@pytest.mark.parametrize("n,depth,p,lam", [(48, 5, 6, 0), (128, 6, 8, 1), (32, 4, 13, 1),
                                           (64, 5, 12, 3)])
def test_m2l_tensor_core_matches_simt(n, depth, p, lam, engine, monkeypatch):
    """Deeper trees than the fp64 oracle reaches: levels >= 2 on tcgen05 (3xTF32, or the
    balanced 3xFP16 split) against the SIMT FP32 gather-GEMM (itself validated against the fp64
    FMM oracle above) on the far field: velocity and stretching within 5e-6; the finest local
    expansions, where both engines' FP32 rounding shows, within 1e-5."""
    f = synthgen.isotropic(n, seed=21)
    monkeypatch.setenv("VFMM_M2L", engine)
    monkeypatch.setenv("VFMM_M2L_SPLIT", "full")
    v1, s1, ev1 = run(f, p=p, depth=depth, image_levels=lam, mode=vf.MODE_FAR_ONLY)
    monkeypatch.setenv("VFMM_M2L", "simt")
    v2, s2, ev2 = run(f, p=p, depth=depth, image_levels=lam, mode=vf.MODE_FAR_ONLY)
    print(f"tc {engine} vs simt n={n} L={depth} p={p} lam={lam}: u {rel(v1, v2):.2e} "
          f"sdot {rel(s1, s2):.2e}")
    assert rel(v1, v2) < 5e-6 and rel(s1, s2) < 5e-6, (rel(v1, v2), rel(s1, s2))
    # the scaled operators span ~(2p)! in FP32, so both engines' finest expansions carry more
    # rounding at p > 10 (DESIGN.md 7 "High p"; 5e-4 against fp64 at p = 16)
    etol = 1e-5 if p <= 10 else 5e-5
    for l in range(depth - 1, depth + 1):
        a, b = ev1.debug_expansions(1, l), ev2.debug_expansions(1, l)
        print(f"  level {l}: {rel(a[..., 1:], b[..., 1:]):.2e}")
        assert rel(a[..., 1:], b[..., 1:]) < etol, (l, rel(a[..., 1:], b[..., 1:]))
    ev1.close()
    ev2.close()


@pytest.mark.parametrize("engine", ["f16", "tf32"])
@pytest.mark.parametrize("n,depth,p,lam", [(64, 4, 10, 1), (128, 6, 8, 3), (32, 4, 13, 1),
                                           (64, 5, 12, 3)])
def test_m2l_order_split(n, depth, p, lam, engine, monkeypatch):
    """Order-split tcgen05 M2L (the default, VFMM_M2L_SPLIT = 6): terms whose
    local and multipole degrees are both below 6 keep the 3-product split, the rest run
    hi x hi alone.  Far field against the full split and against SIMT FP32: u and dgamma/dt
    within 2e-6 of the full split (measured <= 5e-7) and within the tc-vs-SIMT bound 5e-6;
    the local expansions' rows of degree < 6 within 5e-5 of the full split (they also take
    the hi x hi terms of multipole degree >= 6: 1.9e-5 measured at level 2 of 128^3)."""
    f = synthgen.isotropic(n, seed=21)
    monkeypatch.setenv("VFMM_M2L", engine)
    out = {}
    for sp in ("6", "full"):
        monkeypatch.setenv("VFMM_M2L_SPLIT", sp)
        out[sp] = run(f, p=p, depth=depth, image_levels=lam, mode=vf.MODE_FAR_ONLY)
    monkeypatch.setenv("VFMM_M2L", "simt")
    vs, ss, evs = run(f, p=p, depth=depth, image_levels=lam, mode=vf.MODE_FAR_ONLY)
    (v6, s6, ev6), (vfu, sfu, evf) = out["6"], out["full"]
    print(f"order split {engine} n={n} L={depth} p={p} lam={lam}: vs full u {rel(v6, vfu):.2e} "
          f"sdot {rel(s6, sfu):.2e}; vs simt u {rel(v6, vs):.2e} sdot {rel(s6, ss):.2e}")
    assert rel(v6, vfu) < 2e-6 and rel(s6, sfu) < 2e-6, (rel(v6, vfu), rel(s6, sfu))
    assert rel(v6, vs) < 5e-6 and rel(s6, ss) < 5e-6, (rel(v6, vs), rel(s6, ss))
    for l in range(2, depth + 1):
        a, b = ev6.debug_expansions(1, l)[..., 1:36], evf.debug_expansions(1, l)[..., 1:36]
        assert rel(a, b) < 5e-5, (l, rel(a, b))
    for e in (ev6, evf, evs):
        e.close()
