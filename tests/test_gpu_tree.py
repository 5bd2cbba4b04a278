"""NEXT-4: the hybrid treecode's cell-particle traversal (vfmm_evaluate_tree)
on the B200 against (a) the float64 treecode oracle running the same algorithm
(oracle/treecode_ref.py: same adaptive leaves, same MAC, same M2P / P2P split -- only FP32
rounding separates them) and (b) the direct-sum oracle O1 (the definition the traversal
approximates), on clustered fields with leaves at several levels, leaves larger than a warp,
both stretching schemes, free space, 3^3 and 27^3 images."""
import numpy as np
import pytest

import oracle
import synthgen
import tolerances as TOL
from oracle import treecode_ref as T

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1110_2921_b200 as vf  # noqa: E402

DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def run_tree(f, p, depth, lam, theta, ncrit, scheme=0):
    ev = vf.Evaluator(p=p, depth=depth, image_levels=lam, scheme=scheme, sigma=f.sigma,
                      box_lo=f.box_lo, box_len=f.box_len)
    pos = torch.from_numpy(f.pos).to(DEV)
    gam = torch.from_numpy(f.gamma).to(DEV)
    v, s = ev.evaluate_tree(pos, gam, theta, ncrit)
    ev.sync_status()
    st = ev.stats()
    out = v.cpu().numpy().astype(np.float64), s.cpu().numpy().astype(np.float64), st
    ev.close()
    return out


@pytest.mark.parametrize("lam,scheme,p", [(1, 0, 10), (3, 0, 10), (0, 0, 8), (1, 1, 10),
                                          (3, 0, 6)])
def test_tree_vs_tree_oracle_and_direct(lam, scheme, p):
    f = synthgen.clustered(600)
    v, s, st = run_tree(f, p, 4, lam, 0.5, 16, scheme)
    vo, so, info = T.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 4, p, 0.5, 16,
                              image_levels=lam, scheme=scheme, return_info=True)
    vd, sd = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, lam, scheme)
    ev_u, ev_s = rel(v, vo), rel(s, so)
    ed_u, ed_s = rel(v, vd), rel(s, sd)
    print(f"tree lam={lam} scheme={scheme} p={p}: vs tree oracle u {ev_u:.2e} s {ev_s:.2e}; "
          f"vs O1 u {ed_u:.2e} s {ed_s:.2e}; m2p {st['n_m2l']} pairs {st['n_p2p_pairs']}")
    # same algorithm in FP32 vs float64
    assert ev_u < TOL.FMM_VS_FMM_ORACLE[0] and ev_s < TOL.FMM_VS_FMM_ORACLE[1], (ev_u, ev_s)
    # same interaction lists
    assert st["n_m2l"] == info["n_m2p"] and st["n_p2p_pairs"] == info["n_pairs"]
    # the approximation: p = 10, theta = 0.5 is below the oracle's own 1e-6 (plus FP32)
    bound = 1e-5 if p >= 8 else 1e-4
    assert ed_u < bound and ed_s < bound, (ed_u, ed_s)


def test_theta_zero_is_the_direct_sum():
    f = synthgen.clustered(800, seed=7)
    v, s, st = run_tree(f, 4, 4, 1, 0.0, 16)
    vd, sd = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 1, 0)
    print(f"tree theta=0: u {rel(v, vd):.2e} s {rel(s, sd):.2e}")
    assert st["n_m2l"] == 0 and st["n_p2p_pairs"] == 27 * 800 * 800
    # every target sums 27 x 800 = 21600 terms in FP32 sequence (the DIRECT mode sums its image
    # partials in double): the long-list bound of the dense-leaf P2P test applies (measured
    # 2.5e-6 / 6.8e-6 on the B200)
    assert rel(v, vd) < TOL.NEAR_VS_ORACLE_DENSE[0] and rel(s, sd) < TOL.NEAR_VS_ORACLE_DENSE[1]


def test_dense_leaves_and_coincident_particles():
    """Two tight clusters: level-L leaves with hundreds of particles (target chunks and source
    loops longer than a warp) and distinct coincident particles (the r -> 0 limits, R7)."""
    f = synthgen.with_coincident(synthgen.clustered(1500, n_clusters=2, spread=0.15, seed=3))
    v, s, st = run_tree(f, 10, 3, 1, 0.5, 32)
    vo, so = T.evaluate(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 3, 10, 0.5, 32,
                        image_levels=1)
    print(f"tree dense: u {rel(v, vo):.2e} s {rel(s, so):.2e}")
    assert rel(v, vo) < TOL.FMM_VS_FMM_ORACLE[0] and rel(s, so) < TOL.FMM_VS_FMM_ORACLE[1]


def test_lattice_field_vs_direct_sum_at_27_cubed():
    """The benchmark's field family (a jittered isotropic lattice) at 27^3 images."""
    f = synthgen.jitter(synthgen.isotropic(32, seed=5))
    v, s, st = run_tree(f, 10, 3, 3, 0.5, 64)
    tg = synthgen.sample_targets(f.pos.shape[1], 64, n_lattice=32)
    vd, sd = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, 3, 0, targets=tg)
    e_u, e_s = rel(v[:, tg], vd), rel(s[:, tg], sd)
    print(f"tree lattice 32^3 lam=3: u {e_u:.2e} s {e_s:.2e}; m2p {st['n_m2l']}")
    assert e_u < TOL.FMM_VS_DIRECT[10][0] and e_s < TOL.FMM_VS_DIRECT[10][1], (e_u, e_s)


def test_tree_rejects_bad_arguments():
    f = synthgen.clustered(100)
    ev = vf.Evaluator(p=4, depth=3, image_levels=1, sigma=f.sigma, box_lo=f.box_lo,
                      box_len=f.box_len)
    pos = torch.from_numpy(f.pos).to(DEV)
    gam = torch.from_numpy(f.gamma).to(DEV)
    for th, nc in ((1.0, 16), (-0.1, 16), (0.5, 0)):
        with pytest.raises(vf.VfmmError):
            ev.evaluate_tree(pos, gam, th, nc)
    ev.close()


@pytest.mark.parametrize("field", ["lattice", "clustered"])
def test_hybrid_mode_picks_one_candidate_and_reuses_it(field):
    """VFMM_MODE_HYBRID (PAPER.md:150-152 auto-tuning): the result is bitwise the FMM's or the
    treecode's (theta 0.5, n_crit 32 / 64 / 128); on the uniform lattice the FMM is cheapest."""
    f = synthgen.make("c2") if field == "lattice" else synthgen.clustered(20000, seed=9)
    kw = dict(p=8, depth=0, image_levels=3, sigma=f.sigma, box_lo=f.box_lo, box_len=f.box_len)
    pos = torch.from_numpy(f.pos).to(DEV)
    gam = torch.from_numpy(f.gamma).to(DEV)
    ref = vf.Evaluator(**kw)
    cands = {"fmm": ref.evaluate(pos, gam)}
    for nc in (32, 64, 128):
        cands[f"tree{nc}"] = ref.evaluate_tree(pos, gam, 0.5, nc)
    torch.cuda.synchronize()
    ev = vf.Evaluator(mode=vf.MODE_HYBRID, **kw)
    v1, s1 = ev.evaluate(pos, gam)
    v2, s2 = ev.evaluate(pos, gam)  # the cached choice
    torch.cuda.synchronize()
    chosen = [k for k, (v, s) in cands.items() if torch.equal(v1, v) and torch.equal(s1, s)]
    print(f"hybrid {field}: chose {chosen}")
    assert chosen
    assert torch.equal(v1, v2) and torch.equal(s1, s2)
    if field == "lattice":
        assert "fmm" in chosen
    ev.close()
    ref.close()
