"""NEXT-2: reinitialization by RBF interpolation on the device (vfmm_reinit; PAPER.md:113-114,
:191, :272-277) against the plain definition in oracle/rbf.py (Gaussian sums of Eq. 3 over the
image cube, the RBF system solved exactly by dense LU)."""
import math

import numpy as np
import pytest

import synthgen
from oracle import rbf

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1110_2921_b200 as vf  # noqa: E402

DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(DEV)


def test_reinit_jittered_particles_onto_the_lattice():
    """Old particles: a 16^3 isotropic field moved off the lattice (jitter +-0.75 h) with a core
    grown by spreading (sigma_old = 1.25 h); new particles: the cell centres, sigma_new = h
    (PAPER.md:191).  omega at the new points (Eq. 3) and the interpolated strengths match the
    dense solve of the oracle."""
    n = 16
    f0 = synthgen.isotropic(n, seed=13)
    old = synthgen.jitter(f0, 0.75, seed=9)
    h = f0.box_len / n
    s_old, s_new = float(np.float32(1.25 * h)), float(np.float32(h))
    ev = vf.Evaluator(p=4, depth=2, image_levels=1, sigma=s_old, box_lo=f0.box_lo,
                      box_len=f0.box_len)
    g_o, om_o = rbf.reinit(old.pos, old.gamma, s_old, f0.pos, s_new, f0.box_len)
    A = rbf.rbf_matrix(f0.pos, s_new, f0.box_len)
    x0 = om_o * (f0.box_len ** 3 / n ** 3)          # the paper's initial guess
    r0 = np.linalg.norm(om_o - x0 @ A.T, axis=1)
    for tol in (1e-3, 1e-5):
        g, om, info = ev.reinit(_t(old.pos), _t(old.gamma), s_old, _t(f0.pos), s_new, tol=tol,
                                max_iter=400, restart=60)
        g = g.cpu().numpy().astype(np.float64)
        om = om.cpu().numpy().astype(np.float64)
        res = np.linalg.norm(om_o - g @ A.T, axis=1) / r0   # true residual, dense matrix
        e_om, e_g = rel(om, om_o), rel(g, g_o)
        print(f"reinit 16^3 tol {tol:g}: omega {e_om:.2e}, true residual {res.max():.2e} "
              f"(GMRES {max(info['rel_residual']):.2e}), gamma vs dense solve {e_g:.2e}, "
              f"{info['iterations']} iterations, ws {info['ws_old']}/{info['ws_new']}, "
              f"{info['ms']:.2f} ms")
        assert info["converged"] == 1
        assert e_om < 2e-6, e_om
        # the exit test holds for the true (float64, untruncated) residual too, up to the
        # FP32 floor of the matrix-vector products (~1e-6 of omega)
        assert res.max() < 1.5 * tol + 2e-5, res
    # at the tight tolerance the strengths approach the exact solve; the RBF matrix's highest
    # lattice modes are damped by up to e^{-3 pi^2 / 2} (condition ~1e5), which GMRES only
    # resolves as far as the residual asks
    assert e_g < 1e-2, e_g
    assert ev.params.sigma == pytest.approx(s_new)
    ev.close()


def test_reinit_fourier_mode_closed_form():
    """omega = sin(k.x) on the 32^3 lattice: the interpolated strengths are
    h^3 e^{|k|^2 h^2 / 2} sin(k.x_j) (oracle pin test_rbf_oracle_fourier_mode_closed_form);
    the paper's initial guess omega h^3 converges in a few iterations."""
    n = 32
    f = synthgen.taylor_green(n)
    x = f.pos.astype(np.float64)
    h = f.box_len / n
    k = np.array([2.0, -1.0, 1.0])
    mode = np.sin(k @ x)
    damp = math.exp(-0.5 * (k @ k) * f.sigma ** 2)
    # old particles = the lattice itself carrying the exact solution at sigma_old = h: then
    # omega(x_i) = sin(k.x_i) (up to aliasing) and the new strengths reproduce them
    g_true = np.stack([mode, -mode, 0.5 * mode]) * h ** 3 / damp
    ev = vf.Evaluator(p=4, depth=3, image_levels=1, sigma=f.sigma, box_lo=f.box_lo,
                      box_len=f.box_len)
    g, om, info = ev.reinit(_t(f.pos), _t(g_true), f.sigma, _t(f.pos), f.sigma, tol=1e-4)
    g = g.cpu().numpy()
    om = om.cpu().numpy()
    print(f"fourier mode: {info['iterations']} iterations, gamma {rel(g, g_true):.2e}")
    assert rel(om, np.stack([mode, -mode, 0.5 * mode])) < 1e-5
    assert rel(g, g_true) < 1e-4
    assert info["iterations"] <= 10  # "converges in 5-10 iterations"
    ev.close()
