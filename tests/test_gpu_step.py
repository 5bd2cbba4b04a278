"""NEXT-1: forward-Euler time stepping on the device (vfmm_step; Eq. 7,
:100 Eq. 8, :107 Eq. 9, :114) against the oracle's Euler step on the direct sum O1
(oracle/euler.py): K steps from the same initial state, compared on the displacement
x_K - x_0 (periodic) and the strength change gamma_K - gamma_0; the core radius follows
sigma^2 + 2 nu t (core spreading)."""
import math

import numpy as np
import pytest

import synthgen
from oracle.euler import euler_step
import tolerances as TOL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1110_2921_b200 as vf  # noqa: E402

DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def _periodic_disp(x1, x0, L):
    d = np.asarray(x1, np.float64) - np.asarray(x0, np.float64)
    return d - L * np.round(d / L)


@pytest.mark.parametrize("mode,p,tol", [("direct", 2, (2e-5, 2e-5)), ("fmm", 10, None)])
def test_steps_match_oracle_euler(mode, p, tol):
    f = synthgen.isotropic(16, seed=17)
    lam, dt, nu, K = 1, 0.02, 0.005, 3
    m = vf.MODE_DIRECT if mode == "direct" else vf.MODE_FMM
    ev = vf.Evaluator(p=p, depth=2, image_levels=lam, mode=m, sigma=f.sigma, box_lo=f.box_lo,
                      box_len=f.box_len)
    pos = torch.from_numpy(f.pos.copy()).to(DEV)
    gam = torch.from_numpy(f.gamma.copy()).to(DEV)
    x, g, s = f.pos.astype(np.float64), f.gamma.astype(np.float64), f.sigma
    for k in range(K):
        ev.step(pos, gam, dt, nu)
        x, g, s, _, _ = euler_step(x, g, s, nu, dt, f.box_lo, f.box_len, lam)
        ev.sync_status()
        assert ev.params.sigma == pytest.approx(s, rel=1e-6)
    xg = pos.cpu().numpy()
    gg = gam.cpu().numpy()
    assert np.all(xg >= np.float32(f.box_lo)) and np.all(xg < np.float32(f.box_lo + f.box_len))
    d_gpu = _periodic_disp(xg, f.pos, f.box_len)
    d_ora = _periodic_disp(x, f.pos, f.box_len)
    eu = rel(d_gpu, d_ora)
    eg = rel(gg.astype(np.float64) - f.gamma, g - f.gamma)
    print(f"{mode} p={p}: {K} steps: displacement {eu:.2e}, strength change {eg:.2e}")
    tu, tg = tol if tol else TOL.FMM_VS_DIRECT[p]
    assert eu < tu and eg < tg, (eu, eg)
    assert ev.params.sigma == pytest.approx(math.sqrt(f.sigma ** 2 + 2 * nu * dt * K), rel=1e-6)
    ev.close()


def test_step_wraps_across_the_periodic_face():
    """A particle next to the upper face moving outward re-enters at the lower face."""
    f = synthgen.isotropic(8, seed=3)
    ev = vf.Evaluator(p=4, depth=1, image_levels=1, sigma=f.sigma, box_lo=f.box_lo,
                      box_len=f.box_len)
    pos = torch.from_numpy(f.pos.copy()).to(DEV)
    gam = torch.from_numpy(f.gamma.copy()).to(DEV)
    v, _ = ev.evaluate(pos, gam)
    v = v.cpu().numpy()
    i = int(np.argmax(v[0]))
    # put particle i just below the upper x face and step so that it crosses it
    pos[0, i] = float(np.nextafter(np.float32(f.box_lo + f.box_len), np.float32(0)))
    v2, _ = ev.evaluate(pos, gam)
    u = float(v2[0, i].item())
    assert u > 0
    dt = 0.25 * f.box_len / 8 / u
    ev.step(pos, gam, dt)
    xi = float(pos[0, i].item())
    assert f.box_lo <= xi < f.box_lo + 0.5 * f.box_len / 8 + abs(u) * dt
    assert float(pos.min()) >= np.float32(f.box_lo)
    assert float(pos.max()) < np.float32(f.box_lo + f.box_len)
    ev.close()
