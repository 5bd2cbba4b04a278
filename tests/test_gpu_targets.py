"""NEXT-3: velocity at points that are not particles (vfmm_evaluate_at; PAPER.md:152 'targets',
:215 lattice velocity for the spectra) against O1 in probe mode (targets != sources)."""
import numpy as np
import pytest

import oracle
import synthgen
import tolerances as TOL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1110_2921_b200 as vf  # noqa: E402

DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def _targets(f, shift=(0.5, 1 / 3, 0.25)):
    """The particle lattice shifted by a fraction of a cell (re-wrapped): a second lattice of
    points between the particles, as for velocities on an interleaved grid."""
    h = f.box_len / f.n
    t = f.pos.astype(np.float64) + np.array(shift)[:, None] * h
    t = f.box_lo + np.mod(t - f.box_lo, f.box_len)
    t = t.astype(np.float32)
    return np.where(t >= np.float32(f.box_lo + f.box_len), np.float32(f.box_lo), t)


@pytest.mark.parametrize("mode,p,lam", [("direct", 2, 1), ("fmm", 10, 1), ("fmm", 8, 3)])
def test_velocity_at_targets_vs_oracle(mode, p, lam):
    f = synthgen.isotropic(16, seed=19)
    tpos = _targets(f)
    m = vf.MODE_DIRECT if mode == "direct" else vf.MODE_FMM
    ev = vf.Evaluator(p=p, depth=2, image_levels=lam, mode=m, sigma=f.sigma, box_lo=f.box_lo,
                      box_len=f.box_len)
    pos = torch.from_numpy(f.pos).to(DEV)
    gam = torch.from_numpy(f.gamma).to(DEV)
    tv = ev.evaluate_at(pos, gam, torch.from_numpy(tpos).to(DEV))
    ev.sync_status()
    tv = tv.cpu().numpy().astype(np.float64)
    sel = np.arange(0, tpos.shape[1], 7)
    vo, _ = oracle.direct(f.pos, f.gamma, f.sigma, f.box_lo, f.box_len, lam, 0,
                          probe_pos=tpos[:, sel].astype(np.float64),
                          probe_gamma=np.zeros((3, len(sel))), batched=True)
    e = rel(tv[:, sel], vo)
    print(f"targets {mode} p={p} lam={lam}: u {e:.2e}")
    tol = TOL.DIRECT_VS_ORACLE[0] if mode == "direct" else TOL.FMM_VS_DIRECT[p][0]
    assert e < tol, e
    tv2 = ev.evaluate_at(pos, gam, torch.from_numpy(tpos[:, :0].copy()).to(DEV))  # no targets
    assert tv2.shape == (3, 0)
    ev.close()
