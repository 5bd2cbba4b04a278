"""Distributed FMM (Morton partition + halo particles + LET multipoles) validated on one GPU:
R logical ranks run every phase in lockstep with device-copy exchanges (the NCCL transport
moves the same buffers); the assembled result must equal the single-rank evaluation."""
import numpy as np
import pytest

import synthgen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1110_2921_b200 as vf  # noqa: E402

DEV = torch.device("cuda:0")


def _split(f, depth, R):
    leaf = vf.leaf_of(f.pos, depth, f.box_lo, f.box_len)
    per = (1 << (3 * depth)) // R
    return [np.nonzero(leaf // per == r)[0] for r in range(R)]


@pytest.mark.parametrize("R,n,depth,p,lam,jit", [
    (1, 32, 3, 6, 3, False), (2, 32, 3, 6, 3, False), (4, 32, 3, 6, 1, True), (8, 32, 3, 4, 0, False),
    (8, 64, 4, 6, 3, False), (2, 64, 5, 8, 3, False), (4, 48, 5, 6, 2, True)])
def test_logical_ranks_equal_single_rank(R, n, depth, p, lam, jit):
    f = synthgen.isotropic(n, seed=31)
    if jit:
        f = synthgen.jitter(f, seed=4)
    kw = dict(p=p, depth=depth, image_levels=lam, sigma=f.sigma, box_lo=f.box_lo,
              box_len=f.box_len)
    pos = torch.from_numpy(f.pos).to(DEV)
    gam = torch.from_numpy(f.gamma).to(DEV)
    ev1 = vf.Evaluator(**kw)
    v1, s1 = ev1.evaluate(pos, gam)
    ev1.sync_status()
    parts = _split(f, depth, R)
    evR = vf.Evaluator(**kw)
    pl = [torch.from_numpy(np.ascontiguousarray(f.pos[:, ix])).to(DEV) for ix in parts]
    gl = [torch.from_numpy(np.ascontiguousarray(f.gamma[:, ix])).to(DEV) for ix in parts]
    vl, sl = evR.evaluate_logical(pl, gl)
    torch.cuda.synchronize()
    V = np.zeros_like(f.pos, dtype=np.float32)
    S = np.zeros_like(f.pos, dtype=np.float32)
    for ix, v, s in zip(parts, vl, sl):
        V[:, ix] = v.cpu().numpy()
        S[:, ix] = s.cpu().numpy()
    v1, s1 = v1.cpu().numpy(), s1.cpu().numpy()
    ru = np.linalg.norm(V - v1) / np.linalg.norm(v1)
    rs = np.linalg.norm(S - s1) / np.linalg.norm(s1)
    assert ru < 1e-6 and rs < 1e-6, (ru, rs)
    st = evR.stats()
    assert (st["bytes_sent"] > 0) == (R > 1)
    ev1.close()
    evR.close()


def test_nccl_one_rank_context_equals_single_rank():
    """A one-rank NCCL communicator drives the distributed phases with the real NCCL calls
    (unique id, CommInitRank, the all-gathers of per-leaf counts and level-1 multipoles): the
    result equals the single-context evaluation."""
    try:
        uid = vf.nccl_unique_id()
    except Exception as e:  # pragma: no cover
        pytest.skip(f"NCCL unavailable: {e}")
    f = synthgen.isotropic(32, seed=5)
    kw = dict(p=6, depth=3, image_levels=3, sigma=f.sigma, box_lo=f.box_lo, box_len=f.box_len)
    pos = torch.from_numpy(f.pos).to(DEV)
    gam = torch.from_numpy(f.gamma).to(DEV)
    ev1 = vf.Evaluator(**kw)
    v1, s1 = ev1.evaluate(pos, gam)
    ev1.sync_status()
    evn = vf.Evaluator(nranks=1, rank=0, nccl_id=uid, **kw)
    vn, sn = evn.evaluate(pos, gam)
    evn.sync_status()
    torch.cuda.synchronize()
    v1, s1, vn, sn = (t.cpu().numpy() for t in (v1, s1, vn, sn))
    ru = np.linalg.norm(vn - v1) / np.linalg.norm(v1)
    rs = np.linalg.norm(sn - s1) / np.linalg.norm(s1)
    assert ru < 1e-6 and rs < 1e-6, (ru, rs)
    ev1.close()
    evn.close()


def test_particles_outside_rank_range_are_flagged():
    f = synthgen.isotropic(16, seed=2)
    parts = _split(f, 2, 2)
    ev = vf.Evaluator(p=4, depth=2, image_levels=1, sigma=f.sigma)
    swap = [parts[1], parts[0]]  # every particle handed to the wrong rank
    pl = [torch.from_numpy(np.ascontiguousarray(f.pos[:, ix])).to(DEV) for ix in swap]
    gl = [torch.from_numpy(np.ascontiguousarray(f.gamma[:, ix])).to(DEV) for ix in swap]
    with pytest.raises(vf.VfmmError) as e:
        ev.evaluate_logical(pl, gl)
    assert e.value.status == vf.VFMM_EDOMAIN
    ev.close()
