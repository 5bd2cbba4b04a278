"""Distributed FMM (redistribution + Morton partition + halo particles + LET multipoles)
validated on one GPU: R logical ranks run every phase in lockstep with device-copy exchanges
(the NCCL transport moves the same buffers).  Each rank passes arbitrary particles (anywhere in
the box); the per-rank results must equal the single-rank evaluation of the rank-order
concatenation of the inputs."""
import numpy as np
import pytest

import synthgen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1110_2921_b200 as vf  # noqa: E402

DEV = torch.device("cuda:0")


def _split(n_total, R, seed=0, empty_rank=None):
    """Arbitrary per-rank inputs: a random permutation of the particles cut into R chunks of
    random sizes (rank `empty_rank` gets none).  Returns index arrays; the global input order
    of the distributed evaluation is their concatenation in rank order."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n_total)
    cuts = np.sort(rng.integers(0, n_total, R - 1)) if R > 1 else np.array([], np.int64)
    parts = np.split(perm, cuts)
    if empty_rank is not None and R > 1:
        other = (empty_rank + 1) % R
        parts[other] = np.concatenate([parts[other], parts[empty_rank]])
        parts[empty_rank] = parts[empty_rank][:0]
    return parts


@pytest.mark.parametrize("R,n,depth,p,lam,jit", [
    (1, 32, 3, 6, 3, False), (2, 32, 3, 6, 3, False), (4, 32, 3, 6, 1, True), (8, 32, 3, 4, 0, False),
    (8, 64, 4, 6, 3, False), (2, 64, 5, 8, 3, False), (4, 48, 5, 6, 2, True)])
def test_logical_ranks_equal_single_rank(R, n, depth, p, lam, jit):
    f = synthgen.isotropic(n, seed=31)
    if jit:
        f = synthgen.jitter(f, seed=4)
    kw = dict(p=p, depth=depth, image_levels=lam, sigma=f.sigma, box_lo=f.box_lo,
              box_len=f.box_len)
    ev1 = vf.Evaluator(**kw)
    parts = _split(f.pos.shape[1], R, seed=R + depth, empty_rank=1 if R >= 4 else None)
    order = np.concatenate(parts)
    # single-rank reference on the concatenated input order
    pos = torch.from_numpy(np.ascontiguousarray(f.pos[:, order])).to(DEV)
    gam = torch.from_numpy(np.ascontiguousarray(f.gamma[:, order])).to(DEV)
    v1, s1 = ev1.evaluate(pos, gam)
    ev1.sync_status()
    evR = vf.Evaluator(**kw)
    pl = [torch.from_numpy(np.ascontiguousarray(f.pos[:, ix])).to(DEV) for ix in parts]
    gl = [torch.from_numpy(np.ascontiguousarray(f.gamma[:, ix])).to(DEV) for ix in parts]
    vl, sl = evR.evaluate_logical(pl, gl)
    torch.cuda.synchronize()
    V = np.concatenate([v.cpu().numpy() for v in vl], axis=1)
    S = np.concatenate([s.cpu().numpy() for s in sl], axis=1)
    v1, s1 = v1.cpu().numpy(), s1.cpu().numpy()
    ru = np.linalg.norm(V - v1) / np.linalg.norm(v1)
    rs = np.linalg.norm(S - s1) / np.linalg.norm(s1)
    print(f"R={R} n={n} depth={depth}: u {ru:.2e} sdot {rs:.2e}, bitwise "
          f"{np.array_equal(V, v1) and np.array_equal(S, s1)}")
    assert ru < 1e-6 and rs < 1e-6, (ru, rs)
    st = evR.stats()
    assert (st["bytes_sent"] > 0) == (R > 1)
    assert st["ms_comm"] > 0 and st["ms_comm_exposed"] == st["ms_comm"]
    # a second evaluation with other per-rank sizes reuses the rank states (same R)
    parts2 = _split(f.pos.shape[1], R, seed=99)
    pl = [torch.from_numpy(np.ascontiguousarray(f.pos[:, ix])).to(DEV) for ix in parts2]
    gl = [torch.from_numpy(np.ascontiguousarray(f.gamma[:, ix])).to(DEV) for ix in parts2]
    vl, _ = evR.evaluate_logical(pl, gl)
    V2 = np.zeros_like(f.pos)
    for ix, v in zip(parts2, vl):
        V2[:, ix] = v.cpu().numpy()
    V1 = np.zeros_like(f.pos)
    V1[:, order] = v1
    assert np.linalg.norm(V2 - V1) / np.linalg.norm(V1) < 1e-6
    ev1.close()
    evR.close()


def test_logical_rank_count_change_on_one_context():
    """the same context evaluated with R = 8, then R = 2, then R = 4 logical ranks
    (rank state buffers sized for the first R must not be overrun by a later, larger range)."""
    f = synthgen.isotropic(32, seed=8)
    kw = dict(p=6, depth=3, image_levels=2, sigma=f.sigma, box_lo=f.box_lo, box_len=f.box_len)
    ev1 = vf.Evaluator(**kw)
    pos = torch.from_numpy(f.pos).to(DEV)
    gam = torch.from_numpy(f.gamma).to(DEV)
    v1, _ = ev1.evaluate(pos, gam)
    v1 = v1.cpu().numpy()
    evR = vf.Evaluator(**kw)
    for R in (8, 2, 4, 1):
        parts = np.array_split(np.arange(f.pos.shape[1]), R)
        pl = [pos[:, ix[0]:ix[-1] + 1].contiguous() for ix in parts]
        gl = [gam[:, ix[0]:ix[-1] + 1].contiguous() for ix in parts]
        vl, _ = evR.evaluate_logical(pl, gl)
        V = np.concatenate([v.cpu().numpy() for v in vl], axis=1)
        assert np.linalg.norm(V - v1) / np.linalg.norm(v1) < 1e-6, R
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


def test_particles_outside_the_box_are_flagged():
    f = synthgen.isotropic(16, seed=2)
    parts = _split(f.pos.shape[1], 2)
    ev = vf.Evaluator(p=4, depth=2, image_levels=1, sigma=f.sigma)
    pos = f.pos.copy()
    pos[0, parts[1][3]] = np.float32(f.box_lo + f.box_len)  # the upper face is outside
    pl = [torch.from_numpy(np.ascontiguousarray(pos[:, ix])).to(DEV) for ix in parts]
    gl = [torch.from_numpy(np.ascontiguousarray(f.gamma[:, ix])).to(DEV) for ix in parts]
    with pytest.raises(vf.VfmmError) as e:
        ev.evaluate_logical(pl, gl)
    assert e.value.status == vf.VFMM_EDOMAIN
    ev.close()
