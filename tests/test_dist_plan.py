"""Host-side logic of the multi-GPU path (Morton partition + LET exchange plans), on CPU.

* every (receiver, sender) pair agrees on the message contents (each rank's receive list from
  q equals q's send list to it) -- checked across 2 real processes over torch.distributed gloo;
* coverage: owned cells + received cells contain every source a rank's targets need
  (27 neighbours for P2P at the leaf level, the 189-cell interaction list for M2L at
  levels >= 2), recomputed here independently by brute force; nothing received is owned.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1110_2921_b200 as vf


def _enc(x, y, z, l):
    k = 0
    for b in range(l):
        k |= ((x >> b) & 1) << (3 * b) | ((y >> b) & 1) << (3 * b + 1) | ((z >> b) & 1) << (3 * b + 2)
    return k


def _dec(k, l):
    x = y = z = 0
    for b in range(l):
        x |= ((k >> (3 * b)) & 1) << b
        y |= ((k >> (3 * b + 1)) & 1) << b
        z |= ((k >> (3 * b + 2)) & 1) << b
    return x, y, z


def _needed(level, R, r, periodic, kind):
    side, ncell = 1 << level, 1 << (3 * level)
    per = ncell // R
    need = set()
    for t in range(r * per, (r + 1) * per):
        tx, ty, tz = _dec(t, level)
        if kind == 0:
            cand = [(tx + a, ty + b, tz + c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)]
        else:
            px, py, pz = tx >> 1, ty >> 1, tz >> 1
            cand = [(sx, sy, sz) for sx in range(2 * px - 2, 2 * px + 4)
                    for sy in range(2 * py - 2, 2 * py + 4) for sz in range(2 * pz - 2, 2 * pz + 4)
                    if max(abs(sx - tx), abs(sy - ty), abs(sz - tz)) > 1]
        for sx, sy, sz in cand:
            if not periodic and not (0 <= sx < side and 0 <= sy < side and 0 <= sz < side):
                continue
            need.add(_enc(sx % side, sy % side, sz % side, level))
    return {s for s in need if s // per != r}


@pytest.mark.parametrize("depth,R,periodic", [(3, 2, 1), (3, 4, 1), (3, 8, 0), (4, 8, 1)])
def test_plan_covers_needs(depth, R, periodic):
    for r in range(R):
        for kind, level in [(0, depth)] + [(l, l) for l in range(2, depth + 1)]:
            got = set()
            for q in range(R):
                ids = vf.dist_plan(depth, R, r, periodic, kind, 0, q)
                per = (1 << (3 * level)) // R
                assert all(int(i) // per == q for i in ids)  # received from its owner
                assert q != r or len(ids) == 0
                got |= set(int(i) for i in ids)
            assert got == _needed(level, R, r, periodic, 1 if kind else 0), (r, kind)


def _worker(rank, world, port, depth, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = True
    for kind in [0] + list(range(2, depth + 1)):
        sends = [vf.dist_plan(depth, world, rank, 1, kind, 1, q).tolist() for q in range(world)]
        recvs = [vf.dist_plan(depth, world, rank, 1, kind, 0, q).tolist() for q in range(world)]
        gathered = [None] * world
        dist.all_gather_object(gathered, sends)  # gathered[q][r] = what q sends to r
        for q in range(world):
            ok &= gathered[q][rank] == recvs[q]
    # owned leaf ranges tile the tree
    lo, hi = vf.partition(depth, world, rank)
    rng = [None] * world
    dist.all_gather_object(rng, (lo, hi))
    ok &= rng[0][0] == 0 and rng[-1][1] == 1 << (3 * depth)
    ok &= all(rng[i][1] == rng[i + 1][0] for i in range(world - 1))
    out[rank] = bool(ok)
    dist.destroy_process_group()


def test_plans_agree_across_processes_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, 3, out), nprocs=2, join=True)
    assert out[0] and out[1]


def test_partition_and_route_counts():
    lo, hi = vf.partition(4, 8, 3)
    assert (lo, hi) == (3 * 512, 4 * 512)
    with pytest.raises(vf.VfmmError):
        vf.partition(4, 3, 0)
    lo_, ln = float(np.float32(-np.pi)), float(np.float32(2 * np.pi))
    pos = np.array([[-3.0, 3.0, 3.0], [-3.0, 3.0, -3.0], [-3.0, 3.0, -3.0]], np.float32)
    c, st = vf.route_counts(pos, 2, 8, lo_, ln)
    assert st == vf.VFMM_OK
    # octant of each point: x fastest in the Morton bits -> (0,0,0) rank 0, (1,1,1) rank 7,
    # (1,0,0) rank 1
    assert c.tolist() == [1, 1, 0, 0, 0, 0, 0, 1]
    pos[1, 0] = np.float32(lo_ + ln)  # upper face: outside the half-open box
    _, st = vf.route_counts(pos, 2, 8, lo_, ln)
    assert st == vf.VFMM_EDOMAIN


def _route_worker(rank, world, port, out):
    """Each process holds arbitrary particles; the send counts (vfmm_route_counts) of every
    rank, all-gathered over gloo, form the C1 count matrix: column sums are what each owner
    evaluates, and they equal an independent count by brute-force octant membership."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(100 + rank)
    n = 3000 + 777 * rank
    lo_, ln = float(np.float32(-np.pi)), float(np.float32(2 * np.pi))
    pos = rng.uniform(lo_, lo_ + ln, (3, n)).astype(np.float32)
    pos = np.minimum(pos, np.nextafter(np.float32(lo_ + ln), np.float32(0)))
    depth, R = 3, 4
    cnt, st = vf.route_counts(pos, depth, R, lo_, ln)
    rows = [torch.zeros(R, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(rows, torch.from_numpy(cnt))
    mat = torch.stack(rows)
    allpos = [None] * world
    dist.all_gather_object(allpos, pos)
    ok = st == vf.VFMM_OK and int(mat[rank].sum()) == n
    # brute force: rank R's range at depth 3 with R = 4 is two level-1 octants, i.e. the top
    # Morton bits (z1, y1) of the particle's octant = rank (x fastest, so octant = x + 2y + 4z)
    for q in range(R):
        want = 0
        for P_ in allpos:
            ix = np.floor((P_ - np.float32(lo_)) * np.float32(8 / ln)).astype(int).clip(0, 7)
            octant = (ix[0] >> 2) + 2 * (ix[1] >> 2) + 4 * (ix[2] >> 2)
            want += int(np.sum(octant // 2 == q))
        ok &= int(mat[:, q].sum()) == want
    out[rank] = bool(ok)
    dist.destroy_process_group()


def test_route_counts_across_processes_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_route_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] and out[1]
