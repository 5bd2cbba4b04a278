"""B200-native periodic vortex FMM (Yokota & Barba, arXiv:1110.2921) -- Python binding.

Thin ctypes marshalling over the C ABI in ``include/vfmm.h`` (``lib/libvfmm.so``, built
from ``csrc/`` for sm_100a).  Every step of the hot path runs in the CUDA kernels of that
library; this module only passes device pointers, sizes and the current CUDA stream.
PyTorch is used for device memory and streams only.  There is no CPU fallback: if the
library is missing, importing the binding's compute entry points raises.

    ev = Evaluator(p=10, image_levels=3, sigma=h)
    vel, dgamma = ev.evaluate(pos, gamma)      # (3, N) float32 CUDA tensors, input order

Names follow the paper: positions x, vortex strengths gamma (Eq. 3), core
radius sigma (Eq. 4), velocity u (Eq. 5), stretching dgamma/dt (Eq. 8), expansion order p
(Eq. 10), periodic images.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libvfmm.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "vfmm.h")

VFMM_OK, VFMM_EINVAL, VFMM_EDOMAIN, VFMM_ENOMEM, VFMM_ECUDA, VFMM_ENCCL, VFMM_ESTATE = \
    0, -1, -2, -3, -4, -5, -6
MODE_FMM, MODE_DIRECT, MODE_NEAR_ONLY, MODE_FAR_ONLY, MODE_HYBRID = 0, 1, 2, 3, 4
STRETCH_CLASSICAL, STRETCH_TRANSPOSE = 0, 1


class VfmmError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        super().__init__(f"vfmm status {status}: {msg}")


class c_params(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int32), ("depth", ctypes.c_int32),
                ("image_levels", ctypes.c_int32), ("scheme", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("sigma", ctypes.c_float),
                ("box_lo", ctypes.c_float), ("box_len", ctypes.c_float)]


class c_stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in
                ("ms_total", "ms_keys", "ms_sort", "ms_tree", "ms_p2m", "ms_m2m", "ms_m2l",
                 "ms_l2l", "ms_l2p", "ms_p2p")] + \
               [(k, ctypes.c_int64) for k in ("n_p2p_pairs", "n_m2l", "n_m2m", "n_l2l")] + \
               [("depth_used", ctypes.c_int32), ("n_kernel_launches", ctypes.c_int32),
                ("bytes_sent", ctypes.c_int64), ("bytes_recv", ctypes.c_int64),
                ("ms_comm", ctypes.c_double), ("ms_comm_exposed", ctypes.c_double)]


_LIB = None

EXPORTS = ["vfmm_abi_version", "vfmm_params_default", "vfmm_create", "vfmm_evaluate",
           "vfmm_evaluate_host", "vfmm_sync_status", "vfmm_get_stats", "vfmm_set_params",
           "vfmm_debug_tree", "vfmm_debug_expansions", "vfmm_strerror",
           "vfmm_last_error_message", "vfmm_destroy", "vfmm_nccl_get_unique_id",
           "vfmm_create_nccl", "vfmm_partition", "vfmm_evaluate_logical", "vfmm_dist_plan",
           "vfmm_route_counts", "vfmm_step", "vfmm_evaluate_at", "vfmm_reinit",
           "vfmm_evaluate_sigma", "vfmm_evaluate_tree"]


class c_reinit_info(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("rel_residual", ctypes.c_double * 3), ("ms", ctypes.c_double),
                ("depth_used", ctypes.c_int32), ("ws_old", ctypes.c_int32),
                ("ws_new", ctypes.c_int32)]


def load_library(path: str = LIB_PATH):
    """Load libvfmm.so (raises OSError if it is missing -- there is no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise OSError(f"libvfmm.so not built: {path} (run __graft_entry__.build())")
    L = ctypes.CDLL(path)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    L.vfmm_abi_version.restype = ctypes.c_int32
    L.vfmm_params_default.argtypes = [ctypes.POINTER(c_params)]
    L.vfmm_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(c_params), i32]
    L.vfmm_evaluate.argtypes = [vp, i64, vp, vp, vp, vp, vp]
    L.vfmm_evaluate_host.argtypes = [vp, i64, vp, vp, vp, vp]
    L.vfmm_sync_status.argtypes = [vp]
    L.vfmm_get_stats.argtypes = [vp, ctypes.POINTER(c_stats)]
    L.vfmm_set_params.argtypes = [vp, ctypes.POINTER(c_params)]
    L.vfmm_debug_tree.argtypes = [vp, vp, vp, vp]
    L.vfmm_debug_expansions.argtypes = [vp, i32, i32, vp]
    L.vfmm_strerror.argtypes = [i32]
    L.vfmm_strerror.restype = ctypes.c_char_p
    L.vfmm_last_error_message.argtypes = [vp]
    L.vfmm_last_error_message.restype = ctypes.c_char_p
    L.vfmm_destroy.argtypes = [vp]
    L.vfmm_destroy.restype = None
    L.vfmm_nccl_get_unique_id.argtypes = [vp]
    L.vfmm_create_nccl.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(c_params), i32, vp, i32, i32]
    L.vfmm_partition.argtypes = [i32, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.vfmm_evaluate_logical.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp]
    L.vfmm_dist_plan.argtypes = [i32, i32, i32, i32, i32, i32, i32, vp, i64, ctypes.POINTER(i64)]
    L.vfmm_route_counts.argtypes = [i32, i32, i64, vp, ctypes.c_float, ctypes.c_float, vp]
    L.vfmm_step.argtypes = [vp, i64, vp, vp, ctypes.c_float, ctypes.c_float, vp, vp,
                            ctypes.POINTER(ctypes.c_float), vp]
    L.vfmm_step.restype = ctypes.c_int
    L.vfmm_evaluate_at.argtypes = [vp, i64, vp, vp, i64, vp, vp, vp]
    L.vfmm_evaluate_sigma.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp]
    L.vfmm_evaluate_sigma.restype = ctypes.c_int
    L.vfmm_evaluate_at.restype = ctypes.c_int
    L.vfmm_evaluate_tree.argtypes = [vp, i64, vp, vp, vp, vp, ctypes.c_float, ctypes.c_int32, vp]
    L.vfmm_evaluate_tree.restype = ctypes.c_int
    L.vfmm_reinit.argtypes = [vp, i64, vp, vp, ctypes.c_float, i64, vp, ctypes.c_float,
                              ctypes.c_float, ctypes.c_int32, ctypes.c_int32, vp, vp,
                              ctypes.POINTER(c_reinit_info), vp]
    L.vfmm_reinit.restype = ctypes.c_int
    for f in ("vfmm_nccl_get_unique_id", "vfmm_create_nccl", "vfmm_partition",
              "vfmm_evaluate_logical", "vfmm_dist_plan", "vfmm_route_counts"):
        getattr(L, f).restype = ctypes.c_int
    for f in ("vfmm_create", "vfmm_evaluate", "vfmm_evaluate_host", "vfmm_sync_status",
              "vfmm_get_stats", "vfmm_set_params", "vfmm_debug_tree", "vfmm_debug_expansions"):
        getattr(L, f).restype = ctypes.c_int
    _LIB = L
    return L


@dataclass
class Params:
    p: int = 10
    depth: int = 0
    image_levels: int = 3
    scheme: int = STRETCH_CLASSICAL
    mode: int = MODE_FMM
    sigma: float = 2.0 * math.pi / 256.0
    box_lo: float = float(np.float32(-math.pi))
    box_len: float = float(np.float32(2.0 * math.pi))

    def to_c(self) -> c_params:
        return c_params(self.p, self.depth, self.image_levels, self.scheme, self.mode,
                        self.sigma, self.box_lo, self.box_len)


def _check(L, ctx, st):
    if st != VFMM_OK:
        msg = L.vfmm_strerror(st).decode()
        if ctx:
            extra = L.vfmm_last_error_message(ctx)
            if extra:
                msg += " -- " + extra.decode()
        raise VfmmError(st, msg)


def partition(depth: int, nranks: int, rank: int):
    """Owned Morton leaf range [lo, hi) of `rank` (C ABI vfmm_partition)."""
    L = load_library()
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(L, None, L.vfmm_partition(depth, nranks, rank, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def route_counts(pos, depth: int, nranks: int, box_lo: float, box_len: float):
    """Host routing of the redistribution (C ABI vfmm_route_counts): how many of these (3, n)
    float32 host positions each rank's Morton range receives.  Returns (counts, status)."""
    L = load_library()
    pos = np.ascontiguousarray(pos, np.float32)
    out = np.zeros(nranks, np.int64)
    st = L.vfmm_route_counts(depth, nranks, pos.shape[1], pos.ctypes.data, box_lo, box_len,
                             out.ctypes.data)
    if st not in (VFMM_OK, VFMM_EDOMAIN):
        _check(L, None, st)
    return out, st


def dist_plan(depth, nranks, rank, periodic, kind, direction, peer):
    """Static exchange plan (host only): list of leaf/cell ids (see vfmm_dist_plan)."""
    L = load_library()
    cnt = ctypes.c_int64()
    _check(L, None, L.vfmm_dist_plan(depth, nranks, rank, periodic, kind, direction, peer, None,
                                     0, ctypes.byref(cnt)))
    out = np.zeros(cnt.value, np.int32)
    _check(L, None, L.vfmm_dist_plan(depth, nranks, rank, periodic, kind, direction, peer,
                                     out.ctypes.data, cnt.value, ctypes.byref(cnt)))
    return out


def nccl_unique_id() -> bytes:
    L = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(L, None, L.vfmm_nccl_get_unique_id(buf))
    return buf.raw


class Evaluator:
    """One vfmm context on one CUDA device (not thread-safe).

    Distributed (one process per GPU): pass nranks, rank and the 128-byte NCCL unique id
    (rank 0's nccl_unique_id(), broadcast by the caller, e.g. torch.distributed) -- see
    init_distributed().  An NCCL context runs the distributed phases even with nranks = 1."""

    def __init__(self, device: int | None = None, nranks: int = 1, rank: int = 0,
                 nccl_id: bytes | None = None, **kw):
        import torch

        self._L = load_library()
        self.params = Params(**kw)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._ctx = ctypes.c_void_p()
        prm = self.params.to_c()
        self.nranks, self.rank = nranks, rank
        if nranks > 1 or nccl_id is not None:  # NCCL context (also 1 rank: distributed path)
            idb = ctypes.create_string_buffer(nccl_id, 128)
            _check(self._L, None, self._L.vfmm_create_nccl(
                ctypes.byref(self._ctx), ctypes.byref(prm), self.device, idb, nranks, rank))
        else:
            _check(self._L, None, self._L.vfmm_create(ctypes.byref(self._ctx),
                                                       ctypes.byref(prm), self.device))
        self._n = 0

    # -- parameters -------------------------------------------------------------------
    def set_params(self, **kw):
        for k, v in kw.items():
            setattr(self.params, k, v)
        prm = self.params.to_c()
        _check(self._L, self._ctx, self._L.vfmm_set_params(self._ctx, ctypes.byref(prm)))

    # -- evaluation ---------------------------------------------------------------------
    def evaluate_into(self, pos, gamma, vel, dgamma, stream=None):
        """pos, gamma, vel, dgamma: contiguous float32 CUDA tensors of shape (3, N)."""
        import torch

        for t in (pos, gamma, vel, dgamma):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
                    and t.dim() == 2 and t.shape[0] == 3):
                raise ValueError("expected contiguous float32 CUDA tensors of shape (3, N)")
        n = pos.shape[1]
        if stream is None:
            stream = torch.cuda.current_stream(pos.device)
        _check(self._L, self._ctx, self._L.vfmm_evaluate(
            self._ctx, n, pos.data_ptr(), gamma.data_ptr(), vel.data_ptr(), dgamma.data_ptr(),
            ctypes.c_void_p(stream.cuda_stream)))
        self._n = n
        return vel, dgamma

    def evaluate_sigma(self, pos, gamma, sigma, stream=None):
        """Per-particle core radii sigma ((N,) float32 CUDA tensor, Eq. 6's sigma_j) in the near
        field -- C ABI vfmm_evaluate_sigma; the context's sigma must be >= max sigma."""
        import torch

        if not (sigma.is_cuda and sigma.dtype == torch.float32 and sigma.is_contiguous()
                and sigma.dim() == 1 and sigma.shape[0] == pos.shape[1]):
            raise ValueError("sigma: contiguous float32 CUDA tensor of shape (N,)")
        vel = torch.empty_like(pos)
        dg = torch.empty_like(pos)
        if stream is None:
            stream = torch.cuda.current_stream(pos.device)
        _check(self._L, self._ctx, self._L.vfmm_evaluate_sigma(
            self._ctx, pos.shape[1], pos.data_ptr(), gamma.data_ptr(), sigma.data_ptr(),
            vel.data_ptr(), dg.data_ptr(), ctypes.c_void_p(stream.cuda_stream)))
        self._n = pos.shape[1]
        return vel, dg

    def evaluate(self, pos, gamma, stream=None):
        import torch

        vel = torch.empty_like(pos)
        dg = torch.empty_like(pos)
        return self.evaluate_into(pos, gamma, vel, dg, stream)

    def evaluate_tree(self, pos, gamma, theta: float = 0.5, n_crit: int = 64, stream=None):
        """Hybrid treecode, cell-particle traversal (C ABI vfmm_evaluate_tree):
        adaptive leaves of <= n_crit particles, multipole acceptance r_S + r_B < theta d."""
        import torch

        for t in (pos, gamma):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
                    and t.dim() == 2 and t.shape[0] == 3):
                raise ValueError("expected contiguous float32 CUDA tensors of shape (3, N)")
        vel = torch.empty_like(pos)
        dg = torch.empty_like(pos)
        if stream is None:
            stream = torch.cuda.current_stream(pos.device)
        _check(self._L, self._ctx, self._L.vfmm_evaluate_tree(
            self._ctx, pos.shape[1], pos.data_ptr(), gamma.data_ptr(), vel.data_ptr(),
            dg.data_ptr(), ctypes.c_float(theta), int(n_crit), ctypes.c_void_p(stream.cuda_stream)))
        self._n = pos.shape[1]
        return vel, dg

    def evaluate_at(self, pos, gamma, tpos, stream=None):
        """Velocity at target points tpos ((3, T) float32 CUDA tensor) induced by the particles
        (pos, gamma) -- C ABI vfmm_evaluate_at (targets enter the tree with zero strength)."""
        import torch

        for t in (pos, gamma, tpos):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
                    and t.dim() == 2 and t.shape[0] == 3):
                raise ValueError("expected contiguous float32 CUDA tensors of shape (3, N)")
        tvel = torch.empty_like(tpos)
        if stream is None:
            stream = torch.cuda.current_stream(pos.device)
        _check(self._L, self._ctx, self._L.vfmm_evaluate_at(
            self._ctx, pos.shape[1], pos.data_ptr(), gamma.data_ptr(), tpos.shape[1],
            tpos.data_ptr(), tvel.data_ptr(), ctypes.c_void_p(stream.cuda_stream)))
        self._n = pos.shape[1] + tpos.shape[1]
        return tvel

    def reinit(self, pos_old, gamma_old, sigma_old: float, pos_new, sigma_new: float,
               tol: float = 1e-5, max_iter: int = 50, restart: int = 30, stream=None):
        """RBF reinitialization onto new particles (C ABI vfmm_reinit):
        returns (gamma_new, omega_new, info dict); the context's sigma becomes sigma_new."""
        import torch

        for t in (pos_old, gamma_old, pos_new):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
                    and t.dim() == 2 and t.shape[0] == 3):
                raise ValueError("expected contiguous float32 CUDA tensors of shape (3, N)")
        g = torch.empty_like(pos_new)
        om = torch.empty_like(pos_new)
        info = c_reinit_info()
        if stream is None:
            stream = torch.cuda.current_stream(pos_new.device)
        _check(self._L, self._ctx, self._L.vfmm_reinit(
            self._ctx, pos_old.shape[1], pos_old.data_ptr(), gamma_old.data_ptr(),
            float(sigma_old), pos_new.shape[1], pos_new.data_ptr(), float(sigma_new), float(tol),
            int(max_iter), int(restart), g.data_ptr(), om.data_ptr(), ctypes.byref(info),
            ctypes.c_void_p(stream.cuda_stream)))
        self.params.sigma = float(sigma_new)
        d = {k: getattr(info, k) for k, _ in c_reinit_info._fields_}
        d["rel_residual"] = list(info.rel_residual)
        return g, om, d

    def step(self, pos, gamma, dt: float, nu: float = 0.0, vel=None, dgamma=None, stream=None):
        """One forward-Euler step of the vortex method (C ABI vfmm_step, PAPER.md:67, :91,
        :100, :107, :114): pos and gamma ((3, N) float32 CUDA tensors) are updated in place,
        the core radius sigma grows by core spreading (sigma^2 += 2 nu dt).  Returns the
        (vel, dgamma) evaluated at the start of the step."""
        import torch

        for t in (pos, gamma):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
                    and t.dim() == 2 and t.shape[0] == 3):
                raise ValueError("expected contiguous float32 CUDA tensors of shape (3, N)")
        vel = torch.empty_like(pos) if vel is None else vel
        dgamma = torch.empty_like(pos) if dgamma is None else dgamma
        if stream is None:
            stream = torch.cuda.current_stream(pos.device)
        sig = ctypes.c_float()
        _check(self._L, self._ctx, self._L.vfmm_step(
            self._ctx, pos.shape[1], pos.data_ptr(), gamma.data_ptr(), float(dt), float(nu),
            vel.data_ptr(), dgamma.data_ptr(), ctypes.byref(sig),
            ctypes.c_void_p(stream.cuda_stream)))
        self.params.sigma = sig.value
        self._n = pos.shape[1]
        return vel, dgamma

    def evaluate_host(self, pos, gamma):
        """Host (numpy) in/out: H2D copy, evaluate, D2H copy inside the library."""
        pos = np.ascontiguousarray(pos, np.float32)
        gamma = np.ascontiguousarray(gamma, np.float32)
        n = pos.shape[1]
        vel = np.empty_like(pos)
        dg = np.empty_like(pos)
        _check(self._L, self._ctx, self._L.vfmm_evaluate_host(
            self._ctx, n, pos.ctypes.data, gamma.ctypes.data, vel.ctypes.data, dg.ctypes.data))
        self._n = n
        return vel, dg

    def evaluate_host_ptr(self, n, pos_ptr, gamma_ptr, vel_ptr, dg_ptr):
        _check(self._L, self._ctx, self._L.vfmm_evaluate_host(
            self._ctx, n, pos_ptr, gamma_ptr, vel_ptr, dg_ptr))

    def evaluate_logical(self, pos_list, gamma_list, stream=None):
        """Distributed algorithm with len(pos_list) logical ranks on this one GPU (tests):
        pos_list[r], gamma_list[r]: (3, n_r) float32 CUDA tensors, anywhere in the box (n_r may
        be 0).  Returns per-rank (vel, dgamma) lists in each rank's input order."""
        import torch

        R = len(pos_list)
        vel = [torch.empty_like(p) for p in pos_list]
        dg = [torch.empty_like(p) for p in pos_list]
        n = (ctypes.c_int64 * R)(*[p.shape[1] for p in pos_list])
        P = lambda ts: (ctypes.c_void_p * R)(*[t.data_ptr() for t in ts])
        if stream is None:
            stream = torch.cuda.current_stream(pos_list[0].device)
        _check(self._L, self._ctx, self._L.vfmm_evaluate_logical(
            self._ctx, R, n, P(pos_list), P(gamma_list), P(vel), P(dg),
            ctypes.c_void_p(stream.cuda_stream)))
        return vel, dg

    def sync_status(self):
        _check(self._L, self._ctx, self._L.vfmm_sync_status(self._ctx))

    def stats(self) -> dict:
        s = c_stats()
        _check(self._L, self._ctx, self._L.vfmm_get_stats(self._ctx, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in c_stats._fields_}

    # -- debug --------------------------------------------------------------------------
    def debug_tree(self, depth: int):
        n = self._n
        keys = np.zeros(n, np.uint32)
        perm = np.zeros(n, np.uint32)
        ls = np.zeros((1 << (3 * depth)) + 1, np.int32)
        _check(self._L, self._ctx, self._L.vfmm_debug_tree(
            self._ctx, keys.ctypes.data, perm.ctypes.data, ls.ctypes.data))
        return keys, perm, ls

    def debug_expansions(self, kind: int, level: int):
        nc = (self.params.p + 1) ** 2
        out = np.zeros((1 << (3 * level), 3, nc), np.float32)
        _check(self._L, self._ctx, self._L.vfmm_debug_expansions(self._ctx, kind, level,
                                                                  out.ctypes.data))
        return out

    def close(self):
        if self._ctx:
            self._L.vfmm_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_distributed(**kw):
    """Create an Evaluator for this torch.distributed rank (one process per GPU): rank 0 makes
    the NCCL unique id, torch.distributed broadcasts it, every rank joins the communicator."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Evaluator(device=torch.cuda.current_device(), nranks=world, rank=rank,
                     nccl_id=obj[0], **kw)


def evaluate(pos, gamma, sigma, p=10, depth=0, image_levels=3, scheme=0, mode=MODE_FMM,
             box_lo=None, box_len=None):
    """One-shot convenience wrapper around Evaluator."""
    kw = dict(p=p, depth=depth, image_levels=image_levels, scheme=scheme, mode=mode,
              sigma=float(sigma))
    if box_lo is not None:
        kw["box_lo"] = float(box_lo)
    if box_len is not None:
        kw["box_len"] = float(box_len)
    ev = Evaluator(**kw)
    try:
        return ev.evaluate(pos, gamma)
    finally:
        ev.close()
