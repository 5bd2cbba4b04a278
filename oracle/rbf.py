"""TEST INFRASTRUCTURE ONLY -- reinitialization by RBF interpolation, plain definition
(parity reference for vfmm_reinit; never imported by the product).

PAPER.md:113-114: "RBF interpolation is obtained by solving a linear system for Equation (3),
with gamma as the unknown vector and omega as the right-hand side"; new particles
at the cell centres with sigma = h; initial guess gamma_j ~ omega_i (dx)^3.

  zeta_sigma(r) = (2 pi sigma^2)^{-3/2} exp(-r^2 / (2 sigma^2))          Eq. (4)
  omega(x_i)    = sum_n sum_j gamma_j zeta_sigma(x_i - x_j - n len)       Eq. (3)
  A_ij          = sum_n zeta_sigma_new(x_i - x_j - n len),   A gamma' = omega(x_new)

The image sum runs over the 27 nearest images (image_levels = 1): every image left out is at
least one box length (>= 15 sigma here) away.  The system is solved exactly (dense LU) --
the product's GMRES and neighbour-list truncation (reading R18) are approximations of it.
"""
from __future__ import annotations

import math

import numpy as np


def zeta(r2, sigma):
    """Gaussian core, Eq. (4), as a function of r^2."""
    return (2.0 * math.pi * sigma * sigma) ** -1.5 * np.exp(-r2 / (2.0 * sigma * sigma))


def gaussian_sum(x_tgt, x_src, w_src, sigma, box_len, periodic=True, chunk=512):
    """out[:, i] = sum_n sum_j w_src[:, j] zeta(|x_tgt_i - x_src_j - n len|^2)  (Eq. 3).
    x_tgt (3, T), x_src (3, S), w_src (3, S); float64."""
    xt = np.asarray(x_tgt, np.float64)
    xs = np.asarray(x_src, np.float64)
    ws = np.asarray(w_src, np.float64)
    imgs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)] if periodic \
        else [(0, 0, 0)]
    out = np.zeros((3, xt.shape[1]))
    for t0 in range(0, xt.shape[1], chunk):
        t = xt[:, t0:t0 + chunk]
        acc = np.zeros((3, t.shape[1]))
        for n in imgs:
            d = t[:, :, None] - xs[:, None, :] - np.array(n, np.float64)[:, None, None] * box_len
            k = zeta((d * d).sum(0), sigma)          # (T, S)
            acc += ws @ k.T
        out[:, t0:t0 + chunk] = acc
    return out


def rbf_matrix(x, sigma, box_len, periodic=True):
    """Dense A_ij = sum_n zeta_sigma(x_i - x_j - n len) (N x N)."""
    x = np.asarray(x, np.float64)
    imgs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)] if periodic \
        else [(0, 0, 0)]
    A = np.zeros((x.shape[1], x.shape[1]))
    for n in imgs:
        d = x[:, :, None] - x[:, None, :] - np.array(n, np.float64)[:, None, None] * box_len
        A += zeta((d * d).sum(0), sigma)
    return A


def reinit(x_old, g_old, sigma_old, x_new, sigma_new, box_len, periodic=True):
    """(gamma_new, omega_new): omega at the new points from the old particles (Eq. 3), then
    the RBF system A gamma_new = omega solved exactly, per component."""
    om = gaussian_sum(x_new, x_old, g_old, sigma_old, box_len, periodic)
    A = rbf_matrix(x_new, sigma_new, box_len, periodic)
    g = np.linalg.solve(A, om.T).T
    return g, om
