"""TEST INFRASTRUCTURE ONLY -- forward-Euler time step of the vortex particle method on the
direct-sum oracle O1 (parity reference for vfmm_step; never imported by the product).

PAPER.md section 2 (lines 67-111): the vorticity equation is integrated by updating three
separate variables simultaneously --
  convection   dx_i/dt      = u_i                        Eq. (7)
  stretching   dgamma_i/dt  = sum_j grad(gamma_j x grad G g_sigma) . gamma_i   Eq. (8), :100
  diffusion    dsigma^2/dt  = 2 nu  (core spreading)      Eq. (9)
with forward Euler.  u and dgamma/dt come from ``oracle.direct`` (O1, float64).
Positions are wrapped back into the periodic box [lo, lo + len) (image_levels > 0).
"""
from __future__ import annotations

import numpy as np

from . import direct


def euler_step(pos, gamma, sigma, nu, dt, box_lo, box_len, image_levels=3, scheme=0,
               batched=True):
    """One step from (pos, gamma, sigma) -> (pos', gamma', sigma', u, dgamma), float64.

    pos, gamma: (3, N).  All three updates use the state at the start of the step
    (simultaneous).  sigma' = sqrt(sigma^2 + 2 nu dt) (Eq. 9)."""
    pos = np.asarray(pos, np.float64)
    gamma = np.asarray(gamma, np.float64)
    u, dg = direct(pos, gamma, sigma, box_lo, box_len, image_levels, scheme, batched=batched)
    x = pos + dt * u                                     # Eq. (7)
    if image_levels > 0:
        x = box_lo + np.mod(x - box_lo, box_len)         # periodic box
    g = gamma + dt * dg                                  # Eq. (8)
    s = float(np.sqrt(sigma * sigma + 2.0 * nu * dt))    # Eq. (9)
    return x, g, s, u, dg
