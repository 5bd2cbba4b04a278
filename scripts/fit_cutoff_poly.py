"""CUDA-side constant generator (product, not oracle): FP32 polynomial for the Gaussian
cutoff tail used by the P2P kernel (paper_1110_2921_b200/csrc/p2p.cu).

PAPER.md:86, Eq. (6): g = erf(rho) - (2/sqrt(pi)) rho exp(-rho^2).  Write
1 - g = exp(-rho^2) * (erfcx(rho) + 2 rho / sqrt(pi)) and fit erfcx(rho) as a polynomial of degree DEG (default 4)
polynomial in t = 1/(1 + rho/2), weighted for relative accuracy of g over rho in [0.5, 10]
(the closed form is used for rho^2 >= 1/4; beyond rho = 10 the exp(-rho^2) factor is 0 in
FP32), with iteratively reweighted least squares towards the minimax fit: max relative error
in g 4.8e-7 in exact arithmetic at degree 4 (degree 5: 1.6e-8, degree 7: 1.2e-10), below the
1.4e-6 floor that FP32 evaluation reaches near rho = 0.5 at any degree (rounding of t and the
cancellation 1 - (1 - g)).  Degree 4 (round 2) saves one FFMA2 per pair of the P2P.
    python scripts/fit_cutoff_poly.py [degree]
Prints the coefficients (ascending in t) scaled by 1/(4 pi), as pasted into p2p.cu.
"""
import sys

import numpy as np
import numpy.polynomial.polynomial as P
from scipy.special import erf, erfcx

DEG = int(sys.argv[1]) if len(sys.argv) > 1 else 4
x = np.linspace(0.5, 10.0, 400001).astype(np.float32).astype(np.float64)
t = 1.0 / (1.0 + x / 2.0)
g = erf(x) - 2.0 / np.sqrt(np.pi) * x * np.exp(-x * x)
w = np.exp(-x * x) / g
ww = w.copy()
for _ in range(40):
    c = P.polyfit(t, erfcx(x), DEG, w=ww)
    err = np.abs(P.polyval(t, c) - erfcx(x)) * w
    ww = ww * (1 + err / err.max()) ** 2
print("max relative error in g:", err.max())
print(", ".join("%.9ef" % (v / (4 * np.pi)) for v in c))
