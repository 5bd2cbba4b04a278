"""CUDA-side constant generator (product, not oracle): FP32 polynomial for the Gaussian
cutoff tail used by the P2P kernel (paper_1110_2921_b200/csrc/p2p.cu).

PAPER.md:86, Eq. (6): g = erf(rho) - (2/sqrt(pi)) rho exp(-rho^2).  Write
1 - g = exp(-rho^2) * (erfcx(rho) + 2 rho / sqrt(pi)) and fit erfcx(rho) as a degree-7
polynomial in (t - 1/2), t = 1/(1 + rho/2), weighted least squares over rho in [0.5, 8]
for relative accuracy of g.  Prints the coefficients pasted into p2p.cu.
"""
import numpy as np
import numpy.polynomial.polynomial as P
from scipy.special import erf, erfcx

x = np.linspace(0.5, 8.0, 200001)
t = 1.0 / (1.0 + x / 2.0)
g = erf(x) - 2.0 / np.sqrt(np.pi) * x * np.exp(-x * x)
w = np.exp(-x * x) / g
c = P.polyfit(t - 0.5, erfcx(x), 7, w=w)
print(", ".join("%.9ef" % v for v in c))
# p2p.cu folds 1/(4 pi) into the coefficients: (1/4pi)(1 - g) = e (E/4pi + rho 2/(4 pi sqrt(pi)))
print(", ".join("%.9ef" % (v / (4 * np.pi)) for v in c))
