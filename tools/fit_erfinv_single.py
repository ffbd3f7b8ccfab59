"""Fit the single-polynomial inverse-normal kernel used by the fused kernel (mc_device.cuh
normal_quantile_fast): erfinv(y) = y * g(w), w = -ln(1 - y^2) = -ln(4 p (1-p)), for w in [0, 16]
(p in [1.1e-7, 1 - 1.1e-7]), as ONE degree-12 polynomial in s = sqrt(w + 2) - (sqrt2 + sqrt18)/2,
fitted by iteratively reweighted least squares towards the minimax relative error.  Replaces the
central/tail pair of M. Giles' single-precision erfinv (two polynomials and a select per coefficient),
which cost the ALU pipe ten FSELs per call.  Beyond w = 16 the kernel clamps the argument (R24).

Prints the coefficients (highest degree first, pre-multiplied by sqrt(2) so that
Phi^{-1}(p) = g'(w) (p - (1 - p))) and the max relative error of an fp32 Horner evaluation.
"""
import numpy as np
from scipy.special import erfinv

C = 2.0
W = 16.0
DEG = 12
A, B = np.sqrt(C), np.sqrt(W + C)
MID = (A + B) / 2


def g_of_w(w):
    y = np.sqrt(-np.expm1(-w))
    return np.where(w > 1e-12, erfinv(y) / np.where(y > 0, y, 1.0), np.sqrt(np.pi) / 2)


def fit():
    n = 6000
    k = np.arange(n)
    s = MID + (B - A) / 2 * np.cos(np.pi * (k + 0.5) / n)
    y = g_of_w(s * s - C)
    V = np.vander(s - MID, DEG + 1)
    wt = np.ones(n)
    for _ in range(60):
        co, *_ = np.linalg.lstsq(V * (wt / y)[:, None], wt, rcond=None)
        e = np.abs(V @ co / y - 1)
        wt = wt * np.sqrt(e / e.max() + 1e-4)
        wt /= wt.max()
    return co * np.sqrt(2.0)


def check(co):
    ss = np.linspace(A, B, 200001)
    f = np.float32
    x = (ss - MID).astype(f)
    p = f(co[0])
    for c in co[1:]:
        p = (p * x + f(c)).astype(f)
    return np.max(np.abs(p / (np.sqrt(2.0) * g_of_w(ss * ss - C)) - 1))


if __name__ == "__main__":
    co = fit()
    print("mid =", repr(float(MID)))
    print("coef (s^12 .. s^0, x sqrt2) =", [float(c) for c in co])
    print("max rel err (fp32 Horner) = %.2e" % check(co))
