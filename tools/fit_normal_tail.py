"""Fit the fp32 upper-normal-tail approximation used by the fused kernel (mc_device.cuh normal_tail):

    q = Phi(-a) = t * 2^(P(t) - a^2 log2(e) / 2),   t = 1 / (1 + kappa a),   a >= 0,

P a degree-8 polynomial in t (9 coefficients) fitted by iteratively reweighted least squares
(Lawson) towards the minimax error of log2(q) on a in [0, 21] (q >= 1e-98; below, q underflows fp32
anyway).  This is the Numerical-Recipes erfc form (Press et al., "erfcc") refitted in base 2 with one
coefficient fewer.  Prints kappa, the coefficients (highest degree first) and the max relative error
of q evaluated in fp32 with MUFU-like ex2/rcp (numpy float32 emulation).
"""
import numpy as np
from scipy.special import log_ndtr

KAPPA = 0.4 / np.sqrt(2.0)
DEG = 8
AMAX = 21.0


def target(t):
    a = (1.0 / t - 1.0) / KAPPA
    return (log_ndtr(-a) - np.log(t)) / np.log(2.0) + a * a / (2.0 * np.log(2.0))


def fit():
    t_lo = 1.0 / (1.0 + KAPPA * AMAX)
    n = 6000
    j = np.arange(n)
    t = (t_lo + 1) / 2 + (1 - t_lo) / 2 * np.cos(np.pi * (j + 0.5) / n)
    y = target(t)
    V = np.vander(t, DEG + 1)
    w = np.ones(n)
    for _ in range(60):
        c, *_ = np.linalg.lstsq(V * w[:, None], y * w, rcond=None)
        e = np.abs(V @ c - y)
        w = w * np.sqrt(e / e.max() + 1e-4)
        w /= w.max()
    return c


def check(c):
    a = np.linspace(0.0, 11.0, 400001)          # q > 2e-28: fp32 normal range
    f = np.float32
    t = (f(1.0) / (f(1.0) + f(KAPPA) * a.astype(f))).astype(f)
    p = f(c[0])
    for ci in c[1:]:
        p = (p * t + f(ci)).astype(f)
    e = (p + (a.astype(f) * a.astype(f)) * f(-0.5 / np.log(2.0))).astype(f)
    q = (t * np.exp2(e.astype(np.float64)).astype(f)).astype(np.float64)
    ref = np.exp(log_ndtr(-a))
    return np.max(np.abs(q / ref - 1.0))


if __name__ == "__main__":
    c = fit()
    print("kappa =", repr(float(KAPPA)))
    print("coef (t^8 .. t^0) =", [float(x) for x in c])
    print("max rel err (fp32 emulation, a in [0,11]) = %.2e" % check(c))
