"""Fit the division-free upper-normal-tail approximation of the fused kernel (mc_device.cuh normal_tail,
round 2):

    q = Phi(-x) = 2^E(m),   m = min(|a|, A),   a = x sqrt(log2(e)/2)  (the kernel's pre-scaled argument),

E a degree-9 polynomial in m (the exponent log2 q itself, -a^2 included) fitted by iteratively reweighted
least squares (Lawson) towards the minimax error of log2 q on [0, A], A = 5 (x <= 5.887, q(A) = 2.0e-9:
ten stages stay below half the kernel's 2^-23 fixed-point step).  DEG = 11 gives the 3.6e-8 fit (-DMC_PHI_DEG=11).
One MUFU (EX2) per call,
no reciprocal: the Numerical-Recipes t = 1/(1 + kappa x) form of round 1 needed RCP + EX2.
Prints the coefficients (highest degree first) for powers of m, the max relative error of q in exact
arithmetic, and in fp32 (numpy float32 emulation of the Horner chain) for x <= 4 and x <= 5.887.

    python tools/fit_normal_tail_ex2.py
"""
import numpy as np
from scipy.special import log_ndtr

S = np.sqrt(np.log2(np.e) / 2.0)
DEG, A = 9, 5.0


def fit():
    n = 8000
    j = np.arange(n)
    a = A / 2 * (1 - np.cos(np.pi * (j + 0.5) / n))
    y = log_ndtr(-a / S) / np.log(2.0)
    V = np.vander(a / A, DEG + 1)
    w = np.ones(n)
    for _ in range(80):
        c, *_ = np.linalg.lstsq(V * w[:, None], y * w, rcond=None)
        e = np.abs(V @ c - y)
        w = w * np.sqrt(e / e.max() + 1e-5)
        w /= w.max()
    return c / A ** np.arange(DEG, -1, -1)        # powers of m


def check(c, xmax):
    f = np.float32
    x = np.linspace(0.0, xmax, 300001)
    m = (x * S).astype(f)
    p = f(c[0])
    for ci in c[1:]:
        p = (p * m + f(ci)).astype(f)
    q = np.exp2(p.astype(np.float64)).astype(f).astype(np.float64)
    ref = np.exp(log_ndtr(-m.astype(np.float64) / S))
    exact = np.exp2(np.polyval(c, m.astype(np.float64)))
    return np.max(np.abs(q / ref - 1.0)), np.max(np.abs(exact / ref - 1.0))


if __name__ == "__main__":
    c = fit()
    print("A =", A, " q(A) = %.3e" % np.exp(log_ndtr(-A / S)))
    print("coef (m^%d .. m^0) =" % DEG, [float(v) for v in c])
    for xm in (4.0, A / S):
        f32, ex = check(c, xm)
        print("x <= %.3f: max rel err fp32 %.2e, exact %.2e" % (xm, f32, ex))
