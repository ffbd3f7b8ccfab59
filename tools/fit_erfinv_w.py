"""Fit the square-root-free standard normal quantile of the fused kernel (mc_device.cuh
normal_quantile_fast, round 2):

    Phi^{-1}(p) = g(t) (p - pc),   t = w/8 - 1 in [-1, 1],   w = -ln(4 p pc) in [0, 16],   pc = 1 - p,

g a degree-12 polynomial in t (14 with -DMC_QUANT_DEG=14) (sqrt(2) erfinv(y)/y with y = 2p - 1, y^2 = 1 - e^-w, is analytic in w on
[0, 16]) fitted by iteratively reweighted least squares towards the minimax relative error.  The kernel
forms t = lg2(p pc) (-ln2/8) + (-ln4/8 - 1) in one FFMA after MUFU.LG2 and clamps t <= 1 (reading R24);
round 1 used a degree-12 polynomial in sqrt(w + 2), i.e. one MUFU.SQRT more per call.
Prints the coefficients (highest degree first) and the max relative error (exact arithmetic, and fp32
emulation for |Phi^{-1}(p)| > 0.05 with accurate (p, pc) pairs).

    python tools/fit_erfinv_w.py
"""
import numpy as np
from scipy.special import erfinv, ndtri

DEG, W = 12, 16.0


def target(w):
    y = np.sqrt(-np.expm1(-w))
    return np.where(w < 1e-300, np.sqrt(np.pi) / 2, erfinv(y) / np.where(y == 0, 1, y)) * np.sqrt(2.0)


def fit():
    n = 8000
    j = np.arange(n)
    w = W / 2 * (1 - np.cos(np.pi * (j + 0.5) / n))
    y = target(w)
    V = np.vander(w / W * 2 - 1, DEG + 1)
    wt = np.ones(n)
    for _ in range(80):
        c, *_ = np.linalg.lstsq(V * wt[:, None], y * wt, rcond=None)
        e = np.abs(V @ c - y) / y
        wt = wt * np.sqrt(e / e.max() + 1e-5)
        wt /= wt.max()
    return c


def check(c):
    f = np.float32
    pl = np.logspace(np.log10(2.9e-8), np.log10(0.5), 200000).astype(f)
    worst = 0.0
    for lower in (True, False):
        small, big = pl, (f(1) - pl).astype(f)
        p, pc = (small, big) if lower else (big, small)
        L = np.log2((p * pc).astype(f).astype(np.float64)).astype(f)
        t = np.minimum((L * f(-np.log(2) / 8) + f(-np.log(4) / 8 - 1)).astype(f), f(1.0))
        g = f(c[0])
        for ci in c[1:]:
            g = (g * t + f(ci)).astype(f)
        x = (g * (p - pc).astype(f)).astype(np.float64)
        ref = ndtri(small.astype(np.float64)) * (1 if lower else -1)
        ok = np.abs(ref) > 0.05
        worst = max(worst, np.abs(x[ok] / ref[ok] - 1).max())
    ww = np.linspace(0, W, 100001)
    exact = np.abs(np.polyval(c, ww / 8 - 1) / target(ww) - 1).max()
    return worst, exact


if __name__ == "__main__":
    c = fit()
    print("coef (t^%d .. t^0) =" % DEG, [float(v) for v in c])
    f32, ex = check(c)
    print("max rel err: fp32 %.2e, exact %.2e" % (f32, ex))
