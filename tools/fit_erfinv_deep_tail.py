"""Fit the deep-tail polynomial used by the fp32 inverse normal CDF in the CUDA kernel
(paper_2005_10494_b200/csrc/mc_device.cuh, normal_quantile()).

Region: w = -ln(4 p (1-p)) in [16, 88] (p < 1.1e-7), t = sqrt(w).  Fits
g(t) = erfinv(y)/y, y = 2p - 1, as a degree-6 polynomial in (t - 6) by relative least squares
on Chebyshev nodes.  Max relative error of the fp32 Horner evaluation: ~5.6e-7.
Central (w < 5) and near-tail (5 <= w < 16) regions use M. Giles, "Approximating the erfinv
function", GPU Computing Gems Jade Edition (2011), single-precision coefficients.
"""
import numpy as np
from scipy.special import ndtri


def target(t):
    w = t * t
    ew = np.exp(-w)
    p = ew / (2 * (1 + np.sqrt(1 - ew)))
    return ndtri(p) / np.sqrt(2) / (2 * p - 1)


def fit(deg=6, a=4.0, b=np.sqrt(88.0)):
    k = np.arange(2000)
    t = (a + b) / 2 + (b - a) / 2 * np.cos(np.pi * (k + 0.5) / 2000)
    g = target(t)
    V = np.vander(t - 6.0, deg + 1)
    coef, *_ = np.linalg.lstsq(V / g[:, None], np.ones_like(g), rcond=None)
    return np.float32(coef)


if __name__ == "__main__":
    print([float(c) for c in fit()])
