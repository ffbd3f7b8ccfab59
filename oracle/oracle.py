"""CPU ORACLE for arXiv 2005.10494 — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this module.  The product package
``paper_2005_10494_b200`` never imports it and shares no code with it.

Plain fp64: the Monte-Carlo estimator, Philox, the MVN orthant and the alpha grid
are in ``oracle.c`` (ctypes); problem setup (Formula 10, Eq. 9), the closed-form
assurance, thin-plate-spline smoothing with GCV and the argmax are numpy below.
``P:n`` cites /root/reference/PAPER.md line n; ``R#`` are the readings in DESIGN.md §3.

Parity unpinned: none — every function is pinned in tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MAXN = 10
GL_NODES = 20   # Gauss-Legendre points per panel of the MVN orthant quadrature (numpy leggauss)


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, no fast-math: IEEE fp64 semantics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-D_DEFAULT_SOURCE", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        d, i32, i64, u32, u64 = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
        P = ctypes.POINTER
        L.or_philox4x32_10.argtypes = [P(u32), P(u32), P(u32)]
        L.or_word.argtypes = [u64, u32, u64]
        L.or_word.restype = u32
        L.or_Phi.argtypes = [d]; L.or_Phi.restype = d
        L.or_Phi_inv.argtypes = [d]; L.or_Phi_inv.restype = d
        L.or_threshold.argtypes = [d]; L.or_threshold.restype = d
        L.or_cholesky.argtypes = [i32, P(d), P(d)]; L.or_cholesky.restype = i32
        L.or_null_corr.argtypes = [i32, P(d), P(d)]
        L.or_record_uniforms.argtypes = [i32, i32, i32]; L.or_record_uniforms.restype = i32
        L.or_record_words.argtypes = [i32]; L.or_record_words.restype = i32
        L.or_record_field.argtypes = [u64, u32, u32, u64, i32, i32]; L.or_record_field.restype = u32
        L.or_word_tagged.argtypes = [u64, u32, u32, u64]
        L.or_word_tagged.restype = u32
        L.or_draw.argtypes = [i32, i32, P(d), d, P(d), P(d), P(d), i32, u64, u32, u32, u64,
                              P(d), P(d), P(d), P(d)]
        L.or_draw.restype = d
        L.or_design_sums.argtypes = [i32, i32, P(d), d, P(d), P(d), P(d), i32, u64, u32, u32, u64, u64, P(i64)]
        L.or_mvn_orthant.argtypes = [i32, P(d), P(d)]; L.or_mvn_orthant.restype = d
        L.or_fwer.argtypes = [i32, P(d), P(d)]; L.or_fwer.restype = d
        L.or_solve_alpha_n.argtypes = [i32, P(d), d, P(d), d, P(d)]; L.or_solve_alpha_n.restype = i32
        L.or_alpha_grid.argtypes = [i32, P(d), d, i32, d, P(d), P(ctypes.c_uint8)]
        L.or_alpha_grid.restype = i64
        L.or_subset.argtypes = [i64, i64, u64, P(i64)]
        L.or_design_sums_crossed.argtypes = [i32, P(d), d, P(d), P(d), P(d), u64, u32, u64, u64, P(i64)]
        L.or_draw_strata.argtypes = [d, d, P(d), P(d), i32, u64, u32, u32, u64, P(d), P(d), P(d), P(d)]
        L.or_draw_strata.restype = d
        L.or_design_sums_strata.argtypes = [d, d, P(d), P(d), i32, u64, u32, u32, u64, u64, P(i64)]
        L.or_set_gauss_legendre.argtypes = [i32, P(d), P(d)]; L.or_set_gauss_legendre.restype = i32
        # the orthant quadrature's rule: numpy's 20-point Gauss-Legendre nodes and weights (a library
        # routine; oracle.c computes none of its own)
        gx, gw = np.polynomial.legendre.leggauss(GL_NODES)
        if L.or_set_gauss_legendre(GL_NODES, _dp(gx), _dp(gw)) != 0:
            raise RuntimeError("or_set_gauss_legendre rejected the rule")
        _lib = L
    return _lib


def _dp(a):
    return np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# --------------------------------------------------------------------------------------
# Random stream

def philox4x32_10(ctr, key):
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (ctypes.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return [int(x) for x in o]


def word(seed: int, design: int, w: int) -> int:
    return int(lib().or_word(seed, design, w))


def word_tagged(seed: int, ident: int, tag: int, w: int) -> int:
    """Word w of stream (id, tag): lane w mod 4 of the block with counter (q_lo, q_hi, id, tag)."""
    return int(lib().or_word_tagged(seed, ident, tag, w))


def record_uniforms(n: int, p: int, est: int) -> int:
    """Uniforms per record: COND sample pairs 2p + 2(n/2), IND single samples 2 ceil((p+n)/2)."""
    return int(lib().or_record_uniforms(n, p, est))


def record_words(n: int, p: int, est: int) -> int:
    """Words per record: 2 ceil(23 U / 64) for U record uniforms when that is fewer than U (packed), else U
    (DESIGN.md §2.2)."""
    return int(lib().or_record_words(record_uniforms(n, p, est)))


def record_field(seed: int, ident: int, tag: int, w0: int, uniforms: int, i: int) -> int:
    """The 23-bit field of uniform i of the `uniforms`-uniform record starting at word w0 of stream (id, tag)."""
    return int(lib().or_record_field(seed, ident, tag, w0, uniforms, i))


# --------------------------------------------------------------------------------------
# Normal CDF / quantile

def Phi(x: float) -> float:
    return float(lib().or_Phi(float(x)))


def Phi_inv(p: float) -> float:
    return float(lib().or_Phi_inv(float(p)))


def threshold(alpha: float) -> float:
    """Z_{1-alpha}; alpha = 0 -> +inf (reading R13)."""
    return float(lib().or_threshold(float(alpha)))


# --------------------------------------------------------------------------------------
# Problem model (Sec. 2.1, Sec. 3)

def information_units(alpha: float = 0.025, beta: float = 0.1, delta: float = 0.2) -> float:
    """Eq. 9: I3 = (Z_{1-alpha} + Z_{1-beta})^2 / log(1 - Delta)^2."""
    za, zb = Phi_inv(1.0 - alpha), Phi_inv(1.0 - beta)
    return (za + zb) ** 2 / np.log(1.0 - delta) ** 2


def null_corr(r) -> np.ndarray:
    """Formula 1 / A.1: Sigma0[k][l] = sqrt(r_l / r_k), k <= l."""
    r = np.asarray(r, dtype=np.float64)
    n = len(r)
    S = np.empty((n, n))
    for k in range(n):
        for l in range(n):
            a, b = min(k, l), max(k, l)
            S[k, l] = np.sqrt(r[b] / r[a])
    return S


def cholesky(A) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    L = np.zeros((n, n))
    rc = lib().or_cholesky(n, _dp(A), L.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc != 0:
        raise np.linalg.LinAlgError(f"matrix not positive definite at pivot {rc - 1}")
    return L


@dataclass
class Problem:
    """One fixed-r design problem: r, I3, alpha0 and the effect prior f(Delta)."""
    r: np.ndarray
    i3: float
    alpha0: float
    theta: np.ndarray
    prior_cov: np.ndarray
    Lp: np.ndarray = field(init=False)

    def __post_init__(self):
        self.r = np.asarray(self.r, dtype=np.float64)
        self.theta = np.asarray(self.theta, dtype=np.float64)
        self.prior_cov = np.asarray(self.prior_cov, dtype=np.float64)
        self.Lp = cholesky(self.prior_cov) if np.any(self.prior_cov) else np.zeros_like(self.prior_cov)

    @property
    def n(self) -> int:
        return len(self.r)

    @property
    def c(self) -> np.ndarray:
        """Formula 3: mean of X_i is sqrt(r_i I3) Delta_i."""
        return np.sqrt(self.r * self.i3)


def formula10_problem(r, delta0, i3: float, alpha0: float = 0.025, sigma=None) -> Problem:
    """Formula 10: theta_i = -log(1 - Delta0_i), sigma_i = 1/sqrt(80 r_i / 4),
    Sigma_p[k][l] = sqrt(r_l / r_k) sigma_k sigma_l (readings R4, R5)."""
    r = np.asarray(r, dtype=np.float64)
    theta = -np.log(1.0 - np.asarray(delta0, dtype=np.float64))
    if sigma is None:
        sigma = 1.0 / np.sqrt(80.0 * r / 4.0)
    sigma = np.asarray(sigma, dtype=np.float64) * np.ones_like(r)
    cov = null_corr(r) * np.outer(sigma, sigma)
    return Problem(r=r, i3=float(i3), alpha0=float(alpha0), theta=theta, prior_cov=cov)


def point_mass_problem(r, theta, i3: float, alpha0: float = 0.025) -> Problem:
    r = np.asarray(r, dtype=np.float64)
    return Problem(r=r, i3=float(i3), alpha0=float(alpha0), theta=np.asarray(theta, dtype=np.float64),
                   prior_cov=np.zeros((len(r), len(r))))


# --------------------------------------------------------------------------------------
# Monte-Carlo estimator (Formulas 5-7 with the readings of DESIGN.md §2)

EST_COND, EST_IND = 0, 1


def thresholds(alpha) -> np.ndarray:
    return np.array([threshold(a) for a in np.asarray(alpha, dtype=np.float64)])


def draw(prob: Problem, alpha, est: int, seed: int, design: int, s: int, tag: int = 0) -> dict:
    """One draw: returns the prior normals, Delta, b and u (for per-draw parity).  tag 0: the stream of
    `design`; tag 1: the common-random-number stream of problem `design` (NEXT f3)."""
    n = prob.n
    p = n
    z = thresholds(alpha)
    eps, delta, b, wn = np.zeros(p), np.zeros(n), np.zeros(n), np.zeros(n)
    P = ctypes.POINTER(ctypes.c_double)
    u = lib().or_draw(n, p, _dp(prob.r), prob.i3, _dp(prob.theta), _dp(prob.Lp), _dp(z), est,
                      seed, design, tag, s, eps.ctypes.data_as(P), delta.ctypes.data_as(P),
                      b.ctypes.data_as(P), wn.ctypes.data_as(P))
    return {"u": float(u), "eps": eps, "delta": delta, "b": b, "xnull": wn}


def design_sums(prob: Problem, alpha, est: int, seed: int, design: int, s0: int, count: int,
                tag: int = 0) -> np.ndarray:
    """Integer sums (sum q(u), sum q(u^2)) over samples [s0, s0+count), q = round(2^23 x).  With tag 1
    `design` is the problem index of the common-random-number stream (NEXT f3)."""
    n = prob.n
    z = thresholds(alpha)
    sums = np.zeros(2, dtype=np.int64)
    lib().or_design_sums(n, n, _dp(prob.r), prob.i3, _dp(prob.theta), _dp(prob.Lp), _dp(z), est, seed,
                         design, tag, s0, count, sums.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return sums


def finalize(sums, N: int):
    """Formula 5/7 estimate and per-draw variance (A.2): mean = S1/(N 2^23),
    var = (S2/(N 2^23) - mean^2) N/(N-1), SE = sqrt(var/N)."""
    S = np.asarray(sums, dtype=np.float64).reshape(-1, 2)
    mean = S[:, 0] / (N * 2.0 ** 23)
    m2 = S[:, 1] / (N * 2.0 ** 23)
    var = (m2 - mean * mean) * N / max(N - 1, 1)
    return mean, var


# --------------------------------------------------------------------------------------
# Exact references (pins for the estimand)

def mvn_orthant(r, b) -> float:
    """Phi_Sigma0(b) by the Markov-chain iterated integral (A.1 => Markov; see oracle.c)."""
    r = np.asarray(r, dtype=np.float64)
    return float(lib().or_mvn_orthant(len(r), _dp(r), _dp(np.asarray(b, dtype=np.float64))))


def fwer(r, alpha) -> float:
    """Formula 2."""
    r = np.asarray(r, dtype=np.float64)
    return float(lib().or_fwer(len(r), _dp(r), _dp(np.asarray(alpha, dtype=np.float64))))


def solve_alpha_n(r, alpha0: float, partial, tol: float = 1e-13):
    r = np.asarray(r, dtype=np.float64)
    out = ctypes.c_double(0.0)
    ok = lib().or_solve_alpha_n(len(r), _dp(r), float(alpha0), _dp(np.asarray(partial, dtype=np.float64)),
                                tol, ctypes.byref(out))
    if ok < 0:
        raise ValueError("solve_alpha_n: the orthant quadrature is unavailable for this r (node cap)")
    return float(out.value) if ok else None


def assurance_gaussian(prob: Problem, alpha) -> float:
    """Exact P(alpha) for a Gaussian prior (Formula 4): X = c*Delta + E with E ~ N(0, Sigma0)
    independent of Delta ~ N(theta, Sigma_p), so X ~ N(c*theta, V), V = Sigma0 + C Sigma_p C, and
    P = 1 - P(X <= z).  Standardising, the bound is (z_i - c_i theta_i)/sqrt(V_ii) under the
    correlation R = V / sqrt(diag V diag V).  For Formula 10, C Sigma_p C = (I3/20) Sigma0, so R =
    Sigma0 (SURVEY finding 1).  R must have the Formula-1 (Markov) form for some r'; else raise."""
    z = thresholds(alpha)
    c = prob.c
    V = null_corr(prob.r) + np.outer(c, c) * prob.prior_cov
    sd = np.sqrt(np.diag(V))
    R = V / np.outer(sd, sd)
    # R must be a Formula-1 correlation for some r' (then the orthant is Markov).
    rp = R[0, :] ** 2
    if not np.allclose(null_corr(rp), R, rtol=0, atol=1e-12):
        raise ValueError("prior does not preserve the nested (Markov) correlation")
    b = (z - c * prob.theta) / sd
    return 1.0 - mvn_orthant(rp, b)


# --------------------------------------------------------------------------------------
# Candidate designs (Sec. 2.3)

def alpha_grid(r, alpha0: float, m: int, tol: float = 1e-13):
    """All m^(n-1) half-offset grid points: (alpha[G, n], valid[G])."""
    r = np.asarray(r, dtype=np.float64)
    n = len(r)
    G = m ** (n - 1)
    A = np.zeros((G, n))
    V = np.zeros(G, dtype=np.uint8)
    if lib().or_alpha_grid(n, _dp(r), float(alpha0), int(m), tol, A.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                           V.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))) < 0:
        raise ValueError("alpha_grid: the orthant quadrature is unavailable for this r (node cap)")
    return A, V.astype(bool)


def subset(V: int, n3: int, seed: int) -> np.ndarray:
    out = np.zeros(max(n3, 1), dtype=np.int64)
    lib().or_subset(int(V), int(n3), int(seed), out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return out[:n3]


def candidates(r, alpha0: float, m: int, n3: int, seed: int, tol: float = 1e-13) -> np.ndarray:
    """Valid grid points in grid order; if 0 < n3 < #valid, the seeded N3 subset (R11)."""
    A, ok = alpha_grid(r, alpha0, m, tol)
    valid = A[ok]
    if n3 <= 0 or n3 >= len(valid):
        if n3 > len(valid):
            raise ValueError(f"only {len(valid)} valid candidates < N3={n3}")
        return valid
    return valid[subset(len(valid), n3, seed)]


# --------------------------------------------------------------------------------------
# Thin-plate-spline smoothing (Sec. 2.3; readings R16)

def tps_phi(rho: np.ndarray, d: int) -> np.ndarray:
    """Polyharmonic TPS kernel for penalty order m = 2 (Green's function of the m=2 penalty up to a
    positive factor): d=1 -> rho^3, d=2 -> rho^2 log rho, d=3 -> -rho."""
    rho = np.asarray(rho, dtype=np.float64)
    if d == 2:
        with np.errstate(divide="ignore", invalid="ignore"):
            out = np.where(rho > 0, rho * rho * np.log(np.where(rho > 0, rho, 1.0)), 0.0)
        return out
    if d == 1:
        return rho ** 3
    if d == 3:
        return -rho
    raise ValueError(f"TPS dimension d={d} not supported (1..3)")


def tps_system(x: np.ndarray):
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    if x.shape[0] == 1 and x.shape[1] > 1 and x.ndim == 2:
        pass
    N, d = x.shape
    D = np.sqrt(((x[:, None, :] - x[None, :, :]) ** 2).sum(-1))
    K = tps_phi(D, d)
    T = np.hstack([np.ones((N, 1)), x])
    return K, T


def tps_fit(x, y, lam: float):
    """Solve [K + N lam I, T; T^T, 0][w; beta] = [y; 0] (the penalised least-squares TPS,
    1/N sum (y - f)^2 + lam J(f)).  Returns (fitted values, w, beta)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    y = np.asarray(y, dtype=np.float64)
    K, T = tps_system(x)
    N, k = T.shape
    M = np.zeros((N + k, N + k))
    M[:N, :N] = K + N * lam * np.eye(N)
    M[:N, N:] = T
    M[N:, :N] = T.T
    sol = np.linalg.solve(M, np.concatenate([y, np.zeros(k)]))
    w, beta = sol[:N], sol[N:]
    fitted = K @ w + T @ beta
    return fitted, w, beta


def tps_influence(x, lam: float) -> np.ndarray:
    """Influence matrix A(lam): fitted = A y (solve with identity right-hand sides)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    K, T = tps_system(x)
    N, k = T.shape
    M = np.zeros((N + k, N + k))
    M[:N, :N] = K + N * lam * np.eye(N)
    M[:N, N:] = T
    M[N:, :N] = T.T
    rhs = np.zeros((N + k, N))
    rhs[:N, :] = np.eye(N)
    sol = np.linalg.solve(M, rhs)
    return K @ sol[:N] + T @ sol[N:]


GCV_LOG10_GRID = -12.0 + 0.25 * np.arange(49)   # lambda = 10^-12 ... 10^0 (reading R16)


def gcv_score(x, y, lam: float) -> float:
    """Craven & Wahba GCV: V(lam) = (1/N)||(I - A)y||^2 / ((1/N) tr(I - A))^2."""
    A = tps_influence(x, lam)
    y = np.asarray(y, dtype=np.float64)
    N = len(y)
    res = y - A @ y
    return (res @ res / N) / ((np.trace(np.eye(N) - A) / N) ** 2)


def tps_smooth(x, y, lam: float = -1.0):
    """Smoothed values P~ at the sites and the lambda used (lam < 0: GCV over the grid,
    the first minimiser wins)."""
    if lam < 0:
        scores = np.array([gcv_score(x, y, 10.0 ** g) for g in GCV_LOG10_GRID])
        lam = float(10.0 ** GCV_LOG10_GRID[int(np.argmin(scores))])
    fitted, _, _ = tps_fit(x, y, lam)
    return fitted, lam


def argmax(values) -> int:
    """Design with the largest value, lowest index on ties."""
    v = np.asarray(values)
    best = 0
    for i in range(1, len(v)):
        if v[i] > v[best]:
            best = i
    return best


# --------------------------------------------------------------------------------------
# C4: 5-D strata prior (synthetic extension of Formula 3, see oracle.c)

def draw_strata(r2: float, i3: float, sp, alpha, est: int, seed: int, design: int, s: int, tag: int = 0) -> dict:
    z = thresholds(alpha)
    eps, delta, b, wn = np.zeros(5), np.zeros(2), np.zeros(2), np.zeros(2)
    P = ctypes.POINTER(ctypes.c_double)
    u = lib().or_draw_strata(float(r2), float(i3), _dp(np.asarray(sp, dtype=np.float64)), _dp(z), est, seed, design,
                             tag, s, eps.ctypes.data_as(P), delta.ctypes.data_as(P), b.ctypes.data_as(P),
                             wn.ctypes.data_as(P))
    return {"u": float(u), "eps": eps, "delta": delta, "b": b, "xnull": wn}


def design_sums_strata(r2: float, i3: float, sp, alpha, est: int, seed: int, design: int, s0: int,
                       count: int, tag: int = 0) -> np.ndarray:
    z = thresholds(alpha)
    sums = np.zeros(2, dtype=np.int64)
    lib().or_design_sums_strata(float(r2), float(i3), _dp(np.asarray(sp, dtype=np.float64)), _dp(z), est, seed,
                                design, tag, s0, count, sums.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return sums


def strata_b(r2: float, i3: float, sp, z, e):
    """Deterministic map (eps_1..eps_5) -> b of the C4 model (same formulas as oracle.c, vectorised)."""
    e = np.asarray(e, dtype=np.float64)
    pi = 1.0 / (1.0 + np.exp(-(sp[0] + sp[1] * e[..., 0])))
    dp = sp[2] + sp[3] * e[..., 1]
    dm = sp[4] + sp[5] * e[..., 2]
    v = np.exp(sp[6] + sp[7] * e[..., 3])
    d = 1.0 / (1.0 + np.exp(-(sp[8] + sp[9] * e[..., 4])))
    ieff = i3 * (1.0 - d) / v
    qp = np.minimum(1.0, pi / r2)
    qm = np.maximum(0.0, (pi - r2) / (1.0 - r2))
    d2 = qp * dp + (1.0 - qp) * dm
    dneg = qm * dp + (1.0 - qm) * dm
    d1 = r2 * d2 + (1.0 - r2) * dneg
    return np.stack([z[0] - np.sqrt(ieff) * d1, z[1] - np.sqrt(r2 * ieff) * d2], axis=-1)


def assurance_strata_quadrature(r2: float, i3: float, sp, alpha, n_gh: int = 8, n_gl: int = 24) -> float:
    """Tensor-product brute force of Formula 4 under the C4 prior: Gauss-Hermite over the four smooth
    components and Gauss-Legendre on each side of the prevalence kink eps1* = (logit r2 - mu)/sd (where
    q+ = min(1, pi/r2) bends), inner Phi_Sigma0 by the exact bivariate orthant."""
    z = thresholds(alpha)
    xh, wh = np.polynomial.hermite_e.hermegauss(n_gh)
    wh = wh / wh.sum()
    kink = (np.log(r2 / (1 - r2)) - sp[0]) / sp[1] if sp[1] > 0 else None
    xg, wg = np.polynomial.legendre.leggauss(n_gl)
    if kink is None:
        e1 = np.array([0.0]); w1 = np.array([1.0])
    else:
        lo, hi = -9.0, 9.0
        segs = [(lo, min(max(kink, lo), hi)), (min(max(kink, lo), hi), hi)]
        e1, w1 = [], []
        for a, b in segs:
            if b <= a:
                continue
            x = 0.5 * (b - a) * (xg + 1) + a
            e1.append(x)
            w1.append(0.5 * (b - a) * wg * np.exp(-0.5 * x * x) / np.sqrt(2 * np.pi))
        e1 = np.concatenate(e1); w1 = np.concatenate(w1)
    total = 0.0
    r = [1.0, r2]
    for i1, a1 in enumerate(e1):
        for i2 in range(n_gh):
            for i3_ in range(n_gh):
                for i4 in range(n_gh):
                    for i5 in range(n_gh):
                        e = np.array([a1, xh[i2], xh[i3_], xh[i4], xh[i5]])
                        b = strata_b(r2, i3, sp, z, e)
                        total += w1[i1] * wh[i2] * wh[i3_] * wh[i4] * wh[i5] * (1.0 - mvn_orthant(r, b))
    return float(total)


# --------------------------------------------------------------------------------------
# NEXT f1: continuous optimum on the TPS surface (P:123 L-BFGS-B, P:219 start at the best site)

def tps_eval(sites, w, beta, x):
    """f(x) = beta_0 + beta_{1..d} x + sum_i w_i phi(|x - x_i|) and its gradient."""
    sites = np.atleast_2d(np.asarray(sites, dtype=np.float64))
    d = sites.shape[1]
    x = np.asarray(x, dtype=np.float64)
    diff = x[None, :] - sites
    r = np.sqrt((diff ** 2).sum(1))
    f = beta[0] + beta[1:] @ x + w @ tps_phi(r, d)
    with np.errstate(divide="ignore", invalid="ignore"):
        if d == 1:
            dphi_r = 3 * r
        elif d == 2:
            dphi_r = np.where(r > 0, 2 * np.log(np.where(r > 0, r, 1.0)) + 1.0, 0.0)
        else:
            dphi_r = np.where(r > 0, -1.0 / np.where(r > 0, r, 1.0), 0.0)
    grad = beta[1:] + (w * dphi_r) @ diff
    return float(f), grad


def refine(sites, y, lam: float = -1.0):
    """Maximise the fitted TPS by scipy's L-BFGS-B (a library routine) from the fitted site with the
    largest value over the sites' bounding box.  Returns (x*, f*, lambda)."""
    from scipy.optimize import minimize
    sites = np.atleast_2d(np.asarray(sites, dtype=np.float64))
    if lam < 0:
        _, lam = tps_smooth(sites, y, -1.0)
    fitted, w, beta = tps_fit(sites, y, lam)
    x0 = sites[int(np.argmax([tps_eval(sites, w, beta, s)[0] for s in sites]))]
    bounds = list(zip(sites.min(0), sites.max(0)))
    res = minimize(lambda x: tuple(-v for v in tps_eval(sites, w, beta, x)), x0, jac=True, method="L-BFGS-B",
                   bounds=bounds, options={"ftol": 1e-15, "gtol": 1e-12, "maxiter": 500, "maxcor": 10})
    return res.x, -float(res.fun), lam


# --------------------------------------------------------------------------------------
# NEXT f3 (ii): the crossed N1 x N2 estimator of Formula 7

def design_sums_crossed(prob: Problem, alpha, seed: int, design: int, n1: int, n2: int) -> np.ndarray:
    z = thresholds(alpha)
    sums = np.zeros(2, dtype=np.int64)
    lib().or_design_sums_crossed(prob.n, _dp(prob.r), prob.i3, _dp(prob.theta), _dp(prob.Lp), _dp(z), seed, design,
                                 n1, n2, sums.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return sums


def finalize_crossed(sums, n1: int, n2: int):
    S = np.asarray(sums, dtype=np.float64).reshape(-1, 2)
    mean = S[:, 0] / (n1 * n2)
    var = (S[:, 1] / (n2 * n2) - n1 * mean * mean) / max(n1 - 1, 1)
    return mean, var


# --------------------------------------------------------------------------------------
# C4 dense-grid smoother (SURVEY §8(a) a9 "Dense regular grids (C4)"; reading R23 in DESIGN.md):
# the separable Gaussian (Nadaraya-Watson) kernel smoother P~ = S_r P^ S_a^T over the (r2, alpha_1) grid,
# S_x = row-normalised W_x, W_x[i, k] = exp(-(x_i - x_k)^2 / (2 h_x^2)).  Bandwidths h = k * (grid step)
# with k in GRID_H_STEPS, chosen jointly by GCV (first minimiser, r-bandwidth outer), tr S = tr S_r tr S_a.

GRID_H_STEPS = 2.0 ** (np.arange(-2, 9) / 2.0)   # 0.5 ... 16 grid steps, ratio sqrt(2)


def kernel_matrix_nw(x, h: float) -> np.ndarray:
    """Row-normalised Gaussian kernel weights on the 1-D coordinates x with bandwidth h."""
    x = np.asarray(x, dtype=np.float64)
    W = np.exp(-0.5 * ((x[:, None] - x[None, :]) / h) ** 2)
    return W / W.sum(axis=1, keepdims=True)


def grid_kernel_smooth(P, xr, xa, hr: float, ha: float):
    """P~ = S_r P S_a^T for P[nr, na] (rows: r coordinate xr, columns: alpha coordinate xa);
    returns (P~, tr S)."""
    Sr, Sa = kernel_matrix_nw(xr, hr), kernel_matrix_nw(xa, ha)
    P = np.asarray(P, dtype=np.float64)
    return Sr @ P @ Sa.T, float(np.trace(Sr) * np.trace(Sa))


def grid_gcv(P, xr, xa, hr: float, ha: float) -> float:
    """GCV(h) = (1/n) ||P - P~||^2 / (1 - tr S / n)^2 (Craven & Wahba, as for the TPS)."""
    Ps, tr = grid_kernel_smooth(P, xr, xa, hr, ha)
    n = Ps.size
    res = np.asarray(P, dtype=np.float64) - Ps
    return float((res * res).sum() / n / (1.0 - tr / n) ** 2)


def grid_smooth(P, xr, xa, hr: float = -1.0, ha: float = -1.0):
    """Smoothed grid and the bandwidths used; hr, ha <= 0: GCV over GRID_H_STEPS x the grid steps."""
    xr, xa = np.asarray(xr, dtype=np.float64), np.asarray(xa, dtype=np.float64)
    if hr <= 0 or ha <= 0:
        sr = (xr[-1] - xr[0]) / (len(xr) - 1)
        sa = (xa[-1] - xa[0]) / (len(xa) - 1)
        best = None
        for kr in GRID_H_STEPS:
            for ka in GRID_H_STEPS:
                g = grid_gcv(P, xr, xa, kr * sr, ka * sa)
                if best is None or g < best[0]:
                    best = (g, kr * sr, ka * sa)
        hr, ha = best[1], best[2]
    Ps, _ = grid_kernel_smooth(P, xr, xa, hr, ha)
    return Ps, (hr, ha)
