"""Thin ctypes binding of libmc_design.so (include/mc_design.h).

Argument marshalling only: every step of the method runs in the CUDA library.  Torch supplies
device memory (tensor ``data_ptr()``), the current CUDA stream and ``torch.distributed`` for the
one cross-GPU combine (row a7).  There is no CPU fallback: compute calls raise if the library or a
CUDA device is missing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

MC_MAX_N = 10
EST_COND, EST_IND = 0, 1
_STATUS = {0: "MC_OK", 1: "MC_ERR_INVALID", 2: "MC_ERR_NUMERIC", 3: "MC_ERR_INFEASIBLE", 4: "MC_ERR_CUDA",
           5: "MC_ERR_OOM"}


class McError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class mc_problem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("has_prior_chol", ctypes.c_int32), ("i3", ctypes.c_double),
                ("alpha0", ctypes.c_double), ("r", ctypes.c_double * MC_MAX_N),
                ("theta", ctypes.c_double * MC_MAX_N), ("sigma", ctypes.c_double * MC_MAX_N),
                ("prior_chol", ctypes.c_double * (MC_MAX_N * MC_MAX_N)), ("model", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("strata", ctypes.c_double * 10)]


_lib = None


def lib_path() -> str:
    return os.environ.get("MC_LIB_PATH", _build.LIB)


def lib() -> ctypes.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: run `python -m paper_2005_10494_b200.build` "
                               "(no CPU fallback exists)")
        L = ctypes.CDLL(path)
        i32, i64, u64, d, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        P = ctypes.POINTER
        L.mc_last_error.restype = ctypes.c_char_p
        L.mc_version.restype = ctypes.c_char_p
        L.mc_information_units.argtypes = [d, d, d]; L.mc_information_units.restype = d
        L.mc_threshold.argtypes = [d]; L.mc_threshold.restype = d
        L.mc_problem_formula10.argtypes = [i32, P(d), P(d), d, d, P(mc_problem)]; L.mc_problem_formula10.restype = i32
        L.mc_problem_strata.argtypes = [d, d, d, P(d), P(mc_problem)]; L.mc_problem_strata.restype = i32
        L.mc_fwer.argtypes = [P(mc_problem), P(d), i64, P(d), i32]; L.mc_fwer.restype = i32
        L.mc_solve_alpha_n.argtypes = [P(mc_problem), i32, P(i32), i64, P(d), P(ctypes.c_uint8), i32]
        L.mc_solve_alpha_n.restype = i32
        L.mc_candidates.argtypes = [P(mc_problem), i32, i32, i64, u64, P(d), P(i32), i64, P(i64), i32]
        L.mc_candidates.restype = i32
        L.mc_design_init.argtypes = [P(vp), P(mc_problem), i32, P(d), P(i32), i64, u64, i32, i32]
        L.mc_design_init.restype = i32
        L.mc_design_upload.argtypes = [vp, P(d), vp]; L.mc_design_upload.restype = i32
        L.mc_set_launch.argtypes = [vp, i32, i32]; L.mc_set_launch.restype = i32
        L.mc_set_sampling.argtypes = [vp, i32]; L.mc_set_sampling.restype = i32
        L.mc_destroy.argtypes = [vp]; L.mc_destroy.restype = None
        L.mc_evaluate_grid.argtypes = [vp, i64, i64, u64, u64, vp, vp]; L.mc_evaluate_grid.restype = i32
        L.mc_evaluate_crossed.argtypes = [vp, u64, u64, vp, vp]; L.mc_evaluate_crossed.restype = i32
        L.mc_finalize_crossed.argtypes = [vp, vp, u64, u64, vp, vp, vp]; L.mc_finalize_crossed.restype = i32
        L.mc_finalize.argtypes = [vp, vp, u64, vp, vp, vp]; L.mc_finalize.restype = i32
        L.mc_smooth_plan.argtypes = [vp, vp, vp]; L.mc_smooth_plan.restype = i32
        L.mc_smooth.argtypes = [vp, vp, d, vp, vp, vp]; L.mc_smooth.restype = i32
        L.mc_tps_fit.argtypes = [vp, vp, d, vp]; L.mc_tps_fit.restype = i32
        L.mc_tps_eval.argtypes = [vp, i32, P(d), i64, P(d), P(d)]; L.mc_tps_eval.restype = i32
        L.mc_refine.argtypes = [vp, vp, d, P(d), P(d), P(i32), vp]; L.mc_refine.restype = i32
        L.mc_surface_fit.argtypes = [P(d), i64, i32, P(d), d, P(vp), P(d)]; L.mc_surface_fit.restype = i32
        L.mc_surface_eval.argtypes = [vp, P(d), i64, P(d), P(d)]; L.mc_surface_eval.restype = i32
        L.mc_surface_max.argtypes = [vp, P(d), P(d)]; L.mc_surface_max.restype = i32
        L.mc_surface_destroy.argtypes = [vp]; L.mc_surface_destroy.restype = None
        L.mc_argmax.argtypes = [vp, vp, vp, vp, P(i64), P(d), vp]; L.mc_argmax.restype = i32
        L.mc_grid_smooth.argtypes = [vp, i32, i32, P(d), P(d), d, d, vp, P(d), vp]; L.mc_grid_smooth.restype = i32
        L.mc_num_designs.argtypes = [vp]; L.mc_num_designs.restype = i64
        L.mc_num_problems.argtypes = [vp]; L.mc_num_problems.restype = i32
        L.mc_words_per_record.argtypes = [vp]; L.mc_words_per_record.restype = i32
        L.mc_philox_dump.argtypes = [u64, ctypes.c_uint32, i32, vp, vp, i64, vp, vp]; L.mc_philox_dump.restype = i32
        L.mc_draw_dump.argtypes = [vp, vp, vp, i64, vp, vp]; L.mc_draw_dump.restype = i32
        L.mc_draw_dump_stride.argtypes = [vp]; L.mc_draw_dump_stride.restype = i32
        L.mc_kernel_launches.argtypes = [vp]; L.mc_kernel_launches.restype = i64
        _lib = L
    return _lib


EXPORTED = ["mc_information_units", "mc_threshold", "mc_problem_formula10", "mc_problem_strata", "mc_fwer",
            "mc_solve_alpha_n", "mc_candidates",
            "mc_design_init", "mc_design_upload", "mc_set_sampling", "mc_set_launch", "mc_destroy", "mc_evaluate_grid", "mc_evaluate_crossed", "mc_finalize_crossed", "mc_finalize", "mc_smooth_plan",
            "mc_smooth", "mc_tps_fit", "mc_tps_eval", "mc_refine", "mc_surface_fit", "mc_surface_eval", "mc_surface_max", "mc_surface_destroy", "mc_grid_smooth", "mc_argmax", "mc_num_designs", "mc_num_problems", "mc_words_per_record", "mc_philox_dump",
            "mc_draw_dump", "mc_draw_dump_stride", "mc_kernel_launches", "mc_last_error", "mc_version"]


def _check(status: int):
    if status != 0:
        raise McError(status, lib().mc_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2005_10494_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


# ------------------------------------------------------------------------------------------
# problem helpers (host fp64, inside the library)

def information_units(alpha: float = 0.025, beta: float = 0.1, delta: float = 0.2) -> float:
    return float(lib().mc_information_units(alpha, beta, delta))


def threshold(alpha: float) -> float:
    return float(lib().mc_threshold(alpha))


def problem_formula10(r, delta0, i3: float, alpha0: float = 0.025) -> mc_problem:
    r = np.ascontiguousarray(r, dtype=np.float64)
    d0 = np.ascontiguousarray(delta0, dtype=np.float64)
    p = mc_problem()
    _check(lib().mc_problem_formula10(len(r), _dp(r), _dp(d0), float(i3), float(alpha0), ctypes.byref(p)))
    return p


def problem_strata(r2: float, i3: float, strata, alpha0: float = 0.025) -> mc_problem:
    """C4 strata prior (n = 2)."""
    sp = np.ascontiguousarray(strata, dtype=np.float64)
    p = mc_problem()
    _check(lib().mc_problem_strata(float(r2), float(i3), float(alpha0), _dp(sp), ctypes.byref(p)))
    return p


def problem_general(r, theta, prior_chol, i3: float, alpha0: float = 0.025) -> mc_problem:
    """A Gaussian prior N(theta, L L^T) given by its lower Cholesky factor L (n x n)."""
    p = mc_problem()
    n = len(r)
    p.n, p.has_prior_chol, p.i3, p.alpha0 = n, 1, float(i3), float(alpha0)
    L = np.asarray(prior_chol, dtype=np.float64)
    for i in range(n):
        p.r[i] = float(r[i])
        p.theta[i] = float(theta[i])
        for j in range(i + 1):
            p.prior_chol[i * MC_MAX_N + j] = float(L[i, j])
    return p


def problem_point_mass(r, theta, i3: float, alpha0: float = 0.025) -> mc_problem:
    p = mc_problem()
    n = len(r)
    p.n, p.has_prior_chol, p.i3, p.alpha0 = n, 0, float(i3), float(alpha0)
    for i in range(n):
        p.r[i], p.theta[i], p.sigma[i] = float(r[i]), float(theta[i]), 0.0
    return p


def _problem_array(problems):
    arr = (mc_problem * len(problems))()
    for i, p in enumerate(problems):
        arr[i] = p
    return arr


def fwer(problem: mc_problem, alpha, device: int = 0) -> np.ndarray:
    a = np.ascontiguousarray(np.atleast_2d(alpha), dtype=np.float64)
    out = np.zeros(a.shape[0])
    _check(lib().mc_fwer(ctypes.byref(problem), _dp(a), a.shape[0], _dp(out), device))
    return out


def solve_alpha_n(problems, alpha, problem_of_design, device: int = 0):
    """Row a1 for explicit partial designs: alpha_n solved on the GPU (Formula 2).  alpha[count, n] (the last
    column is overwritten).  Returns (alpha with alpha_n, valid mask)."""
    arr = _problem_array(problems)
    n = problems[0].n
    A = np.array(alpha, dtype=np.float64, order="C").reshape(-1, n)
    pod = np.ascontiguousarray(problem_of_design, dtype=np.int32)
    ok = np.zeros(len(A), dtype=np.uint8)
    _check(lib().mc_solve_alpha_n(arr, len(problems), pod.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(A),
                                  _dp(A), ok.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), device))
    return A, ok.astype(bool)


def candidates(problems, m: int = 64, n3: int = 0, seed: int = 0, device: int = 0):
    """Row a1: the alpha grid with alpha_n solved on the GPU and the seeded N3 subset.
    Returns (alpha[D, n], problem_of_design[D])."""
    arr = _problem_array(problems)
    n = problems[0].n
    need = ctypes.c_int64(0)
    # capacity: at most min(grid size, N3) designs per problem, so one call solves the grid (a size query
    # first would run the whole GPU solve twice)
    G = m ** (n - 1)
    cap = max(len(problems) * (min(G, n3) if n3 > 0 else G), 1)
    A = np.zeros((cap, n))
    pod = np.zeros(cap, dtype=np.int32)
    _check(lib().mc_candidates(arr, len(problems), m, n3, seed, _dp(A), pod.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                               cap, ctypes.byref(need), device))
    D = int(need.value)
    return A[:D], pod[:D]


PHILOX_FORM_STEADY, PHILOX_FORM_MASKED, PHILOX_FORM_PLAIN = 0, 1, 2


def philox_dump(seed: int, design, word, tag: int = 0, form: int = PHILOX_FORM_STEADY, stream=None):
    """K3: Philox words of stream (id, tag) for (id, word-index) pairs, in the block form `form` the kernels
    use (device tensors in, device tensor out)."""
    torch = _torch()
    design = design.to(torch.int32).contiguous()
    word = word.to(torch.int64).contiguous()
    out = torch.empty(design.numel(), dtype=torch.int32, device=design.device)
    _check(lib().mc_philox_dump(seed, tag, form, design.data_ptr(), word.data_ptr(), design.numel(), out.data_ptr(),
                                _stream(stream)))
    return out


# ------------------------------------------------------------------------------------------

class Design:
    """A device design table (mc_design_init) and the hot-path calls on it."""

    def __init__(self, problems, alpha, problem_of_design, seed: int, estimator: int = EST_COND, device: int = 0):
        torch = _torch()
        self.device = device
        self.problems = list(problems)
        self.n = self.problems[0].n
        a = np.ascontiguousarray(alpha, dtype=np.float64).reshape(-1, self.n)
        pod = np.ascontiguousarray(problem_of_design, dtype=np.int32)
        self.alpha = a
        self.pod = pod
        self.D = a.shape[0]
        self.seed = int(seed)
        self.estimator = int(estimator)
        arr = _problem_array(self.problems)
        ctx = ctypes.c_void_p()
        torch.cuda.set_device(device)
        _check(lib().mc_design_init(ctypes.byref(ctx), arr, len(self.problems), _dp(a),
                                    pod.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), self.D, self.seed,
                                    self.estimator, device))
        self._ctx = ctx
        self.n_probs = len(self.problems)

    def close(self):
        try:
            self._join_plan()
        except McError:
            pass
        if getattr(self, "_ctx", None) is not None and self._ctx.value:
            lib().mc_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def words_per_record(self) -> int:
        return int(lib().mc_words_per_record(self._ctx))

    @property
    def launches(self) -> int:
        return int(lib().mc_kernel_launches(self._ctx))

    def upload(self, alpha_host, stream=None):
        """Replace the design table from host memory (H2D + device thresholds); alpha_host may be a
        pinned torch CPU tensor (async copy) or a numpy array."""
        self._join_plan()
        if hasattr(alpha_host, "data_ptr"):
            ptr = ctypes.cast(alpha_host.data_ptr(), ctypes.POINTER(ctypes.c_double))
        else:
            alpha_host = np.ascontiguousarray(alpha_host, dtype=np.float64)
            ptr = _dp(alpha_host)
        _check(lib().mc_design_upload(self._ctx, ptr, _stream(stream)))

    def set_sampling(self, crn: bool):
        """NEXT f3: common random numbers per problem (True) or independent draws per design."""
        _check(lib().mc_set_sampling(self._ctx, 1 if crn else 0))

    def set_launch(self, block_threads: int = 0, grid_blocks: int = 0):
        _check(lib().mc_set_launch(self._ctx, block_threads, grid_blocks))

    def _check_sums(self, sums, where: str):
        """The sums buffer the kernels' 64-bit atomics write: a contiguous int64 (D, 2) CUDA tensor on the
        ctx device (anything else would be written past its end or into the wrong elements)."""
        torch = _torch()
        if not (isinstance(sums, torch.Tensor) and sums.is_cuda and sums.dtype == torch.int64
                and sums.is_contiguous() and tuple(sums.shape) == (self.D, 2)
                and sums.device.index == self.device):
            raise ValueError(f"{where}: sums must be a contiguous int64 CUDA tensor of shape ({self.D}, 2) on "
                             f"cuda:{self.device}; got {getattr(sums, 'dtype', type(sums))} "
                             f"{tuple(getattr(sums, 'shape', ()))} on {getattr(sums, 'device', '?')}")

    def new_sums(self):
        torch = _torch()
        return torch.zeros((self.D, 2), dtype=torch.int64, device=f"cuda:{self.device}")

    def evaluate(self, sums, sample_begin: int, sample_count: int, design_begin: int = 0, design_count=None,
                 stream=None):
        """Rows a2-a6: accumulate the integer sums of samples [begin, begin+count) into `sums`."""
        if design_count is None:
            design_count = self.D - design_begin
        self._check_sums(sums, "evaluate")
        _check(lib().mc_evaluate_grid(self._ctx, design_begin, design_count, sample_begin, sample_count,
                                      _stream(stream), sums.data_ptr()))
        return sums

    def evaluate_crossed(self, sums, n1: int, n2: int, stream=None):
        """NEXT f3 (ii): the paper's crossed N1 x N2 estimator (ctx built with EST_IND)."""
        self._check_sums(sums, "evaluate_crossed")
        _check(lib().mc_evaluate_crossed(self._ctx, n1, n2, _stream(stream), sums.data_ptr()))
        return sums

    def finalize_crossed(self, sums, n1: int, n2: int, stream=None):
        torch = _torch()
        self._check_sums(sums, "finalize_crossed")
        mean = torch.empty(self.D, dtype=torch.float64, device=sums.device)
        var = torch.empty(self.D, dtype=torch.float64, device=sums.device)
        _check(lib().mc_finalize_crossed(self._ctx, sums.data_ptr(), n1, n2, mean.data_ptr(), var.data_ptr(),
                                         _stream(stream)))
        return mean, var

    def finalize(self, sums, total_samples: int, stream=None):
        """Row a8: per-design mean and per-draw variance (fp64 tensors)."""
        torch = _torch()
        self._check_sums(sums, "finalize")
        mean = torch.empty(self.D, dtype=torch.float64, device=sums.device)
        var = torch.empty(self.D, dtype=torch.float64, device=sums.device)
        _check(lib().mc_finalize(self._ctx, sums.data_ptr(), total_samples, mean.data_ptr(), var.data_ptr(),
                                 _stream(stream)))
        return mean, var

    def smooth_plan(self, fit_mask=None, stream=None, wait: bool = True):
        """Row a9 prep: the per-problem TPS eigenbasis (mc_smooth_plan).  wait=False builds it on a host
        thread (its own high-priority CUDA streams) so that it overlaps the Monte-Carlo pass; every call
        that needs the plan (smooth, tps_fit, refine, upload, close) joins it first."""
        m = None
        if fit_mask is not None:
            m = np.ascontiguousarray(fit_mask, dtype=np.uint8)
            assert m.size == self.D
        self._join_plan()
        self._mask_ref = m
        mp = None if m is None else m.ctypes.data_as(ctypes.c_void_p)
        if wait:
            _check(lib().mc_smooth_plan(self._ctx, mp, _stream(stream)))
            return
        import threading
        torch = _torch()
        # the caller's work so far (e.g. the design upload) is complete before the plan reads the table
        torch.cuda.current_stream(self.device).synchronize()
        ctx, dev = self._ctx, self.device
        self._plan_status = None

        def run():
            torch.cuda.set_device(dev)
            side = torch.cuda.Stream(device=dev)
            self._plan_status = (lib().mc_smooth_plan(ctx, mp, ctypes.c_void_p(side.cuda_stream)),
                                 lib().mc_last_error())

        self._plan_thread = threading.Thread(target=run, daemon=True)
        self._plan_thread.start()

    def _join_plan(self):
        t = getattr(self, "_plan_thread", None)
        if t is not None:
            t.join()
            self._plan_thread = None
            st, msg = self._plan_status
            if st != 0:
                raise McError(st, msg.decode() if isinstance(msg, bytes) else str(msg))

    def smooth(self, values, lam: float = -1.0, stream=None):
        """Row a9: TPS-smoothed values and the lambda used per problem."""
        self._join_plan()
        torch = _torch()
        out = torch.empty_like(values)
        lam_used = torch.empty(self.n_probs, dtype=torch.float64, device=values.device)
        _check(lib().mc_smooth(self._ctx, values.data_ptr(), float(lam), out.data_ptr(), lam_used.data_ptr(),
                               _stream(stream)))
        return out, lam_used

    def tps_fit(self, values, lam: float = -1.0, stream=None):
        self._join_plan()
        _check(lib().mc_tps_fit(self._ctx, values.data_ptr(), float(lam), _stream(stream)))

    def tps_eval(self, problem: int, x):
        x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
        f = np.zeros(x.shape[0])
        g = np.zeros_like(x)
        _check(lib().mc_tps_eval(self._ctx, problem, _dp(x), x.shape[0], _dp(f), _dp(g)))
        return f, g

    def refine(self, values, lam: float = -1.0, stream=None):
        """NEXT f1: per-problem continuous optimum on the TPS surface (alpha*, P~*, status)."""
        self._join_plan()
        A = np.zeros((self.n_probs, self.n))
        v = np.zeros(self.n_probs)
        st = np.zeros(self.n_probs, dtype=np.int32)
        _check(lib().mc_refine(self._ctx, values.data_ptr(), float(lam), _dp(A), _dp(v),
                               st.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _stream(stream)))
        return A, v, st

    # ---- multi-GPU smoothing: each rank plans and smooths the problems it owns (problem k -> rank k mod G) ----
    def owned_problems(self, rank: int, world: int) -> np.ndarray:
        return np.arange(self.n_probs) % world == rank

    def smooth_plan_sharded(self, rank: int, world: int, fit_mask=None, stream=None):
        """Row a9 prep across G ranks: this rank builds the TPS plans of the problems it owns (k mod G = rank);
        every other problem is masked out of the fit (a passthrough plan, no eigensolve).  G = 1: smooth_plan."""
        if world <= 1:
            return self.smooth_plan(fit_mask, stream)
        own = self.owned_problems(rank, world)[self.pod]
        m = own.astype(np.uint8) if fit_mask is None else (np.asarray(fit_mask, dtype=np.uint8) & own.astype(np.uint8))
        return self.smooth_plan(m, stream)

    def _combine_owned(self, t, rank: int, world: int, per_design: bool):
        """Sum over ranks of each rank's values for the problems it owns (zeros elsewhere): exactly the
        owner's values, on every rank (one all_reduce)."""
        import torch.distributed as dist
        torch = _torch()
        own = self.owned_problems(rank, world)
        mask = torch.from_numpy(own[self.pod] if per_design else own).to(t.device)
        if t.dim() == 2:
            mask = mask[:, None]
        out = torch.where(mask, t, torch.zeros_like(t))
        if dist.get_backend() == "gloo":
            host = out.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.SUM)
            return host.to(t.device)
        dist.all_reduce(out, op=dist.ReduceOp.SUM)
        return out

    def smooth_sharded(self, values, lam: float = -1.0, rank: int = 0, world: int = 1, stream=None):
        """Row a9 across G ranks (after smooth_plan_sharded): each rank smooths its own problems, one all_reduce
        assembles every problem's smoothed values and lambda on all ranks.  G = 1: smooth."""
        sm, lam_used = self.smooth(values, lam, stream)
        if world <= 1:
            return sm, lam_used
        return self._combine_owned(sm, rank, world, True), self._combine_owned(lam_used, rank, world, False)

    def refine_sharded(self, values, lam: float = -1.0, rank: int = 0, world: int = 1, stream=None):
        """NEXT f1 across G ranks: each rank runs L-BFGS on the TPS of its own problems; the optima are
        assembled on every rank by one all_reduce.  G = 1: refine."""
        A, v, st = self.refine(values, lam, stream)
        if world <= 1:
            return A, v, st
        torch = _torch()
        dev = values.device
        packed = torch.from_numpy(np.concatenate([A, v[:, None], st[:, None].astype(np.float64)], axis=1)).to(dev)
        packed = self._combine_owned(packed, rank, world, False).cpu().numpy()
        return packed[:, :self.n].copy(), packed[:, self.n].copy(), packed[:, self.n + 1].astype(np.int32)

    def argmax(self, values, with_host: bool = True, stream=None):
        """Row a10: per-problem argmax (device) and, if with_host, the overall (index, value)."""
        torch = _torch()
        idx = torch.empty(self.n_probs, dtype=torch.int64, device=values.device)
        val = torch.empty(self.n_probs, dtype=torch.float64, device=values.device)
        bi = ctypes.c_int64(-1)
        bv = ctypes.c_double(float("nan"))
        _check(lib().mc_argmax(self._ctx, values.data_ptr(), idx.data_ptr(), val.data_ptr(),
                               ctypes.byref(bi) if with_host else None, ctypes.byref(bv) if with_host else None,
                               _stream(stream)))
        return idx, val, (int(bi.value), float(bv.value)) if with_host else None

    def draw_dump(self, design, sample, stream=None):
        torch = _torch()
        design = design.to(torch.int64).contiguous()
        sample = sample.to(torch.int64).contiguous()
        stride = int(lib().mc_draw_dump_stride(self._ctx))
        out = torch.empty((design.numel(), stride), dtype=torch.float32, device=design.device)
        _check(lib().mc_draw_dump(self._ctx, design.data_ptr(), sample.data_ptr(), design.numel(), out.data_ptr(),
                                  _stream(stream)))
        return out


class Surface:
    """NEXT f2: host TPS through arbitrary points (the optimal power over the r-lattice)."""

    def __init__(self, x, y, lam: float = -1.0):
        x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
        if x.shape[0] == 1 and np.ndim(y) and len(y) > 1:
            x = x.T.copy()
        y = np.ascontiguousarray(y, dtype=np.float64)
        self.d = x.shape[1]
        h = ctypes.c_void_p()
        lu = ctypes.c_double(0.0)
        _check(lib().mc_surface_fit(_dp(x), x.shape[0], self.d, _dp(y), float(lam), ctypes.byref(h), ctypes.byref(lu)))
        self._h, self.lam = h, lu.value

    def __call__(self, x):
        x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
        f = np.zeros(x.shape[0])
        g = np.zeros_like(x)
        _check(lib().mc_surface_eval(self._h, _dp(x), x.shape[0], _dp(f), _dp(g)))
        return f, g

    def maximum(self):
        x = np.zeros(self.d)
        f = ctypes.c_double(0.0)
        _check(lib().mc_surface_max(self._h, _dp(x), ctypes.byref(f)))
        return x, f.value

    def __del__(self):
        try:
            if self._h:
                lib().mc_surface_destroy(self._h)
        except Exception:
            pass


def grid_smooth(values, xr, xa, hr: float = -1.0, ha: float = -1.0, out=None, stream=None):
    """Row a9 for dense regular grids (C4): separable Gaussian kernel smoother of values[nr, na] (a CUDA
    fp64 tensor, row i at xr[i], column j at xa[j]); hr, ha <= 0: GCV.  Returns (smoothed, (hr, ha))."""
    torch = _torch()
    if not (values.is_cuda and values.dtype == torch.float64 and values.dim() == 2):
        raise RuntimeError("grid_smooth: values must be a 2-D CUDA float64 tensor (no CPU fallback)")
    values = values.contiguous()
    nr, na = values.shape
    xr = np.ascontiguousarray(xr, dtype=np.float64)
    xa = np.ascontiguousarray(xa, dtype=np.float64)
    if xr.shape != (nr,) or xa.shape != (na,):
        raise ValueError("grid_smooth: coordinate lengths must match the grid")
    out = torch.empty_like(values) if out is None else out
    h = (ctypes.c_double * 2)()
    _check(lib().mc_grid_smooth(values.data_ptr(), nr, na, _dp(xr), _dp(xa), float(hr), float(ha), out.data_ptr(),
                                h, _stream(stream)))
    return out, (h[0], h[1])


# ------------------------------------------------------------------------------------------
# Multi-GPU: samples shard by rank; one all_reduce of the int64 sums (row a7).

def shard_range(total: int, rank: int, world: int, align: int = 64):
    """Rank `rank`'s sample range [begin, begin + count) of `total` samples: contiguous blocks
    in multiples of `align` (the last rank takes the remainder)."""
    per = (total // world) // align * align
    begin = rank * per
    count = per if rank < world - 1 else total - per * (world - 1)
    return begin, count


def allreduce_sums(sums):
    """Row a7: the single cross-GPU combine.  Integer SUM => bit-identical for any world size.  Over NCCL
    the device tensor is reduced in place; a gloo process group (CPU tests, bench --dist-backend gloo)
    reduces a host copy and writes it back."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        if sums.is_cuda and dist.get_backend() == "gloo":
            host = sums.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.SUM)
            sums.copy_(host)
        else:
            dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    return sums


@dataclass
class Result:
    mean: object
    var: object
    smoothed: object
    lam_used: object
    idx: object
    val: object
    best: tuple


def evaluate_design_objective(design: Design, total_samples: int, lam: float = -1.0, smooth: bool = True,
                              rank: int = 0, world: int = 1, stream=None) -> Result:
    """One pass of the whole hot path (rows a2-a10) for this rank's sample shard."""
    sums = design.new_sums()
    b, c = shard_range(total_samples, rank, world)
    design.evaluate(sums, b, c, stream=stream)
    allreduce_sums(sums)
    mean, var = design.finalize(sums, total_samples, stream=stream)
    if smooth:
        sm, lam_used = design.smooth(mean, lam, stream=stream)
    else:
        sm, lam_used = mean, None
    idx, val, best = design.argmax(sm, stream=stream)
    return Result(mean, var, sm, lam_used, idx, val, best)


# ------------------------------------------------------------------------------------------
# Checkpoint / resume: the integer sums add exactly, so a run is resumed by continuing the
# sample range from `samples_done` into the saved sums — bit-identical to an uninterrupted run.

def checkpoint_save(path: str, sums, samples_done: int, seed: int, meta: dict = None):
    import json as _json
    s = sums.detach().to("cpu").numpy() if hasattr(sums, "detach") else np.asarray(sums)
    np.savez(path, sums=s.astype(np.int64), samples_done=np.int64(samples_done), seed=np.uint64(seed),
             meta=np.array(_json.dumps(meta or {})))


def checkpoint_load(path: str):
    import json as _json
    z = np.load(path if path.endswith(".npz") else path + ".npz")
    return z["sums"], int(z["samples_done"]), int(z["seed"]), _json.loads(str(z["meta"]))
