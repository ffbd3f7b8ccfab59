// mc_surface.cu — NEXT f2: a thin-plate spline through a small set of points
// (the optimal powers of the r-lattice problems, "we fit TPS of optimal power as functions of r")
// and its box-constrained maximum.  Host fp64: the r-surface has O(100) sites (171 for the paper's
// lattice), so a dense solve per lambda is microseconds to milliseconds; GCV as in DESIGN.md §2.9.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "mc_internal.h"

struct mc_surface {
  int d = 0;
  int64_t N = 0;
  std::vector<double> X, w, beta;
  double lambda = 0.0;
};

namespace mci {

static double phi_d(double r, int d) {
  if (d == 1) return r * r * r;
  if (d == 2) return r > 0.0 ? r * r * std::log(r) : 0.0;
  return -r;
}

// Dense LU with partial pivoting: solves A X = B in place (A n x n row-major, B n x m row-major).
static bool lu_solve(std::vector<double>& A, std::vector<double>& B, int64_t n, int64_t m) {
  std::vector<int64_t> piv(n);
  for (int64_t k = 0; k < n; ++k) {
    int64_t p = k;
    for (int64_t i = k + 1; i < n; ++i)
      if (std::fabs(A[i * n + k]) > std::fabs(A[p * n + k])) p = i;
    if (std::fabs(A[p * n + k]) < 1e-300) return false;
    if (p != k) {
      for (int64_t j = 0; j < n; ++j) std::swap(A[k * n + j], A[p * n + j]);
      for (int64_t j = 0; j < m; ++j) std::swap(B[k * m + j], B[p * m + j]);
    }
    const double inv = 1.0 / A[k * n + k];
    for (int64_t i = k + 1; i < n; ++i) {
      const double f = A[i * n + k] * inv;
      if (f == 0.0) continue;
      for (int64_t j = k; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
      for (int64_t j = 0; j < m; ++j) B[i * m + j] -= f * B[k * m + j];
    }
  }
  for (int64_t k = n - 1; k >= 0; --k)
    for (int64_t j = 0; j < m; ++j) {
      double acc = B[k * m + j];
      for (int64_t i = k + 1; i < n; ++i) acc -= A[k * n + i] * B[i * m + j];
      B[k * m + j] = acc / A[k * n + k];
    }
  return true;
}

// The bordered TPS system [K + N lambda I, T; T^T, 0] with right-hand sides B ((N + d + 1) x m).
static bool tps_solve(const std::vector<double>& X, int64_t N, int d, double lam, std::vector<double>& B, int64_t m) {
  const int64_t k = d + 1, S = N + k;
  std::vector<double> A(S * S, 0.0);
  for (int64_t i = 0; i < N; ++i) {
    for (int64_t j = 0; j < N; ++j) {
      double r2 = 0.0;
      for (int c = 0; c < d; ++c) {
        const double t = X[i * d + c] - X[j * d + c];
        r2 += t * t;
      }
      A[i * S + j] = phi_d(std::sqrt(r2), d) + (i == j ? (double)N * lam : 0.0);
    }
    A[i * S + N] = A[N * S + i] = 1.0;
    for (int c = 0; c < d; ++c) A[i * S + N + 1 + c] = A[(N + 1 + c) * S + i] = X[i * d + c];
  }
  return lu_solve(A, B, S, m);
}

static double surface_eval(const mc_surface& s, const double* x, double* grad) {
  const int d = s.d;
  double f = s.beta[0];
  for (int j = 0; j < d; ++j) {
    f += s.beta[j + 1] * x[j];
    if (grad) grad[j] = s.beta[j + 1];
  }
  for (int64_t i = 0; i < s.N; ++i) {
    double diff[3], r2 = 0.0;
    for (int j = 0; j < d; ++j) { diff[j] = x[j] - s.X[i * d + j]; r2 += diff[j] * diff[j]; }
    const double r = std::sqrt(r2);
    double dpr;
    if (d == 1) dpr = 3.0 * r;
    else if (d == 2) dpr = r > 0.0 ? 2.0 * std::log(r) + 1.0 : 0.0;
    else dpr = r > 0.0 ? -1.0 / r : 0.0;
    f += s.w[i] * phi_d(r, d);
    if (grad) for (int j = 0; j < d; ++j) grad[j] += s.w[i] * dpr * diff[j];
  }
  return f;
}

}  // namespace mci

using namespace mci;

extern "C" {

mc_status mc_surface_fit(const double* x, int64_t N, int32_t d, const double* y, double lambda, mc_surface** out,
                         double* lambda_used) {
  if (!x || !y || !out || d < 1 || d > 3 || N < d + 2) {
    set_error("mc_surface_fit: null pointer, d outside [1,3] or fewer than d + 2 points");
    return MC_ERR_INVALID;
  }
  const int64_t k = d + 1, S = N + k;
  std::vector<double> X(x, x + N * d);
  double lam = lambda;
  if (lambda < 0.0) {
    // GCV: V(lambda) = N |(I - A) y|^2 / tr(I - A)^2, A the influence matrix (identity right-hand sides)
    double best = INFINITY;
    for (int g = 0; g < 49; ++g) {
      const double l = std::pow(10.0, -12.0 + 0.25 * g);
      std::vector<double> B(S * N, 0.0);
      for (int64_t i = 0; i < N; ++i) B[i * N + i] = 1.0;
      if (!tps_solve(X, N, d, l, B, N)) continue;
      // fitted = y - N l w, so (I - A) = N l W with W = rows 0..N-1 of the solution
      double tr = 0.0, rss = 0.0;
      for (int64_t i = 0; i < N; ++i) {
        tr += (double)N * l * B[i * N + i];
        double ri = 0.0;
        for (int64_t j = 0; j < N; ++j) ri += B[i * N + j] * y[j];
        ri *= (double)N * l;
        rss += ri * ri;
      }
      const double v = (double)N * rss / (tr * tr);
      if (v < best) { best = v; lam = l; }
    }
  }
  std::vector<double> B(S, 0.0);
  for (int64_t i = 0; i < N; ++i) B[i] = y[i];
  if (!tps_solve(X, N, d, lam, B, 1)) {
    set_error("mc_surface_fit: singular TPS system (coincident or collinear sites)");
    return MC_ERR_NUMERIC;
  }
  mc_surface* s = new mc_surface();
  s->d = d;
  s->N = N;
  s->X = X;
  s->w.assign(B.begin(), B.begin() + N);
  s->beta.assign(B.begin() + N, B.end());
  s->lambda = lam;
  if (lambda_used) *lambda_used = lam;
  *out = s;
  return MC_OK;
}

mc_status mc_surface_eval(const mc_surface* s, const double* x, int64_t q, double* f, double* grad) {
  if (!s || (q > 0 && (!x || !f))) { set_error("mc_surface_eval: null pointer"); return MC_ERR_INVALID; }
  for (int64_t i = 0; i < q; ++i) f[i] = surface_eval(*s, x + i * s->d, grad ? grad + i * s->d : nullptr);
  return MC_OK;
}

mc_status mc_surface_max(const mc_surface* s, double* x_out, double* f_out) {
  if (!s || !x_out || !f_out) { set_error("mc_surface_max: null pointer"); return MC_ERR_INVALID; }
  const int d = s->d;
  std::vector<double> lo(d, INFINITY), hi(d, -INFINITY), x0(d);
  double best = -INFINITY;
  for (int64_t i = 0; i < s->N; ++i) {
    const double fi = surface_eval(*s, &s->X[i * d], nullptr);
    if (fi > best) { best = fi; for (int j = 0; j < d; ++j) x0[j] = s->X[i * d + j]; }
    for (int j = 0; j < d; ++j) { lo[j] = std::min(lo[j], s->X[i * d + j]); hi[j] = std::max(hi[j], s->X[i * d + j]); }
  }
  std::vector<double> beta = s->beta;
  const RefineOut r = refine_box(s->X, s->w, beta, d, x0, lo, hi);
  for (int j = 0; j < d; ++j) x_out[j] = r.x[j];
  *f_out = r.f;
  return MC_OK;
}

void mc_surface_destroy(mc_surface* s) { delete s; }

}  // extern "C"
