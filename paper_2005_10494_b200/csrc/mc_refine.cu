// mc_refine.cu — NEXT f1: the continuous optimum on the smoothed surface.
//
// P:123 re-parametrises the constrained problem into (alpha_1..alpha_{n-1}) and applies L-BFGS-B;
// P:219 starts it from the fitted design with the largest P~ and evaluates the TPS surface and its
// derivatives "with no error".  Here: the TPS coefficients come from the GPU (mc_smooth.cu
// tps_coefficients), the box-constrained limited-memory quasi-Newton (projected L-BFGS, memory 10,
// Armijo backtracking on the projected path) runs on the host per problem (threads over problems),
// and alpha_n is re-solved from Formula 2 on the GPU (K4).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "mc_internal.h"

namespace mci {

// TPS surface f(x) = beta_0 + beta_{1..d} x + sum_i w_i phi(|x - x_i|) and its gradient.
static double tps_value_grad(const std::vector<double>& X, const std::vector<double>& w, const std::vector<double>& beta,
                             int d, const double* x, double* grad) {
  double f = beta[0];
  for (int j = 0; j < d; ++j) {
    f += beta[j + 1] * x[j];
    if (grad) grad[j] = beta[j + 1];
  }
  const int64_t N = (int64_t)w.size();
  for (int64_t i = 0; i < N; ++i) {
    double diff[3], r2 = 0.0;
    for (int j = 0; j < d; ++j) {
      diff[j] = x[j] - X[i * d + j];
      r2 += diff[j] * diff[j];
    }
    const double r = std::sqrt(r2);
    double phi, dphi_over_r;   // phi(r) and phi'(r)/r
    if (d == 1) { phi = r2 * r; dphi_over_r = 3.0 * r; }
    else if (d == 2) {
      if (r > 0.0) { const double lr = std::log(r); phi = r2 * lr; dphi_over_r = 2.0 * lr + 1.0; }
      else { phi = 0.0; dphi_over_r = 0.0; }
    } else { phi = -r; dphi_over_r = r > 0.0 ? -1.0 / r : 0.0; }
    f += w[i] * phi;
    if (grad)
      for (int j = 0; j < d; ++j) grad[j] += w[i] * dphi_over_r * diff[j];
  }
  return f;
}


// maximise f over lo <= x <= hi from x0: projected L-BFGS (m = 10) with Armijo backtracking on the
// projected path; stops on |projected gradient|_inf <= 1e-10, relative change <= 1e-15, or 500 iterations
// (SPEC: L-BFGS-B).
RefineOut refine_box(const std::vector<double>& X, const std::vector<double>& w,
                               const std::vector<double>& beta, int d, const std::vector<double>& x0,
                               const std::vector<double>& lo, const std::vector<double>& hi) {
  const int M = 10;
  std::vector<double> x = x0, G(d), xn(d), Gn(d), dir(d), q(d);
  auto proj = [&](std::vector<double>& v) {
    for (int j = 0; j < d; ++j) v[j] = std::min(hi[j], std::max(lo[j], v[j]));
  };
  proj(x);
  // minimise g = -f
  double g = -tps_value_grad(X, w, beta, d, x.data(), G.data());
  for (int j = 0; j < d; ++j) G[j] = -G[j];
  std::vector<std::vector<double>> S, Y;
  std::vector<double> rho;
  int it = 0;
  for (; it < 500; ++it) {
    double pgn = 0.0;
    std::vector<bool> free_(d);
    for (int j = 0; j < d; ++j) {
      const double pj = std::min(hi[j], std::max(lo[j], x[j] - G[j])) - x[j];
      pgn = std::max(pgn, std::fabs(pj));
      free_[j] = !((x[j] <= lo[j] && G[j] > 0.0) || (x[j] >= hi[j] && G[j] < 0.0));
    }
    if (pgn <= 1e-10) break;
    // two-loop recursion on the free coordinates
    for (int j = 0; j < d; ++j) q[j] = free_[j] ? G[j] : 0.0;
    const int k = (int)S.size();
    std::vector<double> al(k);
    for (int i = k - 1; i >= 0; --i) {
      double sq = 0.0;
      for (int j = 0; j < d; ++j) if (free_[j]) sq += S[i][j] * q[j];
      al[i] = rho[i] * sq;
      for (int j = 0; j < d; ++j) if (free_[j]) q[j] -= al[i] * Y[i][j];
    }
    if (k > 0) {
      double sy = 0.0, yy = 0.0;
      for (int j = 0; j < d; ++j) { sy += S[k - 1][j] * Y[k - 1][j]; yy += Y[k - 1][j] * Y[k - 1][j]; }
      const double gam = yy > 0.0 ? sy / yy : 1.0;
      for (int j = 0; j < d; ++j) q[j] *= gam;
    }
    for (int i = 0; i < k; ++i) {
      double yq = 0.0;
      for (int j = 0; j < d; ++j) if (free_[j]) yq += Y[i][j] * q[j];
      const double b = rho[i] * yq;
      for (int j = 0; j < d; ++j) if (free_[j]) q[j] += S[i][j] * (al[i] - b);
    }
    double gd = 0.0;
    for (int j = 0; j < d; ++j) {
      dir[j] = free_[j] ? -q[j] : 0.0;
      gd += G[j] * dir[j];
    }
    if (!(gd < 0.0)) {
      for (int j = 0; j < d; ++j) dir[j] = free_[j] ? -G[j] : 0.0;
      S.clear(); Y.clear(); rho.clear();
    }
    double t = 1.0, gn = g;
    bool ok = false;
    for (int ls = 0; ls < 60; ++ls) {
      for (int j = 0; j < d; ++j) xn[j] = x[j] + t * dir[j];
      proj(xn);
      gn = -tps_value_grad(X, w, beta, d, xn.data(), Gn.data());
      double dec = 0.0;
      for (int j = 0; j < d; ++j) dec += G[j] * (xn[j] - x[j]);
      if (gn <= g + 1e-4 * dec) { ok = true; break; }
      t *= 0.5;
    }
    if (!ok) break;
    for (int j = 0; j < d; ++j) Gn[j] = -Gn[j];
    std::vector<double> s(d), yv(d);
    double sy = 0.0;
    for (int j = 0; j < d; ++j) { s[j] = xn[j] - x[j]; yv[j] = Gn[j] - G[j]; sy += s[j] * yv[j]; }
    const double change = std::fabs(g - gn);
    x = xn; G = Gn;
    const double gold = g;
    g = gn;
    if (sy > 1e-300) {
      S.push_back(s); Y.push_back(yv); rho.push_back(1.0 / sy);
      if ((int)S.size() > M) { S.erase(S.begin()); Y.erase(Y.begin()); rho.erase(rho.begin()); }
    }
    if (change <= 1e-15 * std::max(1.0, std::fabs(gold))) { ++it; break; }
  }
  RefineOut r;
  r.x = x;
  r.f = -g;
  r.iters = it;
  return r;
}

}  // namespace mci

using namespace mci;

extern "C" {

mc_status mc_tps_fit(mc_ctx* c, const double* values, double lambda, void* stream) {
  if (!c || !values) { set_error("mc_tps_fit: null pointer"); return MC_ERR_INVALID; }
  MC_CUDA(cudaSetDevice(c->device));
  return tps_coefficients(c, values, lambda, (cudaStream_t)stream);
}

mc_status mc_tps_eval(const mc_ctx* c, int32_t problem, const double* x, int64_t q, double* f, double* grad) {
  if (!c || problem < 0 || problem >= c->n_probs || (q > 0 && (!x || !f))) {
    set_error("mc_tps_eval: null pointer or problem out of range");
    return MC_ERR_INVALID;
  }
  if ((int)c->tps_w.size() != c->n_probs || c->tps_w[problem].empty()) {
    set_error("mc_tps_eval: no TPS fitted for this problem (call mc_tps_fit or mc_refine first)");
    return MC_ERR_INVALID;
  }
  const int d = c->n - 1;
  for (int64_t i = 0; i < q; ++i)
    f[i] = tps_value_grad(c->tps_x[problem], c->tps_w[problem], c->tps_beta[problem], d, x + i * d,
                          grad ? grad + i * d : nullptr);
  return MC_OK;
}

mc_status mc_refine(mc_ctx* c, const double* values, double lambda, double* alpha_out, double* value_out,
                    int32_t* status_out, void* stream) {
  if (!c || !values || !alpha_out || !value_out || !status_out) {
    set_error("mc_refine: null pointer");
    return MC_ERR_INVALID;
  }
  MC_CUDA(cudaSetDevice(c->device));
  mc_status s = tps_coefficients(c, values, lambda, (cudaStream_t)stream);
  if (s != MC_OK) return s;
  const int n = c->n, d = n - 1;
  std::vector<double> hv(c->D);
  MC_CUDA(cudaMemcpy(hv.data(), values, sizeof(double) * c->D, cudaMemcpyDeviceToHost));
  std::vector<RefineOut> res(c->n_probs);
  std::vector<int> todo;
  for (int k = 0; k < c->n_probs; ++k) {
    const int64_t b = c->prob_begin[k], e = c->prob_begin[k + 1];
    if (c->tps_w[k].empty()) {
      // no surface: the best evaluated design
      int64_t best = -1;
      for (int64_t i = b; i < e; ++i)
        if (!(hv[i] != hv[i]) && (best < 0 || hv[i] > hv[best])) best = i;
      status_out[k] = 2;
      for (int i = 0; i < n; ++i) alpha_out[k * n + i] = best >= 0 ? c->alpha[best * n + i] : NAN;
      value_out[k] = best >= 0 ? hv[best] : NAN;
    } else {
      todo.push_back(k);
    }
  }
  auto work = [&](size_t t0, size_t stride) {
    for (size_t t = t0; t < todo.size(); t += stride) {
      const int k = todo[t];
      const auto& X = c->tps_x[k];
      const auto& w = c->tps_w[k];
      const auto& beta = c->tps_beta[k];
      const int64_t N = (int64_t)w.size();
      // start: the fitted site with the largest P~, from the TPS values at the sites y - N lambda w
      // (O(N); evaluating the spline at every site would be O(N^2)); box: the candidate box of the sites
      const auto& fv = c->tps_fitted[k];
      std::vector<double> lo(d, INFINITY), hi(d, -INFINITY), x0(d);
      double bestf = -INFINITY;
      for (int64_t i = 0; i < N; ++i) {
        if (fv[i] > bestf) { bestf = fv[i]; for (int j = 0; j < d; ++j) x0[j] = X[i * d + j]; }
        for (int j = 0; j < d; ++j) { lo[j] = std::min(lo[j], X[i * d + j]); hi[j] = std::max(hi[j], X[i * d + j]); }
      }
      res[k] = refine_box(X, w, beta, d, x0, lo, hi);
    }
  };
  const size_t nt = std::max<size_t>(1, std::min<size_t>(todo.size(), std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (size_t t = 1; t < nt; ++t) th.emplace_back(work, t, nt);
  work(0, nt);
  for (auto& t : th) t.join();
  if (!todo.empty()) {
    std::vector<double> A(todo.size() * n);
    std::vector<int32_t> pidx(todo.size());
    std::vector<uint8_t> ok(todo.size());
    for (size_t t = 0; t < todo.size(); ++t) {
      const int k = todo[t];
      pidx[t] = k;
      for (int j = 0; j < d; ++j) A[t * n + j] = res[k].x[j] * c->probs[k].alpha0;
      A[t * n + n - 1] = 0.0;
    }
    s = alpha_points_solve(c->probs.data(), c->n_probs, pidx.data(), (int64_t)todo.size(), c->device, A.data(), ok.data());
    if (s != MC_OK) return s;
    for (size_t t = 0; t < todo.size(); ++t) {
      const int k = todo[t];
      for (int i = 0; i < n; ++i) alpha_out[k * n + i] = A[t * n + i];
      value_out[k] = res[k].f;
      status_out[k] = ok[t] ? 0 : 1;
    }
  }
  return MC_OK;
}

}  // extern "C"
