// mc_api.cu — host side of the C ABI (include/mc_design.h): validation, fp64 design prep (row a1),
// context lifetime and the launches of the device stages.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "mc_internal.h"
#include <nvtx3/nvToolsExt.h>

namespace mci {

// NVTX range for the duration of a C-ABI call (visible in Nsight / ncu --nvtx); header-only NVTX3.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

mc_status cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? MC_ERR_OOM : MC_ERR_CUDA;
}

// ---------------------------------------------------------------------------------------------
// fp64 standard normal quantile for the thresholds Z_{1-alpha}: Acklam's rational
// approximation (relative error < 1.2e-9) polished by one Halley step on erfc (full double).
static double norm_quantile(double p) {
  if (!(p > 0.0)) return -INFINITY;
  if (!(p < 1.0)) return INFINITY;
  static const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                              1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                              6.680131188771972e+01,  -1.328068155288572e+01};
  static const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                              -2.549732539343734e+00, 4.374664141464968e+00,  2.938163982698783e+00};
  static const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                              3.754408661907416e+00};
  const double plow = 0.02425;
  double x;
  if (p < plow) {
    const double q = std::sqrt(-2.0 * std::log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else if (p <= 1.0 - plow) {
    const double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  } else {
    const double q = std::sqrt(-2.0 * std::log1p(-p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  // Halley step on F(x) = Phi(x) - p, evaluated on the smaller tail to avoid cancellation.
  for (int it = 0; it < 2; ++it) {
    double e;
    if (x < 0) e = 0.5 * std::erfc(-x / std::sqrt(2.0)) - p;
    else e = (1.0 - p) - 0.5 * std::erfc(x / std::sqrt(2.0));
    const double u = e * std::sqrt(2.0 * M_PI) * std::exp(0.5 * x * x);
    x = x - u / (1.0 + 0.5 * x * u);
  }
  return x;
}

// Z_{1-alpha} = -Phi^{-1}(alpha) (upper tail, no cancellation for small alpha).
static double threshold(double alpha) {
  if (alpha == 0.0) return INFINITY;
  return -norm_quantile(alpha);
}

static mc_status validate_problem(const mc_problem& p, int idx) {
  char buf[256];
  auto bad = [&](const char* what) {
    snprintf(buf, sizeof buf, "problem %d: %s", idx, what);
    set_error(buf);
    return MC_ERR_INVALID;
  };
  if (p.n < 1 || p.n > MC_MAX_N) return bad("n must be in [1, 10] (P:47)");
  if (p.model != 0 && p.model != 1) return bad("model must be 0 (Gaussian prior) or 1 (C4 strata prior)");
  if (p.model == 1) {
    if (p.n != 2) return bad("the C4 strata prior has n = 2");
    for (int k = 0; k < 10; ++k)
      if (!std::isfinite(p.strata[k]) || (k % 2 == 1 && !(p.strata[k] >= 0.0)))
        return bad("strata parameters must be finite with sd >= 0");
  }
  if (p.r[0] != 1.0) return bad("r[0] must be exactly 1 (P:47: 1 = r_1 > r_2 > ...)");
  for (int i = 0; i + 1 < p.n; ++i) {
    if (!(p.r[i + 1] > 0.0) || !(p.r[i + 1] < p.r[i])) return bad("r must be strictly decreasing and > 0 (P:47)");
    if (p.r[i + 1] / p.r[i] > 1.0 - 1e-6) return bad("adjacent ratio r[i+1]/r[i] > 1 - 1e-6: Sigma0 near-singular (S:32)");
  }
  if (!(p.alpha0 > 0.0 && p.alpha0 < 0.5)) return bad("alpha0 must be in (0, 0.5) (Formula 2)");
  if (!(p.i3 > 0.0) || !std::isfinite(p.i3)) return bad("i3 must be finite and > 0 (Eq. 9)");
  for (int i = 0; i < p.n && p.model == 0; ++i) {
    if (!std::isfinite(p.theta[i])) return bad("theta must be finite (Formula 10)");
    if (!p.has_prior_chol && !(p.sigma[i] >= 0.0 && std::isfinite(p.sigma[i])))
      return bad("sigma must be finite and >= 0 (Formula 10)");
  }
  if (p.has_prior_chol && p.model == 0) {
    for (int i = 0; i < p.n; ++i) {
      if (!(p.prior_chol[i * MC_MAX_N + i] >= 0.0)) return bad("prior_chol diagonal must be >= 0");
      for (int j = 0; j <= i; ++j)
        if (!std::isfinite(p.prior_chol[i * MC_MAX_N + j])) return bad("prior_chol must be finite");
    }
  }
  return MC_OK;
}

constexpr double BM_K = 1.17741002251547469;   // sqrt(2 ln 2), see mc_device.cuh
constexpr double PHI_SCALE = 0.84932180028801904;   // sqrt(log2(e) / 2): COND carries every normal-CDF
                                                     // argument pre-scaled by it (mc_device.cuh normal_tail)

// COND stage coefficients of the SOV order (2, 4, ..., 1, 3, ...) for the Formula-1 Markov chain
// (A.1): X_{j+1} = rho_j X_j + s_j W (0-based j).  Even populations (0-based p = 2k+1) form the chain
// X_p | X_{p-2} ~ N(mu x, sd^2), mu = rho_{p-2} rho_{p-1}; odd ones (p = 2j) are Gaussian bridges
// X_p | X_{p-1} = a, X_{p+1} = c ~ N(alpha a + beta c, gamma^2).  Returns the conditional sd of
// population p's stage (its row scale is 1/sd) and the stage coefficients.
struct SovCoef {
  double sd[MC_MAX_N];                      // per population
  double emu[MC_MAX_N], esd[MC_MAX_N];      // even stages
  double oa[MC_MAX_N], ob[MC_MAX_N];        // odd stages: alpha, beta (unscaled)
};

static SovCoef sov_coef(const mc_problem& p) {
  const int n = p.n;
  double rho[MC_MAX_N] = {0}, s[MC_MAX_N] = {0};
  for (int i = 0; i + 1 < n; ++i) {
    rho[i] = std::sqrt(p.r[i + 1] / p.r[i]);
    s[i] = std::sqrt(1.0 - p.r[i + 1] / p.r[i]);
  }
  SovCoef c{};
  for (int k = 0; 2 * k + 1 < n; ++k) {
    const int q = 2 * k + 1;
    if (k == 0) { c.emu[k] = 0.0; c.esd[k] = 1.0; }
    else {
      const double mu = rho[q - 2] * rho[q - 1];
      c.emu[k] = mu;
      c.esd[k] = std::sqrt(1.0 - mu * mu);
    }
    c.sd[q] = c.esd[k];
  }
  for (int j = 0; 2 * j < n; ++j) {
    const int q = 2 * j;
    const bool L = q >= 1, R = q + 1 < n;
    double a = 0.0, bb = 0.0, g = 1.0;
    if (L && R) {
      const double prec = 1.0 / (s[q - 1] * s[q - 1]) + rho[q] * rho[q] / (s[q] * s[q]);
      const double g2 = 1.0 / prec;
      a = rho[q - 1] / (s[q - 1] * s[q - 1]) * g2;
      bb = rho[q] / (s[q] * s[q]) * g2;
      g = std::sqrt(g2);
    } else if (R) {             // q = 0: X_0 | X_1 = c ~ N(rho_0 c, s_0^2)
      bb = rho[0];
      g = s[0];
    } else if (L) {             // last population, n odd: X_q | X_{q-1} = a ~ N(rho_{q-1} a, s_{q-1}^2)
      a = rho[q - 1];
      g = s[q - 1];
    }
    c.oa[j] = a;
    c.ob[j] = bb;
    c.sd[q] = g;
  }
  return c;
}

// Row scale of b folded into the record and the thresholds (mc_device.cuh ProbRegs).
static double row_scale(const mc_problem& p, int est, int i) {
  if (est == MC_EST_IND) return 1.0 / BM_K;
  return PHI_SCALE / sov_coef(p).sd[i];
}

// Per-problem device record (fp32): M = diag(c) L_p packed with the folded scales, the IND Markov
// coefficients, the COND stage coefficients and the row scales (Formula 1/3/10, A.1).
static void problem_record(const mc_problem& p, int est, float* rec) {
  const int n = p.n;
  double rho[MC_MAX_N] = {0}, sd[MC_MAX_N] = {0};
  for (int i = 0; i + 1 < n; ++i) {
    rho[i] = std::sqrt(p.r[i + 1] / p.r[i]);
    sd[i] = std::sqrt(1.0 - p.r[i + 1] / p.r[i]);
  }
  // L0: Cholesky factor of the Markov correlation: X_{i+1} = rho_i X_i + s_i W_{i+1}.
  double L0[MC_MAX_N][MC_MAX_N] = {{0}};
  L0[0][0] = 1.0;
  for (int i = 1; i < n; ++i) {
    for (int j = 0; j < i; ++j) L0[i][j] = rho[i - 1] * L0[i - 1][j];
    L0[i][i] = sd[i - 1];
  }
  double Lp[MC_MAX_N][MC_MAX_N] = {{0}};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j)
      Lp[i][j] = p.has_prior_chol ? p.prior_chol[i * MC_MAX_N + j] : p.sigma[i] * L0[i][j];
  const SovCoef sc = sov_coef(p);
  std::fill(rec, rec + PROB_STRIDE, 0.0f);
  for (int i = 0; i < n; ++i) {
    const double c = std::sqrt(p.r[i] * p.i3);
    // the kernel draws eps / BM_K: M carries BM_K times the row scale (= 1 for IND)
    const double f = est == MC_EST_IND ? 1.0 : BM_K * row_scale(p, est, i);
    for (int j = 0; j <= i; ++j) rec[OFF_M + i * (i + 1) / 2 + j] = (float)(f * c * Lp[i][j]);
    rec[OFF_BSC + i] = (float)row_scale(p, est, i);
  }
  for (int i = 0; i + 1 < n; ++i) {
    rec[OFF_RHO + i] = (float)rho[i];
    rec[OFF_SD + i] = (float)sd[i];
  }
  for (int k = 0; 2 * k + 1 < n; ++k) {
    rec[OFF_ER + k] = (float)(PHI_SCALE * sc.emu[k] / sc.esd[k]);
    rec[OFF_EMU + k] = (float)sc.emu[k];
    rec[OFF_ESD + k] = (float)sc.esd[k];
  }
  for (int j = 0; 2 * j < n; ++j) {
    rec[OFF_OA + j] = (float)(PHI_SCALE * sc.oa[j] / sc.sd[2 * j]);
    rec[OFF_OB + j] = (float)(PHI_SCALE * sc.ob[j] / sc.sd[2 * j]);
  }
  if (p.model == 1) {
    // C4 strata prior: the kernel draws eps / BM_K, so every sd carries BM_K
    float* r = rec + OFF_STR;
    for (int k = 0; k < 10; ++k) r[k] = (float)(k % 2 == 1 ? BM_K * p.strata[k] : p.strata[k]);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) rec[OFF_M + i * (i + 1) / 2 + j] = 0.0f;
    const double r2 = p.r[1];
    r[10] = (float)p.i3;
    r[11] = (float)(1.0 / r2);
    r[12] = (float)(1.0 / (1.0 - r2));
    r[13] = (float)r2;
    r[14] = (float)std::sqrt(r2);
    r[15] = (float)row_scale(p, est, 0);
    r[16] = (float)row_scale(p, est, 1);
  }
}

}  // namespace mci

using namespace mci;

extern "C" {

const char* mc_last_error(void) { return g_err.c_str(); }
const char* mc_version(void) { return "mc_design 0.1 (sm_100a)"; }

double mc_threshold(double alpha) {
  if (!(alpha >= 0.0 && alpha < 1.0)) return NAN;
  return threshold(alpha);
}

double mc_information_units(double alpha, double beta, double delta) {
  if (!(alpha > 0 && alpha < 1 && beta > 0 && beta < 1 && delta > 0 && delta < 1)) return NAN;
  const double za = -norm_quantile(alpha), zb = -norm_quantile(beta);
  const double l = std::log1p(-delta);
  return (za + zb) * (za + zb) / (l * l);
}

mc_status mc_problem_formula10(int32_t n, const double* r, const double* delta0, double i3, double alpha0,
                               mc_problem* out) {
  if (!out || !r || !delta0 || n < 1 || n > MC_MAX_N) {
    set_error("mc_problem_formula10: null pointer or n out of [1, 10]");
    return MC_ERR_INVALID;
  }
  mc_problem p;
  std::memset(&p, 0, sizeof p);
  p.n = n;
  p.i3 = i3;
  p.alpha0 = alpha0;
  for (int i = 0; i < n; ++i) {
    if (!(delta0[i] > 0.0 && delta0[i] < 1.0)) {
      set_error("mc_problem_formula10: Delta0 must be in (0,1) (Formula 10)");
      return MC_ERR_INVALID;
    }
    p.r[i] = r[i];
    p.theta[i] = -std::log1p(-delta0[i]);               // theta_i = -log(1 - Delta0_i)
    p.sigma[i] = 1.0 / std::sqrt(80.0 * r[i] / 4.0);    // sigma_i = 1/sqrt(80 r_i / 4)
  }
  mc_status s = validate_problem(p, 0);
  if (s != MC_OK) return s;
  *out = p;
  return MC_OK;
}

mc_status mc_problem_strata(double r2, double i3, double alpha0, const double* strata, mc_problem* out) {
  if (!out || !strata) { set_error("mc_problem_strata: null pointer"); return MC_ERR_INVALID; }
  mc_problem p;
  std::memset(&p, 0, sizeof p);
  p.n = 2;
  p.model = 1;
  p.i3 = i3;
  p.alpha0 = alpha0;
  p.r[0] = 1.0;
  p.r[1] = r2;
  for (int k = 0; k < 10; ++k) p.strata[k] = strata[k];
  mc_status s = validate_problem(p, 0);
  if (s != MC_OK) return s;
  *out = p;
  return MC_OK;
}

mc_status mc_design_init(mc_ctx** ctx, const mc_problem* probs, int32_t n_probs, const double* alpha,
                         const int32_t* pod, int64_t D, uint64_t seed, int32_t estimator, int32_t device) {
  NvtxRange _nvtx("mc_design_init");
  if (!ctx || !probs || n_probs <= 0 || D < 0 || (D > 0 && (!alpha || !pod))) {
    set_error("mc_design_init: null pointer or empty problem list");
    return MC_ERR_INVALID;
  }
  if (estimator != MC_EST_COND && estimator != MC_EST_IND) {
    set_error("mc_design_init: estimator must be MC_EST_COND or MC_EST_IND");
    return MC_ERR_INVALID;
  }
  if (D >= (int64_t)1 << 32) {
    set_error("mc_design_init: D must be < 2^32 (the design index is a 32-bit Philox counter word)");
    return MC_ERR_INVALID;
  }
  const int n = probs[0].n;
  for (int k = 0; k < n_probs; ++k) {
    mc_status s = validate_problem(probs[k], k);
    if (s != MC_OK) return s;
    if (probs[k].n != n || probs[k].model != probs[0].model) {
      set_error("mc_design_init: all problems must share n and the prior model");
      return MC_ERR_INVALID;
    }
  }
  std::vector<int64_t> begin(n_probs + 1, 0);
  for (int64_t d = 0; d < D; ++d) {
    if (pod[d] < 0 || pod[d] >= n_probs || (d > 0 && pod[d] < pod[d - 1])) {
      set_error("mc_design_init: problem_of_design must be non-decreasing and in [0, n_probs)");
      return MC_ERR_INVALID;
    }
    const mc_problem& p = probs[pod[d]];
    for (int i = 0; i < n; ++i) {
      const double a = alpha[d * n + i];
      if (!(a >= 0.0 && a <= p.alpha0)) {
        char buf[160];
        snprintf(buf, sizeof buf, "mc_design_init: design %lld alpha[%d] = %g outside [0, alpha0] (P:221)",
                 (long long)d, i, a);
        set_error(buf);
        return MC_ERR_INVALID;
      }
    }
    begin[pod[d] + 1] += 1;
  }
  for (int k = 0; k < n_probs; ++k) begin[k + 1] += begin[k];

  MC_CUDA(cudaSetDevice(device));
  mc_ctx* c = new mc_ctx();
  c->device = device;
  c->n = n;
  c->est = estimator;
  c->model = probs[0].model;
  c->n_probs = n_probs;
  c->D = D;
  c->seed = seed;
  c->probs.assign(probs, probs + n_probs);
  c->alpha.assign(alpha, alpha + D * n);
  c->pod.assign(pod, pod + D);
  c->prob_begin = begin;

  std::vector<float> rec((size_t)n_probs * PROB_STRIDE);
  for (int k = 0; k < n_probs; ++k) problem_record(probs[k], estimator, &rec[(size_t)k * PROB_STRIDE]);
  std::vector<double> ctheta((size_t)n_probs * n * 2);
  for (int k = 0; k < n_probs; ++k)
    for (int i = 0; i < n; ++i) {
      ctheta[((size_t)k * n + i) * 2] =
          probs[k].model == 1 ? 0.0 : std::sqrt(probs[k].r[i] * probs[k].i3) * probs[k].theta[i];
      ctheta[((size_t)k * n + i) * 2 + 1] = row_scale(probs[k], estimator, i);
    }
  auto fail = [&](cudaError_t e, const char* w) { mc_status s = cuda_fail(e, w); mc_destroy(c); return s; };
  cudaError_t e;
  if ((e = cudaMalloc(&c->d_prob, rec.size() * sizeof(float))) != cudaSuccess) return fail(e, "cudaMalloc prob");
  const size_t Dn = (size_t)std::max<int64_t>(D, 1) * n;
  if ((e = cudaMalloc(&c->d_zc, Dn * sizeof(float))) != cudaSuccess) return fail(e, "cudaMalloc zc");
  if ((e = cudaMalloc(&c->d_alpha, Dn * sizeof(double))) != cudaSuccess) return fail(e, "cudaMalloc alpha");
  if ((e = cudaMalloc(&c->d_ctheta, ctheta.size() * sizeof(double))) != cudaSuccess) return fail(e, "cudaMalloc ctheta");
  if ((e = cudaMalloc(&c->d_pod, std::max<int64_t>(D, 1) * sizeof(int32_t))) != cudaSuccess) return fail(e, "cudaMalloc pod");
  if ((e = cudaMalloc(&c->d_prob_begin, begin.size() * sizeof(int64_t))) != cudaSuccess) return fail(e, "cudaMalloc begin");
  if ((e = cudaMemcpy(c->d_prob, rec.data(), rec.size() * sizeof(float), cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(e, "upload prob");
  if (D > 0 && (e = cudaMemcpy(c->d_alpha, alpha, (size_t)D * n * sizeof(double), cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(e, "upload alpha");
  if ((e = cudaMemcpy(c->d_ctheta, ctheta.data(), ctheta.size() * sizeof(double), cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(e, "upload ctheta");
  if (D > 0 && (e = cudaMemcpy(c->d_pod, pod, D * sizeof(int32_t), cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(e, "upload pod");
  if ((e = cudaMemcpy(c->d_prob_begin, begin.data(), begin.size() * sizeof(int64_t), cudaMemcpyHostToDevice)) !=
      cudaSuccess)
    return fail(e, "upload begin");
  {
    mc_status s = launch_zc(c, nullptr);
    if (s != MC_OK) { mc_destroy(c); return s; }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail(e, "k_zc");
  }
  c->launches = 0;
  *ctx = c;
  return MC_OK;
}

mc_status mc_design_upload(mc_ctx* c, const double* alpha, void* stream) {
  NvtxRange _nvtx("mc_design_upload");
  if (!c || (c->D > 0 && !alpha)) { set_error("mc_design_upload: null pointer"); return MC_ERR_INVALID; }
  const int n = c->n;
  for (int64_t d = 0; d < c->D; ++d) {
    const double a0 = c->probs[c->pod[d]].alpha0;
    for (int i = 0; i < n; ++i) {
      const double a = alpha[d * n + i];
      if (!(a >= 0.0 && a <= a0)) { set_error("mc_design_upload: alpha outside [0, alpha0] (P:221)"); return MC_ERR_INVALID; }
    }
  }
  if (std::memcmp(c->alpha.data(), alpha, sizeof(double) * (size_t)c->D * n) != 0) {
    std::memcpy(c->alpha.data(), alpha, sizeof(double) * (size_t)c->D * n);
    c->plan_built = false;   // TPS sites changed: the plan is rebuilt on the next mc_smooth
  }
  MC_CUDA(cudaSetDevice(c->device));
  if (c->D == 0) return MC_OK;
  MC_CUDA(cudaMemcpyAsync(c->d_alpha, alpha, sizeof(double) * (size_t)c->D * n, cudaMemcpyHostToDevice,
                          (cudaStream_t)stream));
  return launch_zc(c, (cudaStream_t)stream);
}

mc_status mc_set_sampling(mc_ctx* c, int32_t mode) {
  if (!c || (mode != 0 && mode != 1)) { set_error("mc_set_sampling: mode must be 0 (independent) or 1 (CRN)"); return MC_ERR_INVALID; }
  if (mode == 1 && c->n > 3) { set_error("mc_set_sampling: common random numbers are built for n <= 3"); return MC_ERR_INVALID; }
  c->sampling = mode;
  return MC_OK;
}

mc_status mc_set_launch(mc_ctx* c, int32_t threads, int32_t grid) {
  if (!c) { set_error("mc_set_launch: null ctx"); return MC_ERR_INVALID; }
  if (threads == 0) threads = 256;
  if (threads < 32 || threads > MAX_BLOCK || threads % 32 != 0 || grid < 0) {
    set_error("mc_set_launch: block_threads must be a multiple of 32 in [32, 256], grid_blocks >= 0");
    return MC_ERR_INVALID;
  }
  c->block_threads = threads;
  c->grid_blocks = grid;
  return MC_OK;
}

void mc_destroy(mc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaFree(c->d_plan_arena);
  cudaFree(c->d_tps_scratch);
  cudaFree(c->d_crn);
  cudaFree(c->d_prob);
  cudaFree(c->d_zc);
  cudaFree(c->d_alpha);
  cudaFree(c->d_ctheta);
  cudaFree(c->d_pod);
  cudaFree(c->d_prob_begin);
  delete c;
}

mc_status mc_evaluate_grid(mc_ctx* c, int64_t d0, int64_t dcount, uint64_t s0, uint64_t scount, void* stream,
                           int64_t* sums) {
  NvtxRange _nvtx("mc_evaluate_grid");
  if (!c || !sums) { set_error("mc_evaluate_grid: null ctx or sums"); return MC_ERR_INVALID; }
  if (d0 < 0 || dcount < 0 || d0 + dcount > c->D) { set_error("mc_evaluate_grid: design range outside [0, D)"); return MC_ERR_INVALID; }
  if (scount > 0 && s0 + scount < s0) { set_error("mc_evaluate_grid: sample range overflows"); return MC_ERR_INVALID; }
  // S1, S2 <= (samples accumulated) x 2^23 must stay below 2^63: the sample indices stay below 2^40
  // (exactly 2^40 samples of u = 1 would reach 2^63).  The bound covers one call; sums accumulated over
  // several calls into the same buffer must also total fewer than 2^40 samples per design (header).
  if ((s0 + scount) >= ((uint64_t)1 << 40)) { set_error("mc_evaluate_grid: sample indices must stay below 2^40 (int64 sums overflow at 2^40 x 2^23)"); return MC_ERR_INVALID; }
  MC_CUDA(cudaSetDevice(c->device));
  return launch_fused(c, d0, dcount, s0, s0 + scount, (cudaStream_t)stream, sums);
}

mc_status mc_finalize(mc_ctx* c, const int64_t* sums, uint64_t N, double* mean, double* var, void* stream) {
  NvtxRange _nvtx("mc_finalize");
  if (!c || !sums || !mean) { set_error("mc_finalize: null pointer"); return MC_ERR_INVALID; }
  if (N == 0) { set_error("mc_finalize: total_samples must be > 0"); return MC_ERR_INVALID; }
  MC_CUDA(cudaSetDevice(c->device));
  return launch_finalize(c, sums, N, mean, var, (cudaStream_t)stream);
}

mc_status mc_argmax(mc_ctx* c, const double* values, int64_t* idx, double* val, int64_t* best_idx_host,
                    double* best_val_host, void* stream) {
  NvtxRange _nvtx("mc_argmax");
  if (!c || !values || !idx || !val) { set_error("mc_argmax: null pointer"); return MC_ERR_INVALID; }
  MC_CUDA(cudaSetDevice(c->device));
  mc_status s = launch_argmax(c, values, idx, val, (cudaStream_t)stream);
  if (s != MC_OK || !best_idx_host) return s;
  std::vector<int64_t> hi(c->n_probs);
  std::vector<double> hv(c->n_probs);
  MC_CUDA(cudaMemcpyAsync(hi.data(), idx, hi.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  MC_CUDA(cudaMemcpyAsync(hv.data(), val, hv.size() * sizeof(double), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  MC_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  int64_t bi = -1;
  double bv = NAN;
  for (int k = 0; k < c->n_probs; ++k) {
    if (hi[k] < 0) continue;
    if (bi < 0 || hv[k] > bv || (hv[k] == bv && hi[k] < bi)) { bi = hi[k]; bv = hv[k]; }
  }
  *best_idx_host = bi;
  if (best_val_host) *best_val_host = bv;
  return MC_OK;
}

int64_t mc_num_designs(const mc_ctx* c) { return c ? c->D : -1; }
int32_t mc_num_problems(const mc_ctx* c) { return c ? c->n_probs : -1; }
int32_t mc_words_per_record(const mc_ctx* c) { return c ? words_per_record(c->n, c->est, c->model) : -1; }
int32_t mc_draw_dump_stride(const mc_ctx* c) { return c ? draw_dump_stride(c->n, c->est, c->model) : -1; }
int64_t mc_kernel_launches(const mc_ctx* c) { return c ? c->launches.load() : (int64_t)-1; }

mc_status mc_philox_dump(uint64_t seed, uint32_t tag, int32_t form, const uint32_t* id, const uint64_t* word,
                         int64_t count, uint32_t* out, void* stream) {
  if (count > 0 && (!id || !word || !out)) { set_error("mc_philox_dump: null pointer"); return MC_ERR_INVALID; }
  return launch_philox_dump(seed, tag, form, id, word, count, out, (cudaStream_t)stream);
}

mc_status mc_draw_dump(mc_ctx* c, const int64_t* design, const uint64_t* sample, int64_t count, float* out,
                       void* stream) {
  if (!c || (count > 0 && (!design || !sample || !out))) { set_error("mc_draw_dump: null pointer"); return MC_ERR_INVALID; }
  MC_CUDA(cudaSetDevice(c->device));
  return launch_draw_dump(c, design, sample, count, out, (cudaStream_t)stream);
}

mc_status mc_fwer(const mc_problem* p, const double* alpha, int64_t count, double* out, int32_t device) {
  if (!p || (count > 0 && (!alpha || !out))) { set_error("mc_fwer: null pointer"); return MC_ERR_INVALID; }
  mc_status s = validate_problem(*p, 0);
  if (s != MC_OK) return s;
  for (int64_t k = 0; k < count * p->n; ++k)
    if (!(alpha[k] >= 0.0 && alpha[k] < 1.0)) { set_error("mc_fwer: alpha must be in [0, 1)"); return MC_ERR_INVALID; }
  return fwer_eval(p, alpha, count, out, device);
}

mc_status mc_solve_alpha_n(const mc_problem* probs, int32_t n_probs, const int32_t* prob, int64_t count,
                           double* alpha, uint8_t* valid, int32_t device) {
  NvtxRange _nvtx("mc_solve_alpha_n");
  if (!probs || n_probs <= 0 || (count > 0 && (!prob || !alpha || !valid))) {
    set_error("mc_solve_alpha_n: null pointer or no problems");
    return MC_ERR_INVALID;
  }
  const int n = probs[0].n;
  for (int k = 0; k < n_probs; ++k) {
    mc_status s = validate_problem(probs[k], k);
    if (s != MC_OK) return s;
    if (probs[k].n != n) { set_error("mc_solve_alpha_n: all problems must share n"); return MC_ERR_INVALID; }
  }
  for (int64_t t = 0; t < count; ++t) {
    if (prob[t] < 0 || prob[t] >= n_probs) { set_error("mc_solve_alpha_n: problem index out of range"); return MC_ERR_INVALID; }
    for (int i = 0; i + 1 < n; ++i)
      if (!(alpha[t * n + i] >= 0.0 && alpha[t * n + i] <= probs[prob[t]].alpha0)) {
        set_error("mc_solve_alpha_n: alpha_1..alpha_{n-1} must lie in [0, alpha0]");
        return MC_ERR_INVALID;
      }
  }
  return alpha_points_solve(probs, n_probs, prob, count, device, alpha, valid);
}

mc_status mc_candidates(const mc_problem* probs, int32_t n_probs, int32_t m, int64_t n3, uint64_t seed,
                        double* alpha_out, int32_t* problem_out, int64_t cap, int64_t* n_out, int32_t device) {
  NvtxRange _nvtx("mc_candidates");
  if (!probs || n_probs <= 0 || !n_out || m < 1) { set_error("mc_candidates: null pointer, no problems or m < 1"); return MC_ERR_INVALID; }
  const int n = probs[0].n;
  for (int k = 0; k < n_probs; ++k) {
    mc_status s = validate_problem(probs[k], k);
    if (s != MC_OK) return s;
    if (probs[k].n != n) { set_error("mc_candidates: all problems must share n"); return MC_ERR_INVALID; }
  }
  std::vector<double> A;
  std::vector<uint8_t> ok;
  mc_status s = alpha_grid_solve(probs, n_probs, m, device, A, ok);
  if (s != MC_OK) return s;
  int64_t G = 1;
  for (int i = 0; i + 1 < n; ++i) G *= m;
  // per problem: valid list, then the seeded subset with key seed + problem index
  std::vector<std::vector<int64_t>> chosen(n_probs);
  int64_t total = 0;
  for (int k = 0; k < n_probs; ++k) {
    std::vector<int64_t> valid;
    for (int64_t g = 0; g < G; ++g)
      if (ok[k * G + g]) valid.push_back(g);
    const int64_t V = (int64_t)valid.size();
    if (n3 > 0 && V < n3) {
      char buf[160];
      snprintf(buf, sizeof buf, "mc_candidates: problem %d has %lld valid grid points < N3 = %lld (P:221)", k,
               (long long)V, (long long)n3);
      set_error(buf);
      return MC_ERR_INFEASIBLE;
    }
    if (n3 <= 0 || n3 >= V) {
      chosen[k] = valid;
    } else {
      std::vector<int64_t> idx(V);
      for (int64_t i = 0; i < V; ++i) idx[i] = i;
      const uint64_t sk = seed + (uint64_t)k;
      const uint32_t k0 = (uint32_t)sk ^ 0x00C0FFEEu, k1 = (uint32_t)(sk >> 32);
      for (int64_t i = 0; i < n3; ++i) {
        // Philox4x32-10 block (i/4, i>>34, 0, 0xC0FFEE) with key (k0, k1) on the host
        uint32_t c0 = (uint32_t)(i >> 2), c1 = (uint32_t)((uint64_t)i >> 34), c2 = 0u, c3 = 0x00C0FFEEu;
        uint32_t kk0 = k0, kk1 = k1;
        for (int r = 0; r < 10; ++r) {
          if (r) { kk0 += 0x9E3779B9u; kk1 += 0xBB67AE85u; }
          const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
          const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ kk0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ kk1;
          c1 = (uint32_t)p1;
          c3 = (uint32_t)p0;
          c0 = n0;
          c2 = n2;
        }
        const uint32_t o[4] = {c0, c1, c2, c3};
        const uint64_t word = o[i & 3];
        const int64_t j = i + (int64_t)((word * (uint64_t)(V - i)) >> 32);
        std::swap(idx[i], idx[j]);
      }
      std::vector<int64_t> sel(idx.begin(), idx.begin() + n3);
      std::sort(sel.begin(), sel.end());
      chosen[k].resize(n3);
      for (int64_t i = 0; i < n3; ++i) chosen[k][i] = valid[sel[i]];
    }
    total += (int64_t)chosen[k].size();
  }
  *n_out = total;
  if (total > cap || !alpha_out || !problem_out) {
    set_error("mc_candidates: output capacity too small (n_out = capacity needed)");
    return MC_ERR_INVALID;
  }
  int64_t o = 0;
  for (int k = 0; k < n_probs; ++k)
    for (int64_t g : chosen[k]) {
      for (int i = 0; i < n; ++i) alpha_out[o * n + i] = A[((size_t)k * G + g) * n + i];
      problem_out[o] = k;
      ++o;
    }
  return MC_OK;
}

mc_status mc_smooth_plan(mc_ctx* c, const uint8_t* mask, void* stream) {
  NvtxRange _nvtx("mc_smooth_plan");
  if (!c) { set_error("mc_smooth_plan: null ctx"); return MC_ERR_INVALID; }
  MC_CUDA(cudaSetDevice(c->device));
  return smooth_plan(c, mask, (cudaStream_t)stream);
}

mc_status mc_smooth(mc_ctx* c, const double* values, double lambda, double* out, double* lam_used, void* stream) {
  NvtxRange _nvtx("mc_smooth");
  if (!c || !values || !out) { set_error("mc_smooth: null pointer"); return MC_ERR_INVALID; }
  MC_CUDA(cudaSetDevice(c->device));
  if (!c->plan_built) {
    mc_status s = smooth_plan(c, nullptr, (cudaStream_t)stream);
    if (s != MC_OK) return s;
  }
  return smooth_apply(c, values, lambda, out, lam_used, (cudaStream_t)stream);
}

}  // extern "C"
