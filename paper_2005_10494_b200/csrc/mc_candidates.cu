// mc_candidates.cu — K4: FWER (Formula 2) and the alpha_n solve of the Sec. 2.3 candidate grid on
// the GPU in fp64, one thread per grid point (row a1 of DESIGN.md §1).
//
// Phi_Sigma0(z) for the Formula-1 correlation uses the Markov structure of A.1
// (X_{k+1} = rho_k X_k + s_k W): n = 2 and n = 3 reduce to ONE 1-D integral
//   n = 2: int_{-inf}^{z1} phi(x) Phi((z2 - rho1 x)/s1) dx
//   n = 3: int_{-inf}^{z2} phi(x) Phi((z1 - rho1 x)/s1) Phi((z3 - rho2 x)/s2) dx   (X1 _|_ X3 | X2)
// evaluated by composite 10-point Gauss-Legendre on [-9, min(z, 9)] with panels no wider than half
// the narrowest conditional sigmoid; n >= 4 uses the backward transfer recursion over the chain.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "mc_internal.h"

namespace mci {

__constant__ double c_glx[10];
__constant__ double c_glw[10];

static void gauss_legendre10(double* x, double* w) {
  const int G = 10;
  for (int i = 0; i < G; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (G + 0.5)), dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = t;
      for (int k = 2; k <= G; ++k) {
        const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = G * (t * p1 - p0) / (t * t - 1.0);
      const double dt = p1 / dp;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    x[i] = t;
    w[i] = 2.0 / ((1.0 - t * t) * dp * dp);
  }
}

static cudaError_t upload_gl() {
  double x[10], w[10];
  gauss_legendre10(x, w);
  cudaError_t e = cudaMemcpyToSymbol(c_glx, x, sizeof x);
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_glw, w, sizeof w);
}

__device__ __forceinline__ double Phi_d(double x) { return 0.5 * erfc(-x * 0.70710678118654752440); }
__device__ __forceinline__ double phi_d(double x) { return 0.39894228040143267794 * exp(-0.5 * x * x); }
// Phi((z - rho x)/s) with z = +inf -> 1
__device__ __forceinline__ double cond_cdf(double z, double rho, double s, double x) {
  return isinf(z) ? 1.0 : Phi_d((z - rho * x) / s);
}

constexpr double QLO = -9.0, QHI = 9.0;

struct Chain {
  int n;
  double rho[MC_MAX_N], sd[MC_MAX_N];
};

// 1-D integrand families for n = 2, 3
template <int NN>
__device__ double orthant_1d(const double* z, const Chain& ch) {
  const double up = fmin(NN == 2 ? z[0] : z[1], QHI);
  if (up <= QLO) return 0.0;
  double wmin = 1.0;
  wmin = fmin(wmin, ch.sd[0] / ch.rho[0]);
  if (NN == 3) wmin = fmin(wmin, ch.sd[1] / ch.rho[1]);
  const double h = 0.5 * wmin;
  int P = (int)ceil((up - QLO) / h);
  if (P > 4000) P = 4000;
  const double len = (up - QLO) / P;
  double acc = 0.0;
  for (int k = 0; k < P; ++k) {
    const double lo = QLO + k * len;
    double pacc = 0.0;
#pragma unroll
    for (int g = 0; g < 10; ++g) {
      const double x = lo + 0.5 * len * (c_glx[g] + 1.0);
      double f = phi_d(x);
      if (NN == 2) f *= cond_cdf(z[1], ch.rho[0], ch.sd[0], x);
      else f *= cond_cdf(z[0], ch.rho[0], ch.sd[0], x) * cond_cdf(z[2], ch.rho[1], ch.sd[1], x);
      pacc += c_glw[g] * f;
    }
    acc += 0.5 * len * pacc;
  }
  return acc;
}

// n >= 4: backward transfer h_k(x) = int p(y | x) h_{k+1}(y) dy over the chain, level nodes on
// [-9, min(z_k, 9)], with the last conditional in closed form.
constexpr int TQ = 320;   // nodes per level (32 panels x 10)
__device__ double orthant_chain(const double* z, const Chain& ch) {
  const int n = ch.n;
  double xs[2][TQ], ws[2][TQ], hv[2][TQ];
  int m[2];
  auto nodes = [&](int k, int slot) {
    const double up = fmin(z[k], QHI);
    if (up <= QLO) { m[slot] = 0; return; }
    const int P = TQ / 10;
    const double len = (up - QLO) / P;
    for (int p = 0; p < P; ++p)
      for (int g = 0; g < 10; ++g) {
        xs[slot][p * 10 + g] = QLO + p * len + 0.5 * len * (c_glx[g] + 1.0);
        ws[slot][p * 10 + g] = 0.5 * len * c_glw[g];
      }
    m[slot] = P * 10;
  };
  // level n-2 (0-based): h(x) = Phi((z_{n-1} - rho x)/s)
  int cur = 0;
  nodes(n - 2, cur);
  if (m[cur] == 0) return 0.0;
  for (int j = 0; j < m[cur]; ++j) hv[cur][j] = cond_cdf(z[n - 1], ch.rho[n - 2], ch.sd[n - 2], xs[cur][j]);
  for (int k = n - 3; k >= 0; --k) {
    const int nxt = cur ^ 1;
    nodes(k, nxt);
    if (m[nxt] == 0) return 0.0;
    const double is = 1.0 / ch.sd[k];
    for (int i = 0; i < m[nxt]; ++i) {
      double acc = 0.0;
      for (int j = 0; j < m[cur]; ++j)
        acc += ws[cur][j] * phi_d((xs[cur][j] - ch.rho[k] * xs[nxt][i]) * is) * is * hv[cur][j];
      hv[nxt][i] = acc;
    }
    cur = nxt;
  }
  double acc = 0.0;
  for (int j = 0; j < m[cur]; ++j) acc += ws[cur][j] * phi_d(xs[cur][j]) * hv[cur][j];
  return acc;
}

// CHAIN = false: n <= 3 only (no local-memory frame); CHAIN = true: n >= 4.
template <bool CHAIN>
__device__ double orthant(const double* z, const Chain& ch) {
  if constexpr (CHAIN) return orthant_chain(z, ch);
  switch (ch.n) {
    case 1: return Phi_d(z[0]);
    case 2: return orthant_1d<2>(z, ch);
    default: return orthant_1d<3>(z, ch);
  }
}

__device__ double z_of_alpha(double a) { return a <= 0.0 ? INFINITY : -normcdfinv(a); }

template <bool CHAIN>
__device__ double fwer_dev(const double* alpha, const Chain& ch) {
  double z[MC_MAX_N];
  for (int i = 0; i < ch.n; ++i) z[i] = z_of_alpha(alpha[i]);
  return 1.0 - orthant<CHAIN>(z, ch);
}

struct ProbChain {
  Chain ch;
  double alpha0;
};

template <bool CHAIN>
__global__ void k_fwer(ProbChain pc, const double* __restrict__ alpha, int64_t count, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  double a[MC_MAX_N];
  for (int k = 0; k < pc.ch.n; ++k) a[k] = alpha[i * pc.ch.n + k];
  out[i] = fwer_dev<CHAIN>(a, pc.ch);
}

// Feasibility and alpha_n for partial alpha a[0..n-2] by the Illinois method on
// f(x) = FWER(alpha_1..alpha_{n-1}, x) - alpha0, increasing in x.  Writes a[n-1].
template <bool CHAIN>
__device__ uint8_t solve_alpha_n_dev(const ProbChain& pc, double* a) {
  const int n = pc.ch.n;
  double an = pc.alpha0;
  uint8_t ok = 1;
  if (n > 1) {
    a[n - 1] = 0.0;
    double flo = fwer_dev<CHAIN>(a, pc.ch) - pc.alpha0;
    if (flo > 1e-12) {
      ok = 0;
      an = NAN;
    } else if (flo >= -1e-12) {
      an = 0.0;
    } else {
      double lo = 0.0, hi = pc.alpha0;
      a[n - 1] = hi;
      double fhi = fwer_dev<CHAIN>(a, pc.ch) - pc.alpha0;
      double x0 = lo, f0 = flo, x1 = hi, f1 = fhi;
      an = hi;
      for (int it = 0; it < 100; ++it) {
        double c = x1 - f1 * (x1 - x0) / (f1 - f0);
        if (!(c > fmin(x0, x1) && c < fmax(x0, x1))) c = 0.5 * (x0 + x1);
        a[n - 1] = c;
        const double fc = fwer_dev<CHAIN>(a, pc.ch) - pc.alpha0;
        an = c;
        if (fabs(fc) < 2e-16) break;   // FWER resolved to its quadrature accuracy
        if ((fc > 0.0) != (f1 > 0.0)) { x0 = x1; f0 = f1; }
        else f0 *= 0.5;
        x1 = c;
        f1 = fc;
        if (fabs(x1 - x0) < 1e-15) break;
      }
    }
  }
  a[n - 1] = an;
  return ok;
}

// One thread per (problem, grid point) of the half-offset m^(n-1) grid.
template <bool CHAIN>
__global__ void k_alpha_grid(const ProbChain* __restrict__ pcs, int32_t n_probs, int32_t m, int64_t G,
                             double* __restrict__ A, uint8_t* __restrict__ valid) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)n_probs * G) return;
  const int k = (int)(t / G);
  const int64_t g = t % G;
  const ProbChain pc = pcs[k];
  const int n = pc.ch.n;
  double a[MC_MAX_N];
  int64_t rem = g;
  for (int i = n - 2; i >= 0; --i) {
    a[i] = ((double)(rem % m) + 0.5) * pc.alpha0 / m;
    rem /= m;
  }
  const uint8_t ok = solve_alpha_n_dev<CHAIN>(pc, a);
  for (int i = 0; i < n; ++i) A[t * n + i] = a[i];
  valid[t] = ok;
}

// One thread per explicit partial point (problem index, alpha_1..alpha_{n-1}): alpha_n in place.
template <bool CHAIN>
__global__ void k_alpha_points(const ProbChain* __restrict__ pcs, const int32_t* __restrict__ prob, int64_t count,
                               double* __restrict__ A, uint8_t* __restrict__ valid) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  const ProbChain pc = pcs[prob[t]];
  const int n = pc.ch.n;
  double a[MC_MAX_N];
  for (int i = 0; i < n; ++i) a[i] = A[t * n + i];
  valid[t] = solve_alpha_n_dev<CHAIN>(pc, a);
  A[t * n + n - 1] = a[n - 1];
}

static ProbChain make_chain(const mc_problem& p) {
  ProbChain pc{};
  pc.ch.n = p.n;
  pc.alpha0 = p.alpha0;
  for (int i = 0; i + 1 < p.n; ++i) {
    pc.ch.rho[i] = std::sqrt(p.r[i + 1] / p.r[i]);
    pc.ch.sd[i] = std::sqrt(1.0 - p.r[i + 1] / p.r[i]);
  }
  return pc;
}

mc_status alpha_grid_solve(const mc_problem* probs, int32_t n_probs, int32_t m, int device, std::vector<double>& A,
                           std::vector<uint8_t>& valid) {
  MC_CUDA(cudaSetDevice(device));
  MC_CUDA(upload_gl());
  const int n = probs[0].n;
  int64_t G = 1;
  for (int i = 0; i + 1 < n; ++i) G *= m;
  const int64_t T = G * n_probs;
  std::vector<ProbChain> pcs(n_probs);
  for (int k = 0; k < n_probs; ++k) pcs[k] = make_chain(probs[k]);
  ProbChain* d_pcs = nullptr;
  double* d_A = nullptr;
  uint8_t* d_v = nullptr;
  mc_status s = MC_OK;
  cudaError_t e;
  if ((e = cudaMalloc(&d_pcs, sizeof(ProbChain) * n_probs)) != cudaSuccess ||
      (e = cudaMalloc(&d_A, sizeof(double) * T * n)) != cudaSuccess || (e = cudaMalloc(&d_v, T)) != cudaSuccess) {
    s = cuda_fail(e, "alpha_grid_solve alloc");
  } else if ((e = cudaMemcpy(d_pcs, pcs.data(), sizeof(ProbChain) * n_probs, cudaMemcpyHostToDevice)) != cudaSuccess) {
    s = cuda_fail(e, "alpha_grid_solve upload");
  } else {
    const int threads = n >= 4 ? 32 : 128;
    if (n >= 4) k_alpha_grid<true><<<(unsigned)((T + threads - 1) / threads), threads>>>(d_pcs, n_probs, m, G, d_A, d_v);
    else k_alpha_grid<false><<<(unsigned)((T + threads - 1) / threads), threads>>>(d_pcs, n_probs, m, G, d_A, d_v);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess) {
      s = cuda_fail(e, "k_alpha_grid");
    } else {
      A.resize((size_t)T * n);
      valid.resize((size_t)T);
      if ((e = cudaMemcpy(A.data(), d_A, sizeof(double) * T * n, cudaMemcpyDeviceToHost)) != cudaSuccess ||
          (e = cudaMemcpy(valid.data(), d_v, T, cudaMemcpyDeviceToHost)) != cudaSuccess)
        s = cuda_fail(e, "alpha_grid_solve download");
    }
  }
  cudaFree(d_pcs);
  cudaFree(d_A);
  cudaFree(d_v);
  return s;
}

mc_status alpha_points_solve(const mc_problem* probs, int32_t n_probs, const int32_t* prob, int64_t count, int device,
                             double* A, uint8_t* valid) {
  if (count <= 0) return MC_OK;
  MC_CUDA(cudaSetDevice(device));
  MC_CUDA(upload_gl());
  const int n = probs[0].n;
  std::vector<ProbChain> pcs(n_probs);
  for (int k = 0; k < n_probs; ++k) pcs[k] = make_chain(probs[k]);
  ProbChain* d_pcs = nullptr;
  int32_t* d_prob = nullptr;
  double* d_A = nullptr;
  uint8_t* d_v = nullptr;
  mc_status s = MC_OK;
  cudaError_t e;
  if ((e = cudaMalloc(&d_pcs, sizeof(ProbChain) * n_probs)) != cudaSuccess ||
      (e = cudaMalloc(&d_prob, sizeof(int32_t) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_A, sizeof(double) * count * n)) != cudaSuccess ||
      (e = cudaMalloc(&d_v, count)) != cudaSuccess) {
    s = cuda_fail(e, "alpha_points_solve alloc");
  } else if ((e = cudaMemcpy(d_pcs, pcs.data(), sizeof(ProbChain) * n_probs, cudaMemcpyHostToDevice)) != cudaSuccess ||
             (e = cudaMemcpy(d_prob, prob, sizeof(int32_t) * count, cudaMemcpyHostToDevice)) != cudaSuccess ||
             (e = cudaMemcpy(d_A, A, sizeof(double) * count * n, cudaMemcpyHostToDevice)) != cudaSuccess) {
    s = cuda_fail(e, "alpha_points_solve upload");
  } else {
    const int threads = n >= 4 ? 32 : 128;
    const unsigned blocks = (unsigned)((count + threads - 1) / threads);
    if (n >= 4) k_alpha_points<true><<<blocks, threads>>>(d_pcs, d_prob, count, d_A, d_v);
    else k_alpha_points<false><<<blocks, threads>>>(d_pcs, d_prob, count, d_A, d_v);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess ||
        (e = cudaMemcpy(A, d_A, sizeof(double) * count * n, cudaMemcpyDeviceToHost)) != cudaSuccess ||
        (e = cudaMemcpy(valid, d_v, count, cudaMemcpyDeviceToHost)) != cudaSuccess)
      s = cuda_fail(e, "k_alpha_points");
  }
  cudaFree(d_pcs);
  cudaFree(d_prob);
  cudaFree(d_A);
  cudaFree(d_v);
  return s;
}

mc_status fwer_eval(const mc_problem* p, const double* alpha, int64_t count, double* out, int device) {
  if (count <= 0) return MC_OK;
  MC_CUDA(cudaSetDevice(device));
  MC_CUDA(upload_gl());
  ProbChain pc = make_chain(*p);
  double *d_a = nullptr, *d_o = nullptr;
  mc_status s = MC_OK;
  cudaError_t e;
  if ((e = cudaMalloc(&d_a, sizeof(double) * count * p->n)) != cudaSuccess ||
      (e = cudaMalloc(&d_o, sizeof(double) * count)) != cudaSuccess) {
    s = cuda_fail(e, "mc_fwer alloc");
  } else if ((e = cudaMemcpy(d_a, alpha, sizeof(double) * count * p->n, cudaMemcpyHostToDevice)) != cudaSuccess) {
    s = cuda_fail(e, "mc_fwer upload");
  } else {
    const int threads = p->n >= 4 ? 32 : 128;
    if (p->n >= 4) k_fwer<true><<<(unsigned)((count + threads - 1) / threads), threads>>>(pc, d_a, count, d_o);
    else k_fwer<false><<<(unsigned)((count + threads - 1) / threads), threads>>>(pc, d_a, count, d_o);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess ||
        (e = cudaMemcpy(out, d_o, sizeof(double) * count, cudaMemcpyDeviceToHost)) != cudaSuccess)
      s = cuda_fail(e, "k_fwer");
  }
  cudaFree(d_a);
  cudaFree(d_o);
  return s;
}

}  // namespace mci
