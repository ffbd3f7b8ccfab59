// mc_candidates.cu — K4: FWER (Formula 2) and the alpha_n solve of the Sec. 2.3 candidate grid on
// the GPU in fp64 (row a1 of DESIGN.md §1).
//
// Phi_Sigma0(z) for the Formula-1 correlation uses the Markov structure of A.1
// (X_{k+1} = rho_k X_k + s_k W): n = 2 and n = 3 reduce to ONE 1-D integral
//   n = 2: int_{-inf}^{z1} phi(x) Phi((z2 - rho1 x)/s1) dx
//   n = 3: int_{-inf}^{z2} phi(x) Phi((z1 - rho1 x)/s1) Phi((z3 - rho2 x)/s2) dx   (X1 _|_ X3 | X2)
// evaluated by composite 10-point Gauss-Legendre on [-9, min(z, 9)] with panels no wider than half
// the narrowest conditional sigmoid, one warp per point (node factors that do not depend on alpha_n are
// computed once per point; k_fwer keeps one thread per point).  n >= 4 runs the chain's forward filtering
// recursion with one CTA per point (k_chain): the densities of X_1..X_{n-1} restricted to their
// orthant are built once per point, so each step of the alpha_n solve is one 1-D sum.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
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
  if (P > 40000) P = 40000;   // never reached in the validated range (s >= 1e-3 needs <= 36000 panels)
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

// n >= 4: the chain's FORWARD filtering recursion, one CTA per point.  The restricted densities
//   f_1(x) = phi(x) 1[x <= z_1],
//   f_k(y) = 1[y <= z_k] int f_{k-1}(x) phi((y - rho_{k-1} x)/s_{k-1}) / s_{k-1} dx   (k = 2 .. n-1)
// depend only on z_1 .. z_{n-1}, and Phi_Sigma0(z) = int f_{n-1}(x) Phi((z_n - rho_{n-1} x)/s_{n-1}) dx,
// so each step of the alpha_n solve re-evaluates only that last 1-D sum.  Level k's nodes: composite
// 10-point Gauss-Legendre on [-9, min(z_k, 9)] with panels no wider than h = 0.5 min_k s_k (the n <= 3
// rule); the transfer sums only the panels within 9 s_{k-1}/rho_{k-1} of y/rho_{k-1} (phi(9) ~ 1e-18).
constexpr int CHAIN_THREADS = 128;
constexpr int CHAIN_CAP = 12288;   // nodes per level; two levels live in shared memory (192 KB)

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();                                   // red[] of the previous sum has been read
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];   // same order in every thread
  return s;
}

struct ChainLevel {
  double lo, len;
  int P;   // panels (10 P nodes); 0: the orthant is empty
};

__device__ __forceinline__ ChainLevel chain_level(double z, double h) {
  ChainLevel L;
  L.lo = QLO;
  const double up = fmin(z, QHI);
  L.P = up <= QLO ? 0 : (int)ceil((up - QLO) / h);
  L.len = L.P > 0 ? (up - QLO) / L.P : 0.0;
  return L;
}
__device__ __forceinline__ double chain_x(const ChainLevel& L, int i) {
  return L.lo + L.len * ((double)(i / 10) + 0.5 * (c_glx[i % 10] + 1.0));
}
__device__ __forceinline__ double chain_w(const ChainLevel& L, int i) { return 0.5 * L.len * c_glw[i % 10]; }

// Forward pass for z[0..n-2]: leaves w_i f_{n-1}(x_i) of the last restricted level in *fout (shared
// memory) and returns that level's geometry (P = 0 when some level is empty: Phi_Sigma0 = 0).
__device__ ChainLevel chain_forward(const double* z, const Chain& ch, double h, double* fa, double* fb,
                                    const double*& fout) {
  ChainLevel prev = chain_level(z[0], h);
  double* cur = fa;
  for (int i = threadIdx.x; i < 10 * prev.P; i += blockDim.x) cur[i] = phi_d(chain_x(prev, i)) * chain_w(prev, i);
  for (int k = 1; k <= ch.n - 2 && prev.P > 0; ++k) {
    const ChainLevel L = chain_level(z[k], h);
    double* nxt = cur == fa ? fb : fa;
    __syncthreads();
    const double rho = ch.rho[k - 1], is = 1.0 / ch.sd[k - 1], reach = 9.0 * ch.sd[k - 1] / rho;
    for (int i = threadIdx.x; i < 10 * L.P; i += blockDim.x) {
      const double y = chain_x(L, i), xc = y / rho;
      const int p0 = max(0, (int)floor((xc - reach - prev.lo) / prev.len));
      const int p1 = min(prev.P - 1, (int)floor((xc + reach - prev.lo) / prev.len));
      double acc = 0.0;
      for (int j = 10 * p0; j < 10 * (p1 + 1); ++j) acc += cur[j] * phi_d((y - rho * chain_x(prev, j)) * is);
      nxt[i] = acc * is * chain_w(L, i);
    }
    cur = nxt;
    prev = L;
  }
  __syncthreads();
  fout = cur;
  return prev;
}

// Phi_Sigma0 with last threshold zl from the forward densities (block-wide; the same value in every thread)
__device__ double chain_last(const double* f, const ChainLevel& L, const Chain& ch, double zl, double* red) {
  double acc = 0.0;
  const double rho = ch.rho[ch.n - 2], sd = ch.sd[ch.n - 2];
  for (int i = threadIdx.x; i < 10 * L.P; i += blockDim.x) acc += f[i] * cond_cdf(zl, rho, sd, chain_x(L, i));
  return block_sum(acc, red);
}

// n <= 3: closed-form 1-D integrals, one thread per point.
__device__ double orthant(const double* z, const Chain& ch) {
  switch (ch.n) {
    case 1: return Phi_d(z[0]);
    case 2: return orthant_1d<2>(z, ch);
    default: return orthant_1d<3>(z, ch);
  }
}

__device__ double z_of_alpha(double a) { return a <= 0.0 ? INFINITY : -normcdfinv(a); }

__device__ double fwer_dev(const double* alpha, const Chain& ch) {
  double z[MC_MAX_N];
  for (int i = 0; i < ch.n; ++i) z[i] = z_of_alpha(alpha[i]);
  return 1.0 - orthant(z, ch);
}

struct ProbChain {
  Chain ch;
  double alpha0;
  double h;   // n >= 4: panel width 0.5 min_k s_k
};

__global__ void k_fwer(ProbChain pc, const double* __restrict__ alpha, int64_t count, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  double a[MC_MAX_N];
  for (int k = 0; k < pc.ch.n; ++k) a[k] = alpha[i * pc.ch.n + k];
  out[i] = fwer_dev(a, pc.ch);
}

// Feasibility and alpha_n for partial alpha a[0..n-2] by the Illinois method on
// f(x) = FWER(alpha_1..alpha_{n-1}, x) - alpha0, increasing in x.  Writes a[n-1].
// FW(x) returns FWER(alpha_1..alpha_{n-1}, x); with a block-wide FW every thread runs the same
// iteration on the same values, so control flow stays uniform.
template <class FW>
__device__ uint8_t illinois_alpha_n(int n, double alpha0, double* a, FW fw) {
  double an = alpha0;
  uint8_t ok = 1;
  if (n > 1) {
    const double flo = fw(0.0) - alpha0;
    if (flo > 1e-12) {
      ok = 0;
      an = NAN;
    } else if (flo >= -1e-12) {
      an = 0.0;
    } else {
      double x0 = 0.0, f0 = flo, x1 = alpha0, f1 = fw(alpha0) - alpha0;
      an = x1;
      for (int it = 0; it < 100; ++it) {
        double c = x1 - f1 * (x1 - x0) / (f1 - f0);
        if (!(c > fmin(x0, x1) && c < fmax(x0, x1))) c = 0.5 * (x0 + x1);
        const double fc = fw(c) - alpha0;
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

// n <= 3, one WARP per point (the candidate grid and explicit points).  The orthant is the 1-D integral
// over x = X_1 (n = 2) or X_2 (n = 3) of orthant_1d with the same panels and nodes; during the alpha_n solve
// only the last factor Phi((z_n - rho x)/s) changes, so the rest of each node's integrand,
// g_i = w_i phi(x_i) [Phi((z_1 - rho_1 x_i)/s_1) for n = 3], is computed once into shared memory (up to
// W1_CAP nodes; recomputed beyond) and every Illinois step costs one Phi per node, spread over the lanes.
// The lane sums are combined by a xor butterfly, which leaves the same value in every lane (IEEE addition
// commutes), so all lanes run the identical iteration.
constexpr int W1_WARPS = 4, W1_CAP = 1024;
template <int MODE>   // 0: grid point t of the m^(n-1) grid; 1: explicit partial point t (problem prob[t])
__global__ void __launch_bounds__(32 * W1_WARPS) k_alpha_warp(const ProbChain* __restrict__ pcs,
                                                               const int32_t* __restrict__ prob, int32_t m, int64_t G,
                                                               int64_t T, double* __restrict__ A,
                                                               uint8_t* __restrict__ valid) {
  __shared__ double sg[W1_WARPS][W1_CAP];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t t = blockIdx.x * (int64_t)W1_WARPS + wid;
  if (t >= T) return;                                   // uniform per warp
  const ProbChain pc = pcs[MODE == 0 ? (int)(t / G) : prob[t]];
  const int n = pc.ch.n;
  double a[MC_MAX_N];
  if (MODE == 0) {
    int64_t rem = t % G;
    for (int i = n - 2; i >= 0; --i) {
      a[i] = ((double)(rem % m) + 0.5) * pc.alpha0 / m;
      rem /= m;
    }
  } else {
    for (int i = 0; i < n; ++i) a[i] = A[t * n + i];
  }
  uint8_t ok = 1;
  if (n >= 2) {
    const double z0 = z_of_alpha(a[0]), z1 = n == 3 ? z_of_alpha(a[1]) : 0.0;
    const double up = fmin(n == 2 ? z0 : z1, QHI);
    double wmin = fmin(1.0, pc.ch.sd[0] / pc.ch.rho[0]);
    if (n == 3) wmin = fmin(wmin, pc.ch.sd[1] / pc.ch.rho[1]);
    int P = up <= QLO ? 0 : (int)ceil((up - QLO) / (0.5 * wmin));
    if (P > 40000) P = 40000;   // never reached in the validated range (s >= 1e-3 needs <= 36000 panels)
    const double len = P > 0 ? (up - QLO) / P : 0.0;
    const int nodes = 10 * P;
    const bool stored = nodes <= W1_CAP;
    const double rl = pc.ch.rho[n - 2], sl = pc.ch.sd[n - 2];
    auto xnode = [&](int i) { return QLO + len * ((double)(i / 10) + 0.5 * (c_glx[i % 10] + 1.0)); };
    auto gnode = [&](int i) {
      const double x = xnode(i);
      double g = 0.5 * len * c_glw[i % 10] * phi_d(x);
      if (n == 3) g *= cond_cdf(z0, pc.ch.rho[0], pc.ch.sd[0], x);
      return g;
    };
    if (stored)
      for (int i = lane; i < nodes; i += 32) sg[wid][i] = gnode(i);
    __syncwarp();
    ok = illinois_alpha_n(n, pc.alpha0, a, [&](double an) {
      const double zl = z_of_alpha(an);
      double acc = 0.0;
      for (int i = lane; i < nodes; i += 32) acc += (stored ? sg[wid][i] : gnode(i)) * cond_cdf(zl, rl, sl, xnode(i));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      return 1.0 - acc;
    });
  } else {
    a[0] = pc.alpha0;
  }
  if (lane == 0) {
    if (MODE == 0)
      for (int i = 0; i < n; ++i) A[t * n + i] = a[i];
    else
      A[t * n + n - 1] = a[n - 1];
    valid[t] = ok;
  }
}

// n >= 4, one CTA per point, grid-strided.  MODE 0: grid point t of the m^(n-1) grid (alpha_n solved);
// 1: explicit partial point t (problem prob[t]; alpha_n solved in place); 2: FWER of the full alpha row t.
template <int MODE>
__global__ void __launch_bounds__(CHAIN_THREADS) k_chain(const ProbChain* __restrict__ pcs, const int32_t* __restrict__ prob,
                                                         int32_t m, int64_t G, int64_t T, double* __restrict__ A,
                                                         uint8_t* __restrict__ valid, double* __restrict__ out) {
  extern __shared__ double sm[];
  __shared__ double red[CHAIN_THREADS / 32];
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const int k = MODE == 0 ? (int)(t / G) : (MODE == 1 ? prob[t] : 0);
    const ProbChain pc = pcs[k];
    const int n = pc.ch.n;
    double a[MC_MAX_N];
    if (MODE == 0) {
      int64_t rem = t % G;
      for (int i = n - 2; i >= 0; --i) {
        a[i] = ((double)(rem % m) + 0.5) * pc.alpha0 / m;
        rem /= m;
      }
    } else {
      for (int i = 0; i < n; ++i) a[i] = A[t * n + i];
    }
    double z[MC_MAX_N];
    for (int i = 0; i + 1 < n; ++i) z[i] = z_of_alpha(a[i]);
    const double* f = nullptr;
    const ChainLevel L = chain_forward(z, pc.ch, pc.h, sm, sm + CHAIN_CAP, f);
    auto fw = [&](double x) { return 1.0 - chain_last(f, L, pc.ch, z_of_alpha(x), red); };
    if (MODE == 2) {
      const double v = fw(a[n - 1]);
      if (threadIdx.x == 0) out[t] = v;
    } else {
      const uint8_t ok = illinois_alpha_n(n, pc.alpha0, a, fw);
      if (threadIdx.x == 0) {
        if (MODE == 0)
          for (int i = 0; i < n; ++i) A[t * n + i] = a[i];
        else
          A[t * n + n - 1] = a[n - 1];
        valid[t] = ok;
      }
    }
    __syncthreads();   // the next point reuses the shared levels
  }
}

static mc_status make_chain(const mc_problem& p, ProbChain& pc) {
  pc = ProbChain{};
  pc.ch.n = p.n;
  pc.alpha0 = p.alpha0;
  double smin = 1.0;
  for (int i = 0; i + 1 < p.n; ++i) {
    pc.ch.rho[i] = std::sqrt(p.r[i + 1] / p.r[i]);
    pc.ch.sd[i] = std::sqrt(1.0 - p.r[i + 1] / p.r[i]);
    smin = std::fmin(smin, pc.ch.sd[i]);
  }
  pc.h = 0.5 * smin;
  if (p.n >= 4 && 10.0 * std::ceil((QHI - QLO) / pc.h) > CHAIN_CAP) {
    char buf[200];
    snprintf(buf, sizeof buf, "n >= 4 FWER quadrature: min conditional sd %.3g needs %.0f nodes per level > %d "
             "(adjacent r ratio too close to 1 for the chain quadrature)", smin, 10.0 * std::ceil((QHI - QLO) / pc.h),
             CHAIN_CAP);
    set_error(buf);
    return MC_ERR_NUMERIC;
  }
  return MC_OK;
}

// Launch of k_chain<MODE> over T points (n >= 4): dynamic shared memory for two levels of CHAIN_CAP nodes.
template <int MODE>
static cudaError_t launch_chain(const ProbChain* d_pcs, const int32_t* d_prob, int32_t m, int64_t G, int64_t T,
                                double* d_A, uint8_t* d_v, double* d_out) {
  const size_t smem = sizeof(double) * 2 * CHAIN_CAP;
  cudaError_t e = cudaFuncSetAttribute(k_chain<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(T, (int64_t)sms * 64);
  if (grid <= 0) return cudaSuccess;
  k_chain<MODE><<<(unsigned)grid, CHAIN_THREADS, smem>>>(d_pcs, d_prob, m, G, T, d_A, d_v, d_out);
  return cudaGetLastError();
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
  for (int k = 0; k < n_probs; ++k) {
    mc_status s = make_chain(probs[k], pcs[k]);
    if (s != MC_OK) return s;
  }
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
    if (n >= 4) e = launch_chain<0>(d_pcs, nullptr, m, G, T, d_A, d_v, nullptr);
    else {
      k_alpha_warp<0><<<(unsigned)((T + W1_WARPS - 1) / W1_WARPS), 32 * W1_WARPS>>>(d_pcs, nullptr, m, G, T, d_A, d_v);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess) {
      s = cuda_fail(e, "k_alpha_warp / k_chain");
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
  for (int k = 0; k < n_probs; ++k) {
    mc_status s = make_chain(probs[k], pcs[k]);
    if (s != MC_OK) return s;
  }
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
    if (n >= 4) e = launch_chain<1>(d_pcs, d_prob, 0, 1, count, d_A, d_v, nullptr);
    else {
      k_alpha_warp<1><<<(unsigned)((count + W1_WARPS - 1) / W1_WARPS), 32 * W1_WARPS>>>(d_pcs, d_prob, 0, 1, count,
                                                                                    d_A, d_v);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess ||
        (e = cudaMemcpy(A, d_A, sizeof(double) * count * n, cudaMemcpyDeviceToHost)) != cudaSuccess ||
        (e = cudaMemcpy(valid, d_v, count, cudaMemcpyDeviceToHost)) != cudaSuccess)
      s = cuda_fail(e, "k_alpha_warp / k_chain");
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
  ProbChain pc;
  mc_status s = make_chain(*p, pc);
  if (s != MC_OK) return s;
  ProbChain* d_pcs = nullptr;
  double *d_a = nullptr, *d_o = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&d_a, sizeof(double) * count * p->n)) != cudaSuccess ||
      (e = cudaMalloc(&d_o, sizeof(double) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_pcs, sizeof(ProbChain))) != cudaSuccess) {
    s = cuda_fail(e, "mc_fwer alloc");
  } else if ((e = cudaMemcpy(d_a, alpha, sizeof(double) * count * p->n, cudaMemcpyHostToDevice)) != cudaSuccess ||
             (e = cudaMemcpy(d_pcs, &pc, sizeof(ProbChain), cudaMemcpyHostToDevice)) != cudaSuccess) {
    s = cuda_fail(e, "mc_fwer upload");
  } else {
    if (p->n >= 4) e = launch_chain<2>(d_pcs, nullptr, 0, 1, count, d_a, nullptr, d_o);
    else {
      k_fwer<<<(unsigned)((count + 127) / 128), 128>>>(pc, d_a, count, d_o);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess ||
        (e = cudaMemcpy(out, d_o, sizeof(double) * count, cudaMemcpyDeviceToHost)) != cudaSuccess)
      s = cuda_fail(e, "k_fwer / k_chain");
  }
  cudaFree(d_a);
  cudaFree(d_o);
  cudaFree(d_pcs);
  return s;
}

}  // namespace mci
