// mc_smooth.cu — K5: thin-plate-spline smoothing of the noisy power surface with GCV
// (Sec. 2.3; row a9 of DESIGN.md §1; contract DESIGN.md §2.9).
//
// Plan (once per design set, per problem with N fitted sites x = alpha_{1..d}/alpha0, d = n-1):
//   K_ij = phi(|x_i - x_j|) (fp64 kernel), T = [1 x] = Q R (host Householder, k = d+1 reflectors),
//   B = (Q^T K Q)[k:, k:] = V Lambda V^T (cuSOLVER Dsyevd), E = Q[:, k:] V  (N x (N-k), kept in HBM).
// Apply (every evaluation): c = E^T y; GCV(lambda) = N sum_j (t_j c_j)^2 / (sum_j t_j)^2 with
//   t_j = N lambda / (Lambda_j + N lambda) over the fixed log grid; y~ = y - E (t .* c).
// This is the penalised TPS [K + N lambda I, T; T^T, 0][w; beta] = [y; 0] (y~ = y - N lambda w)
// written in the eigenbasis, so one plan serves every lambda and every evaluation.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <vector>
#include <thread>
#include <string>

#include "mc_internal.h"

namespace mci {

constexpr int GCV_K = 49;   // lambda = 10^(-12 + 0.25 k), k = 0..48 (reading R16)

__device__ __forceinline__ double tps_phi(double r, int d) {
  if (d == 1) return r * r * r;
  if (d == 2) return r > 0.0 ? r * r * log(r) : 0.0;
  return -r;   // d = 3
}

__global__ void k_tps_kernel_matrix(const double* __restrict__ X, int64_t N, int d, double* __restrict__ K) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // row
  const int64_t j = blockIdx.y;                                        // column
  if (i >= N) return;
  double r2 = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = X[i * d + k] - X[j * d + k];
    r2 += t * t;
  }
  K[i + j * N] = tps_phi(sqrt(r2), d);
}

// w_j = sum_i v_i A_ij (column dots), one block per column
__global__ void k_col_dot(const double* __restrict__ A, int64_t N, int64_t ncols, int64_t lda,
                          const double* __restrict__ v, double* __restrict__ w) {
  __shared__ double sh[32];
  const int64_t j = blockIdx.x;
  if (j >= ncols) return;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) acc += v[i] * A[i + j * lda];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
    w[j] = t;
  }
}

// A <- A - tau v w^T  (left Householder application: (I - tau v v^T) A with w = A^T v)
__global__ void k_rank1_left(double* __restrict__ A, int64_t N, int64_t ncols, int64_t lda, const double* __restrict__ v,
                             const double* __restrict__ w, double tau) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  if (i < N && j < ncols) A[i + j * lda] -= tau * v[i] * w[j];
}

// Two-sided symmetric update A <- H A H, H = I - tau v v^T (LAPACK sytrd form):
// p = tau A v (from k_col_dot, A symmetric), w = p - (tau/2)(p^T v) v, A <- A - v w^T - w v^T.
__global__ void k_sym_w(const double* __restrict__ Av, const double* __restrict__ v, int64_t N, double tau,
                        double* __restrict__ w) {
  __shared__ double sh[32];
  __shared__ double s_alpha;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) acc += tau * Av[i] * v[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
    s_alpha = 0.5 * tau * t;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) w[i] = tau * Av[i] - s_alpha * v[i];
}

__global__ void k_rank2(double* __restrict__ A, int64_t N, const double* __restrict__ v, const double* __restrict__ w) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  if (i < N) A[i + j * N] -= v[i] * w[j] + w[i] * v[j];
}

__global__ void k_embed(const double* __restrict__ V, int64_t ldv, int64_t N, int k, double* __restrict__ Z) {
  // Z (N x (N-k)) = [0_{k x (N-k)}; V], V = (N-k) x (N-k) with leading dimension ldv
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  if (i >= N) return;
  Z[i + j * N] = i < k ? 0.0 : V[(i - k) + j * ldv];
}

// P (m x m, lda m) = K[k:, k:] (K: N x N, lda N), for the batched eigensolver
__global__ void k_pack(const double* __restrict__ K, int64_t N, int k, double* __restrict__ P) {
  const int64_t m = N - k;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  if (i < m) P[i + j * m] = K[(i + k) + (j + k) * N];
}

// ---- apply-side kernels, batched over problems (blockIdx.y or blockIdx.x = problem) ----------
struct PlanDev {
  const double* E;
  const double* lam;
  const int64_t* fit_idx;
  int64_t N;      // fitted sites
  int64_t k;      // N - (d+1) eigen-columns
  int64_t off;    // offset into the c / y scratch
  int32_t prob;   // problem index
  int32_t d;      // TPS dimension
  double alpha0;  // coordinate scale x = alpha / alpha0
};

__global__ void k_gather(const PlanDev* __restrict__ pl, const double* __restrict__ values, double* __restrict__ y) {
  const PlanDev p = pl[blockIdx.y];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.N; i += (int64_t)gridDim.x * blockDim.x)
    y[p.off + i] = values[p.fit_idx[i]];
}

// c_j = sum_i E_ij y_i  (column j contiguous), one warp per column
__global__ void k_et_y(const PlanDev* __restrict__ pl, const double* __restrict__ y, double* __restrict__ c) {
  const PlanDev p = pl[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= p.k) return;
  const double* col = p.E + j * p.N;
  const double* yy = y + p.off;
  double acc = 0.0;
  for (int64_t i = lane; i < p.N; i += 32) acc += col[i] * yy[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) c[p.off + j] = acc;
}

// GCV over the log grid (or the fixed lambda), then c_j <- t_j c_j (mode 0: smoothing,
// t_j = N lambda / (Lambda_j + N lambda)) or c_j <- c_j / (Lambda_j + N lambda) (mode 1: the TPS kernel
// weights w = E (c ./ (Lambda + N lambda))).  One block per problem; lambda written to lam_used[prob].
__global__ void k_gcv(const PlanDev* __restrict__ pl, double lambda_fixed, double* __restrict__ c,
                      double* __restrict__ lam_used, int mode) {
  __shared__ double s_rss[32], s_tr[32];
  __shared__ double s_best;
  const PlanDev p = pl[blockIdx.x];
  const double Nd = (double)p.N;
  double lam = lambda_fixed;
  if (lambda_fixed < 0.0) {
    double best = INFINITY, bestlam = 0.0;
    for (int g = 0; g < GCV_K; ++g) {
      const double l = pow(10.0, -12.0 + 0.25 * g);
      const double nl = Nd * l;
      double rss = 0.0, tr = 0.0;
      for (int64_t j = threadIdx.x; j < p.k; j += blockDim.x) {
        const double t = nl / (p.lam[j] + nl);
        const double tc = t * c[p.off + j];
        rss += tc * tc;
        tr += t;
      }
      for (int o = 16; o > 0; o >>= 1) {
        rss += __shfl_xor_sync(0xffffffffu, rss, o);
        tr += __shfl_xor_sync(0xffffffffu, tr, o);
      }
      if ((threadIdx.x & 31) == 0) { s_rss[threadIdx.x >> 5] = rss; s_tr[threadIdx.x >> 5] = tr; }
      __syncthreads();
      if (threadIdx.x == 0) {
        double R = 0.0, T = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { R += s_rss[k]; T += s_tr[k]; }
        const double v = Nd * R / (T * T);
        if (v < best) { best = v; bestlam = l; }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) s_best = bestlam;
    __syncthreads();
    lam = s_best;
  }
  if (threadIdx.x == 0 && lam_used) lam_used[p.prob] = lam;
  const double nl = Nd * lam;
  for (int64_t j = threadIdx.x; j < p.k; j += blockDim.x)
    c[p.off + j] *= (mode == 0 ? nl : 1.0) / (p.lam[j] + nl);
}

// w_i = sum_j E_ij g_j  (thread per row)
__global__ void k_e_w(const PlanDev* __restrict__ pl, const double* __restrict__ g, double* __restrict__ w) {
  const PlanDev p = pl[blockIdx.y];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= p.N) return;
  const double* gg = g + p.off;
  double acc = 0.0;
  for (int64_t j = 0; j < p.k; ++j) acc += p.E[i + j * p.N] * gg[j];
  w[p.off + i] = acc;
}

// (K w)_i = sum_j phi(|x_i - x_j|) w_j with x = alpha_{1..d} / alpha0 (thread per row)
__global__ void k_tps_kw(const PlanDev* __restrict__ pl, const double* __restrict__ alpha, int n,
                         const double* __restrict__ w, double* __restrict__ kw) {
  const PlanDev p = pl[blockIdx.y];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= p.N) return;
  const double* xi = alpha + p.fit_idx[i] * n;
  double acc = 0.0;
  for (int64_t j = 0; j < p.N; ++j) {
    const double* xj = alpha + p.fit_idx[j] * n;
    double r2 = 0.0;
    for (int k = 0; k < p.d; ++k) {
      const double t = (xi[k] - xj[k]) / p.alpha0;
      r2 += t * t;
    }
    acc += tps_phi(sqrt(r2), p.d) * w[p.off + j];
  }
  kw[p.off + i] = acc;
}

// out[fit_idx[i]] = y_i - sum_j E_ij c_j   (thread per row; the j-loop reads E coalesced)
__global__ void k_e_c(const PlanDev* __restrict__ pl, const double* __restrict__ y, const double* __restrict__ c,
                      double* __restrict__ out) {
  const PlanDev p = pl[blockIdx.y];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= p.N) return;
  const double* cc = c + p.off;
  double acc = 0.0;
  for (int64_t j = 0; j < p.k; ++j) acc += p.E[i + j * p.N] * cc[j];
  out[p.fit_idx[i]] = y[p.off + i] - acc;
}

// ---------------------------------------------------------------------------------------------
// Householder QR of T = [1 x] (N x k, fp64, host): returns reflectors v_r (v_r[r] = 1) and tau_r.
static void householder_T(const std::vector<double>& X, int64_t N, int d, std::vector<double>& V,
                          std::vector<double>& tau) {
  const int k = d + 1;
  std::vector<double> T((size_t)N * k);
  for (int64_t i = 0; i < N; ++i) {
    T[i] = 1.0;
    for (int c = 0; c < d; ++c) T[i + (c + 1) * N] = X[i * d + c];
  }
  V.assign((size_t)N * k, 0.0);
  tau.assign(k, 0.0);
  for (int r = 0; r < k; ++r) {
    double nrm = 0.0;
    for (int64_t i = r; i < N; ++i) nrm += T[i + r * N] * T[i + r * N];
    nrm = std::sqrt(nrm);
    const double a = T[r + r * N];
    const double alpha = a >= 0 ? -nrm : nrm;
    const double v0 = a - alpha;
    // v = (T[r:, r] - alpha e_r) / v0 so that v[r] = 1
    for (int64_t i = 0; i < N; ++i) V[i + r * N] = i < r ? 0.0 : (i == r ? 1.0 : T[i + r * N] / v0);
    double vv = 0.0;
    for (int64_t i = r; i < N; ++i) vv += V[i + r * N] * V[i + r * N];
    tau[r] = 2.0 / vv;
    for (int c = r; c < k; ++c) {
      double s = 0.0;
      for (int64_t i = r; i < N; ++i) s += V[i + r * N] * T[i + c * N];
      for (int64_t i = r; i < N; ++i) T[i + c * N] -= tau[r] * V[i + r * N] * s;
    }
  }
}

#define MC_SOLVER(call)                                                              \
  do {                                                                               \
    cusolverStatus_t _s = (call);                                                    \
    if (_s != CUSOLVER_STATUS_SUCCESS) {                                             \
      set_error(std::string("cuSOLVER error ") + std::to_string((int)_s) + " in " #call); \
      return MC_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

// One lane of the plan builder: its own stream, cuSOLVER handle and scratch (K, workspace, temporaries).
struct PlanLane {
  cudaStream_t st = nullptr;
  cusolverDnHandle_t h = nullptr;
  double *K = nullptr, *work = nullptr, *X = nullptr, *V = nullptr, *w = nullptr, *p = nullptr, *vec = nullptr;
  int* info = nullptr;
  int lwork = 0;
};

// Plan of one problem into arena slices E (N x (N-k)), lam (N-k), fit_idx (N) on the lane's stream.
static mc_status build_one(mc_ctx* c, PlanLane& ln, TpsPlan& pl, const std::vector<int64_t>& fit) {
  const int n = c->n, d = n - 1, k = d + 1;
  const int64_t N = (int64_t)fit.size();
  const double a0 = c->probs[c->pod[fit[0]]].alpha0;
  std::vector<double> X((size_t)N * d);
  for (int64_t i = 0; i < N; ++i)
    for (int j = 0; j < d; ++j) X[i * d + j] = c->alpha[fit[i] * n + j] / a0;
  std::vector<double> Vh, tau;
  householder_T(X, N, d, Vh, tau);
  cudaStream_t st = ln.st;
  MC_CUDA(cudaMemcpyAsync(ln.X, X.data(), sizeof(double) * N * d, cudaMemcpyHostToDevice, st));
  MC_CUDA(cudaMemcpyAsync(ln.V, Vh.data(), sizeof(double) * N * k, cudaMemcpyHostToDevice, st));
  MC_CUDA(cudaMemcpyAsync(pl.d_fit_idx, fit.data(), sizeof(int64_t) * N, cudaMemcpyHostToDevice, st));
  const dim3 g2((unsigned)((N + 255) / 256), (unsigned)N);
  k_tps_kernel_matrix<<<g2, 256, 0, st>>>(ln.X, N, d, ln.K);
  // B_full = H_k..H_1 K H_1..H_k
  for (int r = 0; r < k; ++r) {
    const double* v = ln.V + (int64_t)r * N;
    k_col_dot<<<(unsigned)N, 256, 0, st>>>(ln.K, N, N, N, v, ln.p);   // A v (A symmetric)
    k_sym_w<<<1, 1024, 0, st>>>(ln.p, v, N, tau[r], ln.w);
    k_rank2<<<g2, 256, 0, st>>>(ln.K, N, v, ln.w);
  }
  MC_CUDA(cudaGetLastError());
  const int64_t m = N - k;
  double* B = ln.K + k + (int64_t)k * N;
  MC_SOLVER(cusolverDnDsyevd(ln.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)m, B, (int)N, pl.d_lam, ln.work,
                             ln.lwork, ln.info));
  // E = H_1 .. H_k [0; V]
  const dim3 g3((unsigned)((N + 255) / 256), (unsigned)m);
  k_embed<<<g3, 256, 0, st>>>(B, N, N, k, pl.d_E);
  for (int r = k - 1; r >= 0; --r) {
    const double* v = ln.V + (int64_t)r * N;
    k_col_dot<<<(unsigned)m, 256, 0, st>>>(pl.d_E, N, m, N, v, ln.vec);
    k_rank1_left<<<g3, 256, 0, st>>>(pl.d_E, N, m, N, v, ln.vec, tau[r]);
  }
  MC_CUDA(cudaGetLastError());
  int info = 0;
  MC_CUDA(cudaMemcpyAsync(&info, ln.info, sizeof(int), cudaMemcpyDeviceToHost, st));
  MC_CUDA(cudaStreamSynchronize(st));   // host vectors above go out of scope; lane reuse
  if (info != 0) {
    set_error("mc_smooth_plan: Dsyevd failed (info = " + std::to_string(info) + ")");
    return MC_ERR_NUMERIC;
  }
  pl.nfit = N;
  pl.d = d;
  pl.passthrough = false;
  return MC_OK;
}

// ---- batched plan builder: problems with equal fitted-set sizes N share ONE cusolverDnXsyevBatched call
// (N = 2000: 12.5 ms per matrix at batch 32, 11.5 at 64, 9.9 at 128, 9.5 at 171 — profiles/r02/plan_batch*.jsonl —
// vs 28 ms with Dsyevd one by one).  cuSOLVER 12.9's XsyevBatched rejects large batches with INVALID_VALUE
// (m = 1997: 171 matrices accepted, 192 rejected — profiles/r02/plan_batch_limit.jsonl), so a batch holds at
// most MC_PLAN_BATCH matrices AND at most MC_PLAN_BATCH_ELEMS matrix elements (B m^2),
// and a batch whose workspace query is still rejected is split in halves and retried. ----------------------
#ifndef MC_PLAN_BATCH
#define MC_PLAN_BATCH 256      // matrices per batched eigensolver call
#endif
#ifndef MC_PLAN_BATCH_ELEMS
#define MC_PLAN_BATCH_ELEMS 682000000LL   // 171 x 1997^2 = 6.82e8 accepted (C2 single GPU: 3 batches of 171)
#endif
#ifndef MC_PLAN_BATCH_MIN
#define MC_PLAN_BATCH_MIN 4    // smaller equal-size groups take the per-problem Dsyevd lanes
#endif

struct BatchScratch {
  double *K = nullptr, *X = nullptr, *V = nullptr, *p = nullptr, *w = nullptr, *vec = nullptr, *Ab = nullptr, *W = nullptr;
  int* info = nullptr;
  void* work = nullptr;
  size_t work_bytes = 0;
  std::vector<char> host_work;
  ~BatchScratch() {
    cudaFree(K); cudaFree(X); cudaFree(V); cudaFree(p); cudaFree(w); cudaFree(vec); cudaFree(Ab); cudaFree(W);
    cudaFree(info); cudaFree(work);
  }
};

static mc_status alloc_batch_scratch(BatchScratch& bs, cusolverDnHandle_t h, cusolverDnParams_t prm, int64_t N, int d,
                                     int64_t B) {
  const int k = d + 1;
  const int64_t m = N - k;
  MC_CUDA(cudaMalloc(&bs.K, sizeof(double) * N * N));
  MC_CUDA(cudaMalloc(&bs.X, sizeof(double) * N * 3));
  MC_CUDA(cudaMalloc(&bs.V, sizeof(double) * B * N * k));
  MC_CUDA(cudaMalloc(&bs.p, sizeof(double) * N));
  MC_CUDA(cudaMalloc(&bs.w, sizeof(double) * N));
  MC_CUDA(cudaMalloc(&bs.vec, sizeof(double) * N));
  MC_CUDA(cudaMalloc(&bs.Ab, sizeof(double) * B * m * m));
  MC_CUDA(cudaMalloc(&bs.W, sizeof(double) * B * m));
  MC_CUDA(cudaMalloc(&bs.info, sizeof(int) * B));
  size_t wd = 0, wh = 0;
  MC_SOLVER(cusolverDnXsyevBatched_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, CUDA_R_64F,
                                              bs.Ab, m, CUDA_R_64F, bs.W, CUDA_R_64F, &wd, &wh, B));
  bs.work_bytes = std::max<size_t>(wd, 1);
  MC_CUDA(cudaMalloc(&bs.work, bs.work_bytes));
  bs.host_work.assign(std::max<size_t>(wh, 1), 0);
  return MC_OK;
}

// Plans of the problems ks (all with N fitted sites) through one batched eigensolver call on stream st.
static mc_status build_batch(mc_ctx* c, const std::vector<int>& ks, const std::vector<std::vector<int64_t>>& fits,
                             cudaStream_t st, cusolverDnHandle_t h, cusolverDnParams_t prm, BatchScratch& bs) {
  const int n = c->n, d = n - 1, k = d + 1;
  const int64_t N = (int64_t)fits[ks[0]].size(), m = N - k, B = (int64_t)ks.size();
  std::vector<std::vector<double>> taus(B);
  const dim3 g2((unsigned)((N + 255) / 256), (unsigned)N);
  const dim3 gp((unsigned)((m + 255) / 256), (unsigned)m);
  for (int64_t t = 0; t < B; ++t) {
    const auto& fit = fits[ks[t]];
    TpsPlan& pl = c->plans[ks[t]];
    const double a0 = c->probs[c->pod[fit[0]]].alpha0;
    std::vector<double> X((size_t)N * d), Vh;
    for (int64_t i = 0; i < N; ++i)
      for (int j = 0; j < d; ++j) X[i * d + j] = c->alpha[fit[i] * n + j] / a0;
    householder_T(X, N, d, Vh, taus[t]);
    double* Vt = bs.V + t * N * k;
    MC_CUDA(cudaMemcpyAsync(bs.X, X.data(), sizeof(double) * N * d, cudaMemcpyHostToDevice, st));
    MC_CUDA(cudaMemcpyAsync(Vt, Vh.data(), sizeof(double) * N * k, cudaMemcpyHostToDevice, st));
    MC_CUDA(cudaMemcpyAsync(pl.d_fit_idx, fit.data(), sizeof(int64_t) * N, cudaMemcpyHostToDevice, st));
    MC_CUDA(cudaStreamSynchronize(st));   // the host vectors go out of scope
    k_tps_kernel_matrix<<<g2, 256, 0, st>>>(bs.X, N, d, bs.K);
    for (int r = 0; r < k; ++r) {
      const double* v = Vt + (int64_t)r * N;
      k_col_dot<<<(unsigned)N, 256, 0, st>>>(bs.K, N, N, N, v, bs.p);
      k_sym_w<<<1, 1024, 0, st>>>(bs.p, v, N, taus[t][r], bs.w);
      k_rank2<<<g2, 256, 0, st>>>(bs.K, N, v, bs.w);
    }
    k_pack<<<gp, 256, 0, st>>>(bs.K, N, k, bs.Ab + t * m * m);
    MC_CUDA(cudaGetLastError());
  }
  MC_SOLVER(cusolverDnXsyevBatched(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, CUDA_R_64F, bs.Ab, m,
                                   CUDA_R_64F, bs.W, CUDA_R_64F, bs.work, bs.work_bytes, bs.host_work.data(),
                                   bs.host_work.size(), bs.info, B));
  const dim3 g3((unsigned)((N + 255) / 256), (unsigned)m);
  for (int64_t t = 0; t < B; ++t) {
    TpsPlan& pl = c->plans[ks[t]];
    const double* Vt = bs.V + t * N * k;
    k_embed<<<g3, 256, 0, st>>>(bs.Ab + t * m * m, m, N, k, pl.d_E);
    for (int r = k - 1; r >= 0; --r) {
      const double* v = Vt + (int64_t)r * N;
      k_col_dot<<<(unsigned)m, 256, 0, st>>>(pl.d_E, N, m, N, v, bs.vec);
      k_rank1_left<<<g3, 256, 0, st>>>(pl.d_E, N, m, N, v, bs.vec, taus[t][r]);
    }
    MC_CUDA(cudaMemcpyAsync(pl.d_lam, bs.W + t * m, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
    MC_CUDA(cudaGetLastError());
  }
  std::vector<int> info(B);
  MC_CUDA(cudaMemcpyAsync(info.data(), bs.info, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  MC_CUDA(cudaStreamSynchronize(st));
  for (int64_t t = 0; t < B; ++t) {
    if (info[t] != 0) {
      set_error("mc_smooth_plan: batched syev failed for problem " + std::to_string(ks[t]) + " (info = " +
                std::to_string(info[t]) + ")");
      return MC_ERR_NUMERIC;
    }
    TpsPlan& pl = c->plans[ks[t]];
    pl.nfit = N;
    pl.d = d;
    pl.passthrough = false;
  }
  return MC_OK;
}

#ifndef MC_PLAN_LANES
#define MC_PLAN_LANES 4
#endif
constexpr int PLAN_LANES = MC_PLAN_LANES;   // concurrent plan builders (streams + cuSOLVER handles); cuSOLVER Dsyevd
// barely overlaps across streams: 4 lanes measured best (24 ms/problem at N = 2000; 8 lanes 30-41 ms, 1 lane 28 ms)

mc_status smooth_plan(mc_ctx* c, const uint8_t* mask, cudaStream_t st) {
  cudaFree(c->d_plan_arena);
  c->d_plan_arena = nullptr;
  c->plans.assign(c->n_probs, TpsPlan{});
  c->plan_built = false;
  const int d = c->n - 1;
  if (d > 3) {
    set_error("mc_smooth_plan: TPS over more than 3 free alpha coordinates is not supported (n <= 4)");
    return MC_ERR_INVALID;
  }
  MC_CUDA(cudaStreamSynchronize(st));   // the caller's values / alpha are settled
  // fitted sets, arena layout (E, lam, fit_idx per plan) and the largest set (lane scratch)
  std::vector<std::vector<int64_t>> fits(c->n_probs);
  int64_t Nmax = 0;
  size_t arena = 0;
  std::vector<size_t> offE(c->n_probs), offL(c->n_probs), offI(c->n_probs);
  std::vector<int> todo;
  for (int k = 0; k < c->n_probs; ++k) {
    TpsPlan& pl = c->plans[k];
    pl.begin = c->prob_begin[k];
    pl.count = c->prob_begin[k + 1] - c->prob_begin[k];
    for (int64_t i = pl.begin; i < pl.begin + pl.count; ++i)
      if (!mask || mask[i]) fits[k].push_back(i);
    const int64_t N = (int64_t)fits[k].size();
    if (d >= 1 && N >= d + 2) {
      Nmax = std::max<int64_t>(Nmax, N);
      const int64_t m = N - d - 1;
      offE[k] = arena; arena += (size_t)N * m;
      offL[k] = arena; arena += (size_t)m;
      offI[k] = arena; arena += (size_t)N;    // int64 fits a double slot
      todo.push_back(k);
    }
  }
  if (!todo.empty()) {
    MC_CUDA(cudaMalloc(&c->d_plan_arena, sizeof(double) * arena));
    for (int k : todo) {
      c->plans[k].d_E = c->d_plan_arena + offE[k];
      c->plans[k].d_lam = c->d_plan_arena + offL[k];
      c->plans[k].d_fit_idx = reinterpret_cast<int64_t*>(c->d_plan_arena + offI[k]);
    }
    // equal-size groups of >= MC_PLAN_BATCH_MIN problems: batched eigensolver, in near-equal batches
    std::map<int64_t, std::vector<int>> by_n;
    for (int k : todo) by_n[(int64_t)fits[k].size()].push_back(k);
    std::vector<std::vector<int>> batches;
    std::vector<int> rest;
    for (auto& kv : by_n) {
      const auto& ks = kv.second;
      if ((int)ks.size() < MC_PLAN_BATCH_MIN) { rest.insert(rest.end(), ks.begin(), ks.end()); continue; }
      const int64_t mm = kv.first - d - 1;
      const size_t cap = (size_t)std::max<int64_t>(1, std::min<int64_t>(MC_PLAN_BATCH, MC_PLAN_BATCH_ELEMS / (mm * mm)));
      const size_t nb = (ks.size() + cap - 1) / cap, per = (ks.size() + nb - 1) / nb;
      for (size_t i = 0; i < ks.size(); i += per)
        batches.emplace_back(ks.begin() + i, ks.begin() + std::min(ks.size(), i + per));
    }
    if (!batches.empty()) {
      cudaStream_t bst = nullptr;
      cusolverDnHandle_t bh = nullptr;
      cusolverDnParams_t prm = nullptr;
      mc_status s = MC_OK;
      // highest priority, as the Dsyevd lanes below: built during the MC pass (Design.smooth_plan(wait=False)),
      // the eigensolver's latency-bound blocks are scheduled ahead of queued MC blocks
      int prio_lo = 0, prio_hi = 0;
      cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
      cudaError_t e = cudaStreamCreateWithPriority(&bst, cudaStreamNonBlocking, prio_hi);
      if (e != cudaSuccess) s = cuda_fail(e, "plan batch stream");
      if (s == MC_OK && (cusolverDnCreate(&bh) != CUSOLVER_STATUS_SUCCESS || cusolverDnCreateParams(&prm) != CUSOLVER_STATUS_SUCCESS)) {
        set_error("cusolverDnCreate failed");
        s = MC_ERR_CUDA;
      }
      if (s == MC_OK) cusolverDnSetStream(bh, bst);
      // scratch sized for the largest N and batch
      int64_t bN = 0, bB = 0;
      for (auto& b : batches) { bN = std::max<int64_t>(bN, (int64_t)fits[b[0]].size()); bB = std::max<int64_t>(bB, (int64_t)b.size()); }
      int64_t cur_N = -1, cur_B = -1;
      std::unique_ptr<BatchScratch> bs;
      for (size_t i = 0; i < batches.size() && s == MC_OK; ++i) {
        const int64_t N = (int64_t)fits[batches[i][0]].size(), B = (int64_t)batches[i].size();
        if (N != cur_N || B > cur_B) {
          bs.reset(new BatchScratch());
          const int64_t want = std::max<int64_t>(B, N == bN ? bB : B);
          s = alloc_batch_scratch(*bs, bh, prm, N, d, want);
          if (s != MC_OK && B > 1) {
            // the eigensolver rejected this batch size: split the batch in halves and retry (scratch for B/2)
            bs.reset();
            cudaGetLastError();
            std::vector<int> lo(batches[i].begin(), batches[i].begin() + B / 2), hi(batches[i].begin() + B / 2, batches[i].end());
            batches[i] = lo;
            batches.insert(batches.begin() + i + 1, hi);
            bB = std::min<int64_t>(bB, (int64_t)hi.size());
            cur_N = cur_B = -1;
            s = MC_OK;
            --i;
            continue;
          }
          cur_N = N;
          cur_B = want;
          if (s != MC_OK) break;
        }
        s = build_batch(c, batches[i], fits, bst, bh, prm, *bs);
      }
      bs.reset();
      if (prm) cusolverDnDestroyParams(prm);
      if (bh) cusolverDnDestroy(bh);
      if (bst) cudaStreamDestroy(bst);
      if (s != MC_OK) return s;
    }
    todo = rest;
  }
  if (!todo.empty()) {
    const int nl = std::min<int>(PLAN_LANES, (int)todo.size());
    std::vector<PlanLane> lanes(nl);
    mc_status s = MC_OK;
    for (int t = 0; t < nl && s == MC_OK; ++t) {
      PlanLane& ln = lanes[t];
      cudaError_t e;
      // highest priority: when the plan is built while the fused MC kernel runs (Design.smooth_plan(wait=False)),
      // the plan's latency-bound cuSOLVER blocks are scheduled ahead of queued MC blocks
      int prio_lo = 0, prio_hi = 0;
      cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
      if ((e = cudaStreamCreateWithPriority(&ln.st, cudaStreamNonBlocking, prio_hi)) != cudaSuccess) { s = cuda_fail(e, "plan stream"); break; }
      if (cusolverDnCreate(&ln.h) != CUSOLVER_STATUS_SUCCESS) { set_error("cusolverDnCreate failed"); s = MC_ERR_CUDA; break; }
      cusolverDnSetStream(ln.h, ln.st);
      if ((e = cudaMalloc(&ln.K, sizeof(double) * Nmax * Nmax)) != cudaSuccess ||
          (e = cudaMalloc(&ln.X, sizeof(double) * Nmax * 3)) != cudaSuccess ||
          (e = cudaMalloc(&ln.V, sizeof(double) * Nmax * 4)) != cudaSuccess ||
          (e = cudaMalloc(&ln.w, sizeof(double) * Nmax)) != cudaSuccess ||
          (e = cudaMalloc(&ln.p, sizeof(double) * Nmax)) != cudaSuccess ||
          (e = cudaMalloc(&ln.vec, sizeof(double) * Nmax)) != cudaSuccess ||
          (e = cudaMalloc(&ln.info, sizeof(int))) != cudaSuccess) { s = cuda_fail(e, "plan lane alloc"); break; }
      // workspace for the largest problem (syevd's requirement grows with n)
      int lw = 0;
      for (int k : todo) {
        const int64_t N = (int64_t)fits[k].size();
        int l = 0;
        cusolverDnDsyevd_bufferSize(ln.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)(N - d - 1), ln.K, (int)N,
                                    ln.w, &l);
        lw = std::max(lw, l);
      }
      ln.lwork = lw;
      if ((e = cudaMalloc(&ln.work, sizeof(double) * (size_t)std::max(lw, 1))) != cudaSuccess) { s = cuda_fail(e, "plan workspace"); break; }
    }
    if (s == MC_OK) {
      std::vector<mc_status> st_lane(nl, MC_OK);
      std::vector<std::string> err_lane(nl);
      auto work = [&](int t) {
        cudaSetDevice(c->device);
        for (size_t i = t; i < todo.size(); i += nl) {
          const int k = todo[i];
          const mc_status r = build_one(c, lanes[t], c->plans[k], fits[k]);
          if (r != MC_OK) { st_lane[t] = r; err_lane[t] = mc_last_error(); return; }
        }
      };
      std::vector<std::thread> th;
      for (int t = 1; t < nl; ++t) th.emplace_back(work, t);
      work(0);
      for (auto& x : th) x.join();
      for (int t = 0; t < nl; ++t)
        if (st_lane[t] != MC_OK) { s = st_lane[t]; set_error(err_lane[t]); break; }
    }
    for (auto& ln : lanes) {
      if (ln.h) cusolverDnDestroy(ln.h);
      if (ln.st) cudaStreamDestroy(ln.st);
      cudaFree(ln.K); cudaFree(ln.work); cudaFree(ln.X); cudaFree(ln.V); cudaFree(ln.w); cudaFree(ln.p);
      cudaFree(ln.vec); cudaFree(ln.info);
    }
    if (s != MC_OK) return s;
  }
  // scratch for y and c: sum of fitted sizes
  int64_t tot = 0;
  for (auto& pl : c->plans) tot += pl.passthrough ? 0 : pl.nfit;
  cudaFree(c->d_tps_scratch);
  c->d_tps_scratch = nullptr;
  c->tps_scratch_elems = 0;
  if (tot > 0) {
    // y [tot], c [tot], PlanDev table
    const size_t bytes = sizeof(double) * 2 * tot + sizeof(PlanDev) * c->n_probs + 64;
    c->n_plans = 0;
    MC_CUDA(cudaMalloc(&c->d_tps_scratch, bytes));
    c->tps_scratch_elems = (size_t)tot;
    std::vector<PlanDev> pd;
    int64_t off = 0;
    for (int k = 0; k < c->n_probs; ++k) {
      const auto& pl = c->plans[k];
      if (pl.passthrough) continue;
      pd.push_back(PlanDev{pl.d_E, pl.d_lam, pl.d_fit_idx, pl.nfit, pl.nfit - pl.d - 1, off, k, pl.d,
                           c->probs[k].alpha0});
      off += pl.nfit;
    }
    c->n_plans = (int)pd.size();
    MC_CUDA(cudaMemcpy(reinterpret_cast<char*>(c->d_tps_scratch) + sizeof(double) * 2 * tot, pd.data(),
                       sizeof(PlanDev) * pd.size(), cudaMemcpyHostToDevice));
  }
  c->plan_built = true;
  return MC_OK;
}

mc_status smooth_apply(mc_ctx* c, const double* values, double lambda, double* out, double* lam_used, cudaStream_t st) {
  // pass-through for every design first (designs outside any fit keep P~ = P^)
  MC_CUDA(cudaMemcpyAsync(out, values, sizeof(double) * c->D, cudaMemcpyDeviceToDevice, st));
  int np = 0;
  int64_t Nmax = 0, kmax = 0;
  for (auto& pl : c->plans)
    if (!pl.passthrough) {
      ++np;
      Nmax = std::max(Nmax, pl.nfit);
      kmax = std::max(kmax, pl.nfit - pl.d - 1);
    }
  if (lam_used) {
    // problems without a fit report lambda = 0 (interpolation / pass-through)
    MC_CUDA(cudaMemsetAsync(lam_used, 0, sizeof(double) * c->n_probs, st));
  }
  if (np == 0 || lambda == 0.0) return MC_OK;
  const int64_t tot = (int64_t)c->tps_scratch_elems;
  double* y = c->d_tps_scratch;
  double* cc = y + tot;
  const PlanDev* pd = reinterpret_cast<const PlanDev*>(reinterpret_cast<char*>(c->d_tps_scratch) + sizeof(double) * 2 * tot);
  k_gather<<<dim3(8, np), 256, 0, st>>>(pd, values, y);
  k_et_y<<<dim3((unsigned)((kmax + 7) / 8), np), 256, 0, st>>>(pd, y, cc);
  k_gcv<<<np, 256, 0, st>>>(pd, lambda, cc, lam_used, 0);
  k_e_c<<<dim3((unsigned)((Nmax + 127) / 128), np), 128, 0, st>>>(pd, y, cc, out);
  c->launches += 4;
  MC_CUDA(cudaGetLastError());
  return MC_OK;
}

}  // namespace mci

namespace mci {

// TPS coefficients (w, beta) of every problem's surface through values (row a9 -> NEXT f1): on the GPU
// c = E^T y, lambda by GCV (or fixed), g = c ./ (Lambda + N lambda), w = E g, K w; on the host
// beta = argmin |T beta - (y - N lambda w - K w)| (the fitted values minus the kernel part; exact since
// (K + N lambda I) w + T beta = y).  Cached in the ctx (tps_x, tps_w, tps_beta, tps_lambda).
mc_status tps_coefficients(mc_ctx* c, const double* values, double lambda, cudaStream_t st) {
  if (!c->plan_built) {
    mc_status s = smooth_plan(c, nullptr, st);
    if (s != MC_OK) return s;
  }
  c->tps_x.assign(c->n_probs, {});
  c->tps_w.assign(c->n_probs, {});
  c->tps_beta.assign(c->n_probs, {});
  c->tps_fitted.assign(c->n_probs, {});
  c->tps_lambda.assign(c->n_probs, 0.0);
  const int np = c->n_plans;
  if (np == 0) return MC_OK;
  int64_t Nmax = 0, kmax = 0;
  for (auto& pl : c->plans)
    if (!pl.passthrough) {
      Nmax = std::max(Nmax, pl.nfit);
      kmax = std::max(kmax, pl.nfit - pl.d - 1);
    }
  const int64_t tot = (int64_t)c->tps_scratch_elems;
  double* y = c->d_tps_scratch;
  double* cc = y + tot;
  const PlanDev* pd = reinterpret_cast<const PlanDev*>(reinterpret_cast<char*>(c->d_tps_scratch) + sizeof(double) * 2 * tot);
  double *w = nullptr, *kw = nullptr, *lam = nullptr;
  MC_CUDA(cudaMallocAsync(&w, sizeof(double) * tot, st));
  MC_CUDA(cudaMallocAsync(&kw, sizeof(double) * tot, st));
  MC_CUDA(cudaMallocAsync(&lam, sizeof(double) * c->n_probs, st));
  k_gather<<<dim3(8, np), 256, 0, st>>>(pd, values, y);
  k_et_y<<<dim3((unsigned)((kmax + 7) / 8), np), 256, 0, st>>>(pd, y, cc);
  k_gcv<<<np, 256, 0, st>>>(pd, lambda, cc, lam, 1);
  k_e_w<<<dim3((unsigned)((Nmax + 127) / 128), np), 128, 0, st>>>(pd, cc, w);
  k_tps_kw<<<dim3((unsigned)((Nmax + 127) / 128), np), 128, 0, st>>>(pd, c->d_alpha, c->n, w, kw);
  c->launches += 5;
  MC_CUDA(cudaGetLastError());
  std::vector<double> hy(tot), hw(tot), hkw(tot), hl(c->n_probs);
  MC_CUDA(cudaMemcpyAsync(hy.data(), y, sizeof(double) * tot, cudaMemcpyDeviceToHost, st));
  MC_CUDA(cudaMemcpyAsync(hw.data(), w, sizeof(double) * tot, cudaMemcpyDeviceToHost, st));
  MC_CUDA(cudaMemcpyAsync(hkw.data(), kw, sizeof(double) * tot, cudaMemcpyDeviceToHost, st));
  MC_CUDA(cudaMemcpyAsync(hl.data(), lam, sizeof(double) * c->n_probs, cudaMemcpyDeviceToHost, st));
  MC_CUDA(cudaStreamSynchronize(st));
  cudaFree(w);
  cudaFree(kw);
  cudaFree(lam);
  int64_t off = 0;
  const int n = c->n;
  for (int k = 0; k < c->n_probs; ++k) {
    const TpsPlan& pl = c->plans[k];
    if (pl.passthrough) continue;
    const int64_t N = pl.nfit;
    const int d = pl.d;
    const double a0 = c->probs[k].alpha0;
    std::vector<int64_t> fit(N);
    MC_CUDA(cudaMemcpy(fit.data(), pl.d_fit_idx, sizeof(int64_t) * N, cudaMemcpyDeviceToHost));
    std::vector<double>& X = c->tps_x[k];
    X.resize((size_t)N * d);
    for (int64_t i = 0; i < N; ++i)
      for (int j = 0; j < d; ++j) X[i * d + j] = c->alpha[fit[i] * n + j] / a0;
    c->tps_w[k].assign(hw.begin() + off, hw.begin() + off + N);
    c->tps_lambda[k] = hl[k];
    c->tps_fitted[k].resize(N);
    for (int64_t i = 0; i < N; ++i) c->tps_fitted[k][i] = hy[off + i] - (double)N * hl[k] * hw[off + i];
    // normal equations T^T T beta = T^T r, r = y - N lambda w - K w
    const int m = d + 1;
    double A[4][4] = {{0}}, b[4] = {0};
    for (int64_t i = 0; i < N; ++i) {
      double t[4] = {1.0, 0, 0, 0};
      for (int j = 0; j < d; ++j) t[j + 1] = X[i * d + j];
      const double r = hy[off + i] - (double)N * hl[k] * hw[off + i] - hkw[off + i];
      for (int a = 0; a < m; ++a) {
        b[a] += t[a] * r;
        for (int bb = 0; bb < m; ++bb) A[a][bb] += t[a] * t[bb];
      }
    }
    // Gaussian elimination with partial pivoting on the (d+1) x (d+1) system
    for (int col = 0; col < m; ++col) {
      int piv = col;
      for (int r = col + 1; r < m; ++r)
        if (std::fabs(A[r][col]) > std::fabs(A[piv][col])) piv = r;
      if (std::fabs(A[piv][col]) < 1e-300) { set_error("tps_coefficients: rank-deficient sites"); return MC_ERR_NUMERIC; }
      for (int j = 0; j < m; ++j) std::swap(A[col][j], A[piv][j]);
      std::swap(b[col], b[piv]);
      for (int r = col + 1; r < m; ++r) {
        const double f = A[r][col] / A[col][col];
        for (int j = col; j < m; ++j) A[r][j] -= f * A[col][j];
        b[r] -= f * b[col];
      }
    }
    std::vector<double> beta(m);
    for (int r = m - 1; r >= 0; --r) {
      double acc = b[r];
      for (int j = r + 1; j < m; ++j) acc -= A[r][j] * beta[j];
      beta[r] = acc / A[r][r];
    }
    c->tps_beta[k] = beta;
    off += N;
  }
  return MC_OK;
}

}  // namespace mci
