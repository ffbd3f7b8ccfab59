// mc_gridsmooth.cu — the dense-grid smoother of configuration C4 (SURVEY §8(a) a9 "Dense regular
// grids (C4)", reading R23).
//
// P~ = S_r P^ S_a^T over a regular (r, alpha) design grid P^[nr][na] (row-major), S_x the row-normalised
// Gaussian (Nadaraya-Watson) weights W_x[i][k] = exp(-(x_i - x_k)^2 / (2 h_x^2)).  Bandwidths h = k x
// (grid step) with k = 2^(j/2), j = -2..8, chosen jointly by GCV(h) = (1/n)||P^ - P~||^2 / (1 - tr S/n)^2,
// tr S = tr S_r tr S_a, first minimiser with the r bandwidth outer (the oracle's order).
//
// Kernels: k_nw_matrix builds all 11 S_x (one block per (row, bandwidth), deterministic tree sums);
// the two products per bandwidth pair are fp64 GEMMs in k_dgemm (this file; 256^3 each for C4, batched
// over the alpha bandwidths; DFMA on the FP64 pipe — under 1 ms per GCV scan, so no tensor-core path);
// k_grid_rss reduces ||P^ - P~||^2 per pair in a fixed order (one block per pair), so the GCV choice is
// deterministic.  All fp64, fixed summation orders.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "mc_internal.h"

namespace mci {

constexpr int GS_NH = 11;          // bandwidth grid size
constexpr int GS_THREADS = 256;

// S[j][i][k] = W[i][k] / sum_k W[i][k], W = exp(-(x_i - x_k)^2 / (2 h_j^2)); diag[j][i] = S[j][i][i].
__global__ void __launch_bounds__(GS_THREADS) k_nw_matrix(const double* __restrict__ x, int m,
                                                          const double* __restrict__ h, double* __restrict__ S,
                                                          double* __restrict__ diag) {
  __shared__ double red[GS_THREADS];
  const int i = blockIdx.x, j = blockIdx.y;
  const double xi = x[i], inv = 1.0 / h[j];
  double s = 0.0;
  for (int k = threadIdx.x; k < m; k += GS_THREADS) {
    const double t = (xi - x[k]) * inv;
    s += exp(-0.5 * t * t);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = GS_THREADS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double rs = 1.0 / red[0];
  double* row = S + ((int64_t)j * m + i) * m;
  for (int k = threadIdx.x; k < m; k += GS_THREADS) {
    const double t = (xi - x[k]) * inv;
    row[k] = exp(-0.5 * t * t) * rs;
  }
  if (threadIdx.x == 0) diag[(int64_t)j * m + i] = rs;   // W[i][i] = 1
}

// rss[c] = sum (P - Ps[c])^2 over the n grid values, one block per candidate c (fixed reduction order).
__global__ void __launch_bounds__(GS_THREADS) k_grid_rss(const double* __restrict__ P, const double* __restrict__ Ps,
                                                         int64_t n, double* __restrict__ rss) {
  __shared__ double red[GS_THREADS];
  const double* q = Ps + (int64_t)blockIdx.x * n;
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += GS_THREADS) {
    const double d = P[k] - q[k];
    s = fma(d, d, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = GS_THREADS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) rss[blockIdx.x] = red[0];
}

// C[z] = A[z] op(B[z]) for z = blockIdx.z, row-major: A is M x K (lda), op(B) = B (K x N, ldb) or, with
// BT, B^T for B stored N x K (ldb); element strides sA, sB, sC between batch entries (0 = shared operand).
// 64 x 64 output tile per 256-thread block (4 x 4 outputs per thread), K in slabs of 16 through shared
// memory; each output is one DFMA chain in k order (deterministic).
constexpr int DG_T = 64, DG_K = 16;
template <bool BT>
__global__ void __launch_bounds__(256) k_dgemm(int M, int N, int K, const double* __restrict__ A, int lda, int64_t sA,
                                               const double* __restrict__ B, int ldb, int64_t sB, double* __restrict__ C,
                                               int ldc, int64_t sC) {
  __shared__ double As[DG_K][DG_T + 1];
  __shared__ double Bs[DG_K][DG_T + 1];
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  C += blockIdx.z * sC;
  const int m0 = blockIdx.y * DG_T, n0 = blockIdx.x * DG_T;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += DG_K) {
    for (int e = threadIdx.x; e < DG_T * DG_K; e += blockDim.x) {
      const int r = e / DG_K, kk = e % DG_K, gm = m0 + r, gk = k0 + kk;
      As[kk][r] = (gm < M && gk < K) ? A[(int64_t)gm * lda + gk] : 0.0;
      if (BT) {
        const int gn = n0 + r;
        Bs[kk][r] = (gn < N && gk < K) ? B[(int64_t)gn * ldb + gk] : 0.0;
      } else {
        const int kb = e / DG_T, c = e % DG_T, gkb = k0 + kb, gn = n0 + c;
        Bs[kb][c] = (gkb < K && gn < N) ? B[(int64_t)gkb * ldb + gn] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < DG_K; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
      if (gm < M && gn < N) C[(int64_t)gm * ldc + gn] = acc[i][j];
    }
}

template <bool BT>
static cudaError_t dgemm(int M, int N, int K, const double* A, int lda, int64_t sA, const double* B, int ldb, int64_t sB,
                         double* C, int ldc, int64_t sC, int batch, cudaStream_t st) {
  const dim3 grid((N + DG_T - 1) / DG_T, (M + DG_T - 1) / DG_T, batch);
  k_dgemm<BT><<<grid, 256, 0, st>>>(M, N, K, A, lda, sA, B, ldb, sB, C, ldc, sC);
  return cudaGetLastError();
}

namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
};
}  // namespace

}  // namespace mci

using namespace mci;



extern "C" {

mc_status mc_grid_smooth(const double* values_dev, int32_t nr, int32_t na, const double* xr_host,
                         const double* xa_host, double hr, double ha, double* smoothed_dev, double* h_used_host,
                         void* cuda_stream) {
  if (!values_dev || !smoothed_dev || !xr_host || !xa_host) { set_error("mc_grid_smooth: null pointer"); return MC_ERR_INVALID; }
  if (nr < 2 || na < 2 || nr > 4096 || na > 4096) { set_error("mc_grid_smooth: grid sides must be in [2, 4096]"); return MC_ERR_INVALID; }
  for (int i = 1; i < nr; ++i)
    if (!(xr_host[i] > xr_host[i - 1])) { set_error("mc_grid_smooth: r coordinates must be strictly increasing"); return MC_ERR_INVALID; }
  for (int i = 1; i < na; ++i)
    if (!(xa_host[i] > xa_host[i - 1])) { set_error("mc_grid_smooth: alpha coordinates must be strictly increasing"); return MC_ERR_INVALID; }
  const bool gcv = !(hr > 0.0) || !(ha > 0.0);
  if (!gcv && (!std::isfinite(hr) || !std::isfinite(ha))) { set_error("mc_grid_smooth: bandwidths must be finite"); return MC_ERR_INVALID; }
  cudaStream_t st = (cudaStream_t)cuda_stream;

  const int nh = gcv ? GS_NH : 1;
  std::vector<double> h_r(nh), h_a(nh);
  const double sr = (xr_host[nr - 1] - xr_host[0]) / (nr - 1), sa = (xa_host[na - 1] - xa_host[0]) / (na - 1);
  for (int j = 0; j < nh; ++j) {
    const double k = gcv ? std::exp2((j - 2) / 2.0) : 1.0;   // 2^(j/2), j = -2..8 (oracle GRID_H_STEPS)
    h_r[j] = gcv ? k * sr : hr;
    h_a[j] = gcv ? k * sa : ha;
  }
  const int64_t n = (int64_t)nr * na;
  // workspace: x_r, x_a, h_r, h_a, S_r[nh], S_a[nh], diag_r, diag_a, T, Ps[nh], rss[nh*nh]
  const size_t cnt = (size_t)nr + na + 2 * nh + (size_t)nh * nr * nr + (size_t)nh * na * na + (size_t)nh * (nr + na) +
                     (size_t)n + (size_t)nh * n + (size_t)nh * nh;
  DevBuf ws;
  MC_CUDA(cudaMalloc(&ws.p, cnt * sizeof(double)));
  double* d_xr = (double*)ws.p;
  double* d_xa = d_xr + nr;
  double* d_hr = d_xa + na;
  double* d_ha = d_hr + nh;
  double* d_Sr = d_ha + nh;
  double* d_Sa = d_Sr + (size_t)nh * nr * nr;
  double* d_dr = d_Sa + (size_t)nh * na * na;
  double* d_da = d_dr + (size_t)nh * nr;
  double* d_T = d_da + (size_t)nh * na;
  double* d_Ps = d_T + n;
  double* d_rss = d_Ps + (size_t)nh * n;
  MC_CUDA(cudaMemcpyAsync(d_xr, xr_host, sizeof(double) * nr, cudaMemcpyHostToDevice, st));
  MC_CUDA(cudaMemcpyAsync(d_xa, xa_host, sizeof(double) * na, cudaMemcpyHostToDevice, st));
  MC_CUDA(cudaMemcpyAsync(d_hr, h_r.data(), sizeof(double) * nh, cudaMemcpyHostToDevice, st));
  MC_CUDA(cudaMemcpyAsync(d_ha, h_a.data(), sizeof(double) * nh, cudaMemcpyHostToDevice, st));
  k_nw_matrix<<<dim3(nr, nh), GS_THREADS, 0, st>>>(d_xr, nr, d_hr, d_Sr, d_dr);
  k_nw_matrix<<<dim3(na, nh), GS_THREADS, 0, st>>>(d_xa, na, d_ha, d_Sa, d_da);
  MC_CUDA(cudaGetLastError());
  // T = S_r P (nr x na), then Ps[ja] = T S_a[ja]^T for every alpha bandwidth (row-major)
  int jr_best = 0, ja_best = 0;
  if (gcv) {
    std::vector<double> dr((size_t)nh * nr), da((size_t)nh * na), rss((size_t)nh * nh);
    for (int jr = 0; jr < nh; ++jr) {
      MC_CUDA(dgemm<false>(nr, na, nr, d_Sr + (size_t)jr * nr * nr, nr, 0, values_dev, na, 0, d_T, na, 0, 1, st));
      MC_CUDA(dgemm<true>(nr, na, na, d_T, na, 0, d_Sa, na, (int64_t)na * na, d_Ps, na, n, nh, st));
      k_grid_rss<<<nh, GS_THREADS, 0, st>>>(values_dev, d_Ps, n, d_rss + (size_t)jr * nh);
      MC_CUDA(cudaGetLastError());
    }
    MC_CUDA(cudaMemcpyAsync(rss.data(), d_rss, sizeof(double) * nh * nh, cudaMemcpyDeviceToHost, st));
    MC_CUDA(cudaMemcpyAsync(dr.data(), d_dr, sizeof(double) * nh * nr, cudaMemcpyDeviceToHost, st));
    MC_CUDA(cudaMemcpyAsync(da.data(), d_da, sizeof(double) * nh * na, cudaMemcpyDeviceToHost, st));
    MC_CUDA(cudaStreamSynchronize(st));
    double best = INFINITY;
    for (int jr = 0; jr < nh; ++jr) {
      double tr_r = 0.0;
      for (int i = 0; i < nr; ++i) tr_r += dr[(size_t)jr * nr + i];
      for (int ja = 0; ja < nh; ++ja) {
        double tr_a = 0.0;
        for (int i = 0; i < na; ++i) tr_a += da[(size_t)ja * na + i];
        const double den = 1.0 - tr_r * tr_a / (double)n;
        const double g = rss[(size_t)jr * nh + ja] / (double)n / (den * den);
        if (g < best) { best = g; jr_best = jr; ja_best = ja; }
      }
    }
  }
  MC_CUDA(dgemm<false>(nr, na, nr, d_Sr + (size_t)jr_best * nr * nr, nr, 0, values_dev, na, 0, d_T, na, 0, 1, st));
  MC_CUDA(dgemm<true>(nr, na, na, d_T, na, 0, d_Sa + (size_t)ja_best * na * na, na, 0, smoothed_dev, na, 0, 1, st));
  if (h_used_host) { h_used_host[0] = h_r[jr_best]; h_used_host[1] = h_a[ja_best]; }
  // the workspace is freed below: wait for the products that read it
  MC_CUDA(cudaStreamSynchronize(st));
  return MC_OK;
}

}  // extern "C"
