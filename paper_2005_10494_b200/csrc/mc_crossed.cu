// mc_crossed.cu — NEXT f3 (ii): the paper-literal crossed estimator of Formula 7.
//
// Formula 7 pairs every outer prior draw Delta^(k) (k < N1, Formula 5) with every inner null draw x^(l)
// (l < N2, Formula 6): P^ = 1 - (N1 N2)^-1 sum_k sum_l delta(x^(l) <= z - c Delta^(k)).  Per design:
// outer stream (design, tag 2), 2ceil(p/2) words per draw; inner stream (design, tag 3), 2ceil(n/2)
// words per draw.  Integer sums S1 = sum_k c_k, S2 = sum_k c_k^2 with
// c_k = #{l : exists i, x_i^(l) > b_i^(k)}.
//
// Kernel: a block owns (design, 256 x KO outer draws) with b^(k) in registers; the inner set is
// generated cooperatively in shared-memory chunks of 1024 draws and broadcast to every thread, so each
// (k, l) pair costs n FSETP + a predicate merge + an add.  Requires the IND record folding (ctx built
// with MC_EST_IND): b' = b / BM_K and X' = X / BM_K.
#include <cuda_runtime.h>

#include <cstdint>

#include "mc_device.cuh"
#include "mc_internal.h"

namespace mci {

using namespace mcd;

constexpr int XO_KO = 4;          // outer draws per thread
constexpr int XO_THREADS = 256;
constexpr int XI_CHUNK = 1024;    // inner draws per shared-memory chunk

template <int N>
__device__ __forceinline__ void load_problem_x(const float* __restrict__ rec, ProbRegs<N>& pr) {
#pragma unroll
  for (int k = 0; k < N * (N + 1) / 2; ++k) pr.M[k] = __ldg(rec + OFF_M + k);
#pragma unroll
  for (int k = 0; k < N - 1; ++k) {
    pr.rho[k] = __ldg(rec + OFF_RHO + k);
    pr.sd[k] = __ldg(rec + OFF_SD + k);
  }
}

template <int N>
__global__ void __launch_bounds__(XO_THREADS) k_crossed(const float* __restrict__ prob, const float* __restrict__ zc_all,
                                                        const int32_t* __restrict__ pod, uint64_t seed, uint64_t n1,
                                                        uint64_t n2, int64_t outer_blocks_per_design,
                                                        unsigned long long* __restrict__ sums) {
  __shared__ float xs[XI_CHUNK][N];
  __shared__ unsigned long long red[2][XO_THREADS / 32];
  constexpr int P = N;                          // Gaussian prior dimension
  constexpr int UO = 2 * ((P + 1) / 2);         // outer words per draw
  constexpr int UI = 2 * ((N + 1) / 2);         // inner words per draw
  const int64_t d = blockIdx.x / outer_blocks_per_design;
  const int64_t ob = blockIdx.x % outer_blocks_per_design;
  const float* rec = prob + (int64_t)pod[d] * PROB_STRIDE;
  ProbRegs<N> pr;
  load_problem_x<N>(rec, pr);
  const uint32_t one = 0x3F800000u;
  // outer draws of this thread: b'(k) = zc' - M eps'
  float bo[XO_KO][N];
  bool live[XO_KO];
#pragma unroll
  for (int j = 0; j < XO_KO; ++j) {
    const uint64_t k = (uint64_t)ob * XO_THREADS * XO_KO + (uint64_t)j * XO_THREADS + threadIdx.x;
    live[j] = k < n1;
    uint32_t w[UO];
#pragma unroll
    for (int t = 0; t < UO; ++t) w[t] = philox_word_tagged(seed, (uint32_t)d, 2u, k * UO + t);
    float nrm[UO];
#pragma unroll
    for (int t = 0; t < UO / 2; ++t) box_muller_scaled(w[2 * t], w[2 * t + 1], one, nrm[2 * t], nrm[2 * t + 1]);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      float acc = __ldg(zc_all + d * N + i);
#pragma unroll
      for (int c = 0; c <= i; ++c) acc = fmaf(-pr.M[i * (i + 1) / 2 + c], nrm[c], acc);
      bo[j][i] = live[j] ? acc : __int_as_float(0x7f800000);   // dead slots never count
    }
  }
  uint32_t cnt[XO_KO] = {0};
  for (uint64_t l0 = 0; l0 < n2; l0 += XI_CHUNK) {
    __syncthreads();
    for (int t = threadIdx.x; t < XI_CHUNK; t += XO_THREADS) {
      const uint64_t l = l0 + t;
      if (l < n2) {
        uint32_t w[UI];
#pragma unroll
        for (int u = 0; u < UI; ++u) w[u] = philox_word_tagged(seed, (uint32_t)d, 3u, l * UI + u);
        float nrm[UI];
#pragma unroll
        for (int u = 0; u < UI / 2; ++u) box_muller_scaled(w[2 * u], w[2 * u + 1], one, nrm[2 * u], nrm[2 * u + 1]);
        float x = nrm[0];
        xs[t][0] = x;
#pragma unroll
        for (int i = 1; i < N; ++i) {
          x = fmaf(pr.rho[i - 1], x, pr.sd[i - 1] * nrm[i]);
          xs[t][i] = x;
        }
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) xs[t][i] = -__int_as_float(0x7f800000);   // never exceeds b
      }
    }
    __syncthreads();
    const int lim = (int)min((uint64_t)XI_CHUNK, n2 - l0);
    // per (k, l) pair: one FSETP + (N-1) FSETP.OR on the ALU pipe and ONE predicated FADD on the FMA pipe
    // (the count runs in fp32 within a chunk, exact below 2^24, and is folded into the integer per chunk)
    float cf[XO_KO];
#pragma unroll
    for (int j = 0; j < XO_KO; ++j) cf[j] = 0.0f;
    for (int t = 0; t < lim; ++t) {
      float x[N];
#pragma unroll
      for (int i = 0; i < N; ++i) x[i] = xs[t][i];
#pragma unroll
      for (int j = 0; j < XO_KO; ++j) ind_count<N>(x, bo[j], cf[j]);
    }
#pragma unroll
    for (int j = 0; j < XO_KO; ++j) cnt[j] += (uint32_t)cf[j];
  }
  unsigned long long s1 = 0, s2 = 0;
#pragma unroll
  for (int j = 0; j < XO_KO; ++j) {
    s1 += cnt[j];
    s2 += (unsigned long long)cnt[j] * cnt[j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = s1; red[1][threadIdx.x >> 5] = s2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t1 = 0, t2 = 0;
    for (int k = 0; k < XO_THREADS / 32; ++k) { t1 += red[0][k]; t2 += red[1][k]; }
    atomicAdd(sums + 2 * d, t1);
    atomicAdd(sums + 2 * d + 1, t2);
  }
}

// crossed finalize: mean = S1/(N1 N2); var = sample variance over k of c_k/N2 (SE = sqrt(var/N1))
__global__ void k_finalize_crossed(const long long* __restrict__ sums, int64_t D, double n1, double n2,
                                   double* __restrict__ mean, double* __restrict__ var) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= D) return;
  const double s1 = (double)sums[2 * d], s2 = (double)sums[2 * d + 1];
  const double m = s1 / (n1 * n2);
  mean[d] = m;
  if (var) var[d] = n1 > 1.0 ? (s2 / (n2 * n2) - n1 * m * m) / (n1 - 1.0) : 0.0;
}

}  // namespace mci

using namespace mci;

extern "C" {

mc_status mc_evaluate_crossed(mc_ctx* c, uint64_t n1, uint64_t n2, void* stream, int64_t* sums) {
  if (!c || !sums) { set_error("mc_evaluate_crossed: null pointer"); return MC_ERR_INVALID; }
  if (c->est != MC_EST_IND || c->model != 0) {
    set_error("mc_evaluate_crossed: the crossed estimator needs a ctx built with MC_EST_IND and a Gaussian prior");
    return MC_ERR_INVALID;
  }
  if (c->n > 4) { set_error("mc_evaluate_crossed: built for n <= 4"); return MC_ERR_INVALID; }
  if (n2 >= ((uint64_t)1 << 32) || n1 == 0 || n2 == 0 || c->D == 0) {
    if (n1 == 0 || n2 == 0 || c->D == 0) return MC_OK;
    set_error("mc_evaluate_crossed: N2 must be < 2^32");
    return MC_ERR_INVALID;
  }
  // S2 = sum_k c_k^2 <= N1 N2^2 must fit the int64 that k_finalize_crossed reads
  if ((unsigned __int128)n1 * n2 * n2 >= ((unsigned __int128)1 << 63)) {
    set_error("mc_evaluate_crossed: N1 N2^2 must be < 2^63 (the int64 sum of c_k^2 would overflow)");
    return MC_ERR_INVALID;
  }
  MC_CUDA(cudaSetDevice(c->device));
  const int64_t obpd = (int64_t)((n1 + XO_THREADS * XO_KO - 1) / (XO_THREADS * XO_KO));
  const int64_t blocks = obpd * c->D;
  if (blocks >= ((int64_t)1 << 31)) { set_error("mc_evaluate_crossed: grid too large"); return MC_ERR_INVALID; }
  cudaStream_t st = (cudaStream_t)stream;
  auto* out = reinterpret_cast<unsigned long long*>(sums);
  switch (c->n) {
    case 1: k_crossed<1><<<(unsigned)blocks, XO_THREADS, 0, st>>>(c->d_prob, c->d_zc, c->d_pod, c->seed, n1, n2, obpd, out); break;
    case 2: k_crossed<2><<<(unsigned)blocks, XO_THREADS, 0, st>>>(c->d_prob, c->d_zc, c->d_pod, c->seed, n1, n2, obpd, out); break;
    case 3: k_crossed<3><<<(unsigned)blocks, XO_THREADS, 0, st>>>(c->d_prob, c->d_zc, c->d_pod, c->seed, n1, n2, obpd, out); break;
    default: k_crossed<4><<<(unsigned)blocks, XO_THREADS, 0, st>>>(c->d_prob, c->d_zc, c->d_pod, c->seed, n1, n2, obpd, out); break;
  }
  c->launches += 1;
  MC_CUDA(cudaGetLastError());
  return MC_OK;
}

mc_status mc_finalize_crossed(mc_ctx* c, const int64_t* sums, uint64_t n1, uint64_t n2, double* mean, double* var,
                              void* stream) {
  if (!c || !sums || !mean || n1 == 0 || n2 == 0) { set_error("mc_finalize_crossed: null pointer or empty"); return MC_ERR_INVALID; }
  MC_CUDA(cudaSetDevice(c->device));
  if (c->D == 0) return MC_OK;
  k_finalize_crossed<<<(unsigned)((c->D + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const long long*>(sums), c->D, (double)n1, (double)n2, mean, var);
  c->launches += 1;
  MC_CUDA(cudaGetLastError());
  return MC_OK;
}

}  // extern "C"
