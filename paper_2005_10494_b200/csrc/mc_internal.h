// mc_internal.h — library-internal context and launch helpers (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/mc_design.h"

namespace mci {

constexpr int PROB_STRIDE = 144;         // floats per device problem record
constexpr int OFF_M = 0;                 // packed M = diag(c) L_p with the folded row scales (55 floats for n = 10)
constexpr int OFF_RHO = 56;              // IND: rho_i = sqrt(r_{i+1}/r_i)
constexpr int OFF_SD = 66;               // IND: s_i = sqrt(1 - rho_i^2)
constexpr int OFF_ER = 76;               // COND even stage k: mu_k / sd_k
constexpr int OFF_EMU = 81;              // COND even stage k: mu_k (coefficient of x_{k-1})
constexpr int OFF_ESD = 86;              // COND even stage k: conditional sd_k
constexpr int OFF_OA = 91;               // COND odd stage j: left-neighbour coefficient / gamma_j
constexpr int OFF_OB = 96;               // COND odd stage j: right-neighbour coefficient / gamma_j
constexpr int OFF_BSC = 101;             // row scale of b' = b * bsc (dump only)
constexpr int OFF_STR = 112;             // C4 strata model: 17 floats (mc_device.cuh StrataRegs)
constexpr int SAMPLES_PER_THREAD = 128;  // per-thread sample run inside a warp tile (< 512: u32 sums)
constexpr int MAX_BLOCK = 256;           // fused kernel __launch_bounds__
#ifndef MC_MIN_BLOCKS_COND
#define MC_MIN_BLOCKS_COND 5
#endif
#ifndef MC_MIN_BLOCKS_IND
#define MC_MIN_BLOCKS_IND 5
#endif
constexpr int MIN_BLOCKS_COND = MC_MIN_BLOCKS_COND;   // min resident 256-thread blocks per SM, n <= 3 (COND 5: +1.9 % with the packed pair, profiles/r01/tune_f32x2.jsonl)
constexpr int MIN_BLOCKS_IND = MC_MIN_BLOCKS_IND;     //   (register caps 48 / 48)

void set_error(const std::string& msg);
mc_status cuda_fail(cudaError_t e, const char* where);

#define MC_CUDA(call)                                                   \
  do {                                                                  \
    cudaError_t _e = (call);                                            \
    if (_e != cudaSuccess) return mci::cuda_fail(_e, #call);            \
  } while (0)

struct TpsPlan {
  int64_t begin = 0;       // first design of the problem
  int64_t count = 0;       // designs of the problem
  int64_t nfit = 0;        // fitted designs (mask)
  int32_t d = 0;           // TPS dimension
  bool passthrough = true; // too few points / n == 1
  double* fit_idx_dummy = nullptr;
  int64_t* d_fit_idx = nullptr;   // [nfit] global design indices of the fitted designs
  double* d_E = nullptr;          // [nfit x k] column-major, k = nfit - d - 1 (Q2 V)
  double* d_lam = nullptr;        // [k] eigenvalues of Q2^T K Q2
};

}  // namespace mci

struct mc_ctx {
  int device = 0;
  int n = 0;
  int est = 0;
  int model = 0;                         // 0 Gaussian prior (Formula 10 / general), 1 C4 strata prior
  int sampling = 0;                      // 0 independent draws per design, 1 common random numbers (f3)
  int32_t* d_crn = nullptr;              // CRN design blocks (first, count, problem) for [crn_d0, +crn_dc)
  int64_t crn_blocks = 0, crn_d0 = -1, crn_dc = -1;
  int crn_kd = 0;
  int32_t n_probs = 0;
  int64_t D = 0;
  uint64_t seed = 0;
  std::vector<mc_problem> probs;
  std::vector<double> alpha;             // host copy [D*n]
  std::vector<int32_t> pod;              // host copy [D]
  std::vector<int64_t> prob_begin;       // [n_probs+1]
  float* d_prob = nullptr;               // [n_probs * PROB_STRIDE]
  float* d_zc = nullptr;                 // [D * n]
  double* d_alpha = nullptr;             // [D * n] fp64 design table
  double* d_ctheta = nullptr;            // [n_probs * n * 2] (c_i theta_i, row scale bsc_i)
  int32_t* d_pod = nullptr;              // [D]
  int64_t* d_prob_begin = nullptr;       // [n_probs+1]
  int block_threads = 256;
  int grid_blocks = 0;                   // 0 = auto
  std::atomic<int64_t> launches{0};       // atomic: the plan builder may run on another host thread
  bool plan_built = false;
  std::vector<mci::TpsPlan> plans;
  double* d_tps_scratch = nullptr;       // per-problem scratch for smoothing
  double* d_plan_arena = nullptr;        // all TPS plans (E, Lambda, fitted indices) in one allocation
  size_t tps_scratch_elems = 0;
  int n_plans = 0;
  // TPS coefficients of the last mc_refine (host): per problem sites, w, beta
  std::vector<std::vector<double>> tps_x, tps_w, tps_beta;
  std::vector<std::vector<double>> tps_fitted;   // the TPS value at each fitted site: y - N lambda w
  std::vector<double> tps_lambda;
};

// launchers implemented in the .cu files
namespace mci {
mc_status launch_fused(mc_ctx* c, int64_t d0, int64_t dcount, uint64_t B, uint64_t E, cudaStream_t st,
                       int64_t* sums);
mc_status launch_finalize(mc_ctx* c, const int64_t* sums, uint64_t N, double* mean, double* var, cudaStream_t st);
mc_status launch_philox_dump(uint64_t seed, uint32_t tag, int form, const uint32_t* id, const uint64_t* word,
                             int64_t count, uint32_t* out, cudaStream_t st);
mc_status launch_draw_dump(mc_ctx* c, const int64_t* design, const uint64_t* sample, int64_t count, float* out,
                           cudaStream_t st);
int draw_dump_stride(int n, int est, int model);
int words_per_record(int n, int est, int model);
mc_status launch_zc(mc_ctx* c, cudaStream_t st);
mc_status launch_argmax(mc_ctx* c, const double* values, int64_t* idx, double* val, cudaStream_t st);
mc_status alpha_grid_solve(const mc_problem* probs, int32_t n_probs, int32_t m, int device,
                           std::vector<double>& alpha, std::vector<uint8_t>& valid);
mc_status alpha_points_solve(const mc_problem* probs, int32_t n_probs, const int32_t* prob, int64_t count, int device,
                             double* A, uint8_t* valid);
mc_status fwer_eval(const mc_problem* p, const double* alpha, int64_t count, double* out, int device);
mc_status smooth_plan(mc_ctx* c, const uint8_t* mask, cudaStream_t st);
struct RefineOut {
  std::vector<double> x;
  double f = 0.0;
  int iters = 0;
};
// maximise the TPS f(x) = beta0 + beta.x + sum w_i phi(|x - X_i|) over lo <= x <= hi from x0 (mc_refine.cu)
RefineOut refine_box(const std::vector<double>& X, const std::vector<double>& w, const std::vector<double>& beta, int d,
                     const std::vector<double>& x0, const std::vector<double>& lo, const std::vector<double>& hi);
mc_status tps_coefficients(mc_ctx* c, const double* values, double lambda, cudaStream_t st);
mc_status smooth_apply(mc_ctx* c, const double* values, double lambda, double* out, double* lam_used,
                       cudaStream_t st);
}  // namespace mci
