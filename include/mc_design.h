/*
 * mc_design.h — C ABI of the B200-native Monte-Carlo design-objective library
 * (arXiv 2005.10494, "The Optimal Design of Clinical Trials with Potential Biomarker Effects").
 *
 * Built as paper_2005_10494_b200/libmc_design.so (sm_100a).  All entry points are extern "C",
 * take plain host or device pointers and sizes, and return mc_status (0 = MC_OK).  On error,
 * mc_last_error() returns a thread-local message naming the violated invariant or failing stage.
 * Device pointers ("_dev") are caller-allocated CUDA global memory on the ctx's device; streams are
 * caller streams (cudaStream_t passed as void*, NULL = legacy default stream).  The library never
 * synchronises a stream except where a call returns a host value (documented per call).
 * The library never calls NCCL: the cross-GPU combine of the integer sums is the caller's
 * all_reduce (row a7).
 *
 * Citations: P:n = PAPER.md line n; DESIGN.md §2 is the arithmetic contract (both the CUDA path
 * and the independent oracle implement it).
 */
#ifndef MC_DESIGN_H
#define MC_DESIGN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MC_MAX_N 10   /* nested populations per problem (n; C5 sweeps n = 3..10) */

typedef enum {
    MC_OK = 0,
    MC_ERR_INVALID = 1,     /* a precondition or input invariant is violated (message says which) */
    MC_ERR_NUMERIC = 2,     /* singular Sigma0, non-PD prior, rank-deficient TPS system */
    MC_ERR_INFEASIBLE = 3,  /* fewer valid candidate designs than the requested N3 */
    MC_ERR_CUDA = 4,        /* a CUDA / cuSOLVER call failed */
    MC_ERR_OOM = 5          /* device allocation failed */
} mc_status;

typedef enum {
    MC_EST_COND = 0,  /* per-draw utility u = 1 - Phi_Sigma0(b) by one-sample separation of
                         variables in the order (even populations, then odd): n normal CDFs +
                         floor(n/2) inverse CDFs (readings R6, R21) */
    MC_EST_IND = 1    /* the paper's Formula 6/7 indicator with one independent null draw per sample
                         (reading R1) */
} mc_estimator;

/* One fixed-r design problem: nested fractions r, information units I3 (Eq. 9),
 * FWER budget alpha0 (Formula 2) and the effect prior f(Delta): model 0 = Gaussian (Formula 10 or a
 * general Cholesky factor), model 1 = the C4 strata prior (n = 2, see
 * mc_problem_strata).
 *   r[0] = 1 > r[1] > ... > r[n-1] > 0 with r[i+1]/r[i] <= 1 - 1e-6 (S:32 guard);
 *   0 < alpha0 < 0.5; i3 > 0.
 *   Prior: Delta ~ N(theta, Sigma_p).  has_prior_chol = 0: Sigma_p = diag(sigma) Sigma0 diag(sigma)
 *   (Formula 10; sigma_i >= 0, all zero = point mass).  has_prior_chol = 1: prior_chol holds the
 *   lower Cholesky factor L_p of a general Sigma_p, row-major with leading dimension MC_MAX_N
 *   (entry (i,j) at prior_chol[i*MC_MAX_N + j], j <= i). */
typedef struct {
    int32_t n;
    int32_t has_prior_chol;
    double  i3;
    double  alpha0;
    double  r[MC_MAX_N];
    double  theta[MC_MAX_N];
    double  sigma[MC_MAX_N];
    double  prior_chol[MC_MAX_N * MC_MAX_N];
    int32_t model;            /* 0 = Gaussian prior, 1 = C4 strata prior */
    int32_t reserved;
    double  strata[10];       /* model 1: (mean, sd) of logit prevalence, effect+, effect-, log variance
                                 inflation, logit dropout */
} mc_problem;

typedef struct mc_ctx mc_ctx;

/* ---- problem helpers (host, fp64) ------------------------------------------------------ */

/* Eq. 9: I3 = (Z_{1-alpha} + Z_{1-beta})^2 / log(1 - delta)^2.  Returns NaN on
 * invalid input (each argument must lie in (0,1)). */
double mc_information_units(double alpha, double beta, double delta);

/* Threshold Z_{1-alpha} in fp64; alpha = 0 -> +inf (never rejects); NaN if alpha is not in
 * [0, 1). */
double mc_threshold(double alpha);

/* Formula 10: fills *out with theta_i = -log(1 - delta0[i]),
 * sigma_i = 1/sqrt(80 r_i / 4), has_prior_chol = 0.  delta0[i] in (0,1).
 * MC_ERR_INVALID if r or delta0 violate their invariants. */
mc_status mc_problem_formula10(int32_t n, const double* r, const double* delta0, double i3,
                               double alpha0, mc_problem* out);

/* C4 strata prior (a synthetic extension of Formula 3 — not in the paper): n = 2,
 * r = (1, r2), 0 < r2 < 1; five independent normal components per draw with (mean, sd) pairs
 * strata[10] = (logit pi, delta+, delta-, log v, logit d).  Per draw: I_eff = I3 (1 - d)/v,
 * q+ = min(1, pi/r2), q- = max(0, (pi - r2)/(1 - r2)), Delta_2 = q+ delta+ + (1-q+) delta-,
 * Delta_neg = q- delta+ + (1-q-) delta-, Delta_1 = r2 Delta_2 + (1-r2) Delta_neg, mu_i = sqrt(r_i I_eff) Delta_i.
 * MC_ERR_INVALID if r2 or a standard deviation is out of range. */
mc_status mc_problem_strata(double r2, double i3, double alpha0, const double* strata, mc_problem* out);

/* ---- a1: candidate designs ------------------------------------- */

/* FWER (Formula 2) of `count` designs alpha_host[count*n] (row-major, alpha_i in [0, alpha0],
 * 0 => z = +inf) of one problem, fp64 on the GPU.  Writes fwer_host[count].  Synchronises. */
mc_status mc_fwer(const mc_problem* p, const double* alpha_host, int64_t count, double* fwer_host,
                  int32_t cuda_device);

/* alpha_n of explicit partial designs (Sec. 2.1 re-parametrisation; Formula 2): for each of
 * `count` rows of alpha_host[count*n] (row-major; alpha_1..alpha_{n-1} given, in [0, alpha0]) of problem
 * problem_host[count] (index into probs[n_probs], all sharing n), solves FWER(alpha_1..alpha_n) = alpha0 for
 * alpha_n in [0, alpha0] on the GPU (fp64) and writes it into the row; valid_host[count] =
 * 1 if feasible, 0 if FWER(.., 0) > alpha0 (row's alpha_n = NaN).  Host buffers; synchronises. */
mc_status mc_solve_alpha_n(const mc_problem* probs, int32_t n_probs, const int32_t* problem_host,
                           int64_t count, double* alpha_host, uint8_t* valid_host, int32_t cuda_device);

/* Candidate designs for n_probs problems sharing n: the half-offset m^(n-1) grid on
 * (0, alpha0)^(n-1) (first coordinate slowest), alpha_n solved from Formula 2 on the GPU (fp64,
 * one thread per grid point), infeasible points dropped; then, if 0 < n3 < #valid, the seeded
 * N3 subset (partial Fisher-Yates, key seed + problem index), in grid order.
 * Output: alpha_out[cap * n] row-major and problem_out[cap] (problem index, non-decreasing);
 * *n_out = total designs written.  MC_ERR_INFEASIBLE if a problem has fewer than n3 valid points
 * (n3 > 0); MC_ERR_INVALID if cap is too small (then *n_out is the capacity needed).
 * Host buffers; synchronises. */
mc_status mc_candidates(const mc_problem* probs, int32_t n_probs, int32_t m, int64_t n3,
                        uint64_t seed, double* alpha_out, int32_t* problem_out, int64_t cap,
                        int64_t* n_out, int32_t cuda_device);

/* ---- context ---------------------------------------------------------------------------- */

/* Copies the problems and the D designs (alpha_host[D*n], row-major; problem_of_design_host[D],
 * non-decreasing so each problem's designs are contiguous) into device tables on `cuda_device`:
 * per problem the fp32 factor M = diag(c) L_p (c_i = sqrt(r_i I3), Formula 3) and the Markov
 * coefficients rho_i, s_i of Sigma0 (Formula 1, A.1); per design zc_i = Z_{1-alpha_i} - c_i theta_i
 * (fp64 -> fp32, +inf for alpha_i = 0).  All problems must share n.  `seed` keys the Philox stream
 * (DESIGN.md §2.2).  Synchronises (uploads complete on return). */
mc_status mc_design_init(mc_ctx** ctx, const mc_problem* probs, int32_t n_probs,
                         const double* alpha_host, const int32_t* problem_of_design_host,
                         int64_t D, uint64_t seed, int32_t estimator, int32_t cuda_device);

/* Replaces the design table's alpha (same D, n and problem_of_design) from the HOST buffer
 * alpha_host[D*n] (pinned memory makes the copy asynchronous): H2D copy on `cuda_stream` and an fp64
 * device kernel recomputing zc.  Host-validated like mc_design_init.  The smoothing plan is kept iff
 * the new alpha equals the previous table (the TPS sites are unchanged), else it is invalidated. */
mc_status mc_design_upload(mc_ctx* ctx, const double* alpha_host, void* cuda_stream);

/* Sampling mode (NEXT f3): 0 = independent draws per design (stream keyed (design, sample), tag 0;
 * the default, reading R2); 1 = common random numbers per problem (stream keyed (problem, sample),
 * counter word 3 = 1): every design of a problem sees the same draws, so design differences have far
 * less noise and the draw's design-independent work is shared by blocks of designs (12 COND, 32 IND).
 * n <= 3. */
mc_status mc_set_sampling(mc_ctx* ctx, int32_t mode);

/* Launch shape of the fused kernel (results do not depend on it): threads per block (multiple of
 * 32 in [32, 256]; 0 = default 256) and grid blocks (>= 0; 0 = one 4096-sample warp tile per warp,
 * balanced by the hardware block scheduler; > 0 = a persistent grid of that many blocks striding over
 * the tiles); the same for the common-random-numbers kernel. */
mc_status mc_set_launch(mc_ctx* ctx, int32_t block_threads, int32_t grid_blocks);

void mc_destroy(mc_ctx* ctx);

/* ---- a2-a6: the fused Monte-Carlo kernel --------------------------------------------------- */

/* For designs [design_begin, design_begin + design_count) and samples
 * [sample_begin, sample_begin + sample_count) of each, draws Delta from the prior with the
 * (design, sample)-keyed Philox stream, evaluates the per-draw utility u and ACCUMULATES the exact
 * integer sums (sum round(2^23 u), sum round(2^23 u^2)) into sums_dev[D*2] (int64, caller zeroes;
 * entry 2d, 2d+1 for design d).  Integer accumulation makes the result bit-identical for every
 * split of the samples over calls, launch shapes and GPUs.  sample_begin +
 * sample_count must be < 2^40 (MC_ERR_INVALID otherwise), and the samples accumulated into one sums
 * buffer must total < 2^40 per design: S1, S2 <= samples x 2^23 must stay below 2^63.  Asynchronous. */
mc_status mc_evaluate_grid(mc_ctx* ctx, int64_t design_begin, int64_t design_count,
                           uint64_t sample_begin, uint64_t sample_count, void* cuda_stream,
                           int64_t* sums_dev);

/* NEXT f3 (ii): the paper-literal CROSSED estimator of Formula 7 (reading R1 alternative).
 * Per design d: N1 outer prior draws Delta^(k) (stream (d, tag 2), 2ceil(n/2) words per draw) crossed
 * with N2 inner null draws x^(l) (stream (d, tag 3), 2ceil(n/2) words per draw) — all N1 N2 pairs.
 * ACCUMULATES the exact integers S1 = sum_k c_k and S2 = sum_k c_k^2 into sums_dev[D*2], with
 * c_k = #{l : exists i x_i^(l) > b_i^(k)}.  The ctx must be built with MC_EST_IND and a Gaussian prior;
 * n <= 4; N2 < 2^32 and N1 N2^2 < 2^63 (S2 is an int64; MC_ERR_INVALID otherwise).  Asynchronous. */
mc_status mc_evaluate_crossed(mc_ctx* ctx, uint64_t n1, uint64_t n2, void* cuda_stream, int64_t* sums_dev);

/* Crossed finalize: mean_d = S1/(N1 N2); var_d = sample variance over k of c_k/N2 (the outer-draw
 * variance that governs the crossed estimator: SE = sqrt(var/N1)).  Asynchronous. */
mc_status mc_finalize_crossed(mc_ctx* ctx, const int64_t* sums_dev, uint64_t n1, uint64_t n2, double* mean_dev,
                              double* var_dev, void* cuda_stream);

/* ---- a8: finalize ----------------------------------------------------------------------- */

/* mean_d = S1/(N 2^23); var_d = (S2/(N 2^23) - mean_d^2) N/(N-1) (per-draw variance, A.2),
 * fp64, for all D designs; N = total_samples per design.  Asynchronous. */
mc_status mc_finalize(mc_ctx* ctx, const int64_t* sums_dev, uint64_t total_samples,
                      double* mean_dev, double* var_dev, void* cuda_stream);

/* ---- a9: smoothing (Sec. 2.3) -------------------------------------------------- */

/* Builds, once per design set, each problem's thin-plate-spline plan over x = alpha_{1..n-1}/alpha0
 * (d = n-1 <= 3): K, the QR complement Q2 of [1 x], the eigendecomposition Q2^T K Q2 = V Lambda V^T
 * (cuSOLVER Dsyevd, fp64) and E = Q2 V.  fit_mask_host[D] (NULL = all): designs with mask 0 are left
 * out of the fit and keep P~ = P^.  Problems with fewer than d + 2 fitted designs (or n = 1) are
 * passed through.  Synchronises.  Device memory ~ 8 N^2 bytes per problem of N fitted designs. */
mc_status mc_smooth_plan(mc_ctx* ctx, const uint8_t* fit_mask_host, void* cuda_stream);

/* P~ = P^ - N lambda w per problem.  lambda < 0: GCV over 10^(-12 + 0.25k),
 * k = 0..48 (first minimiser); lambda >= 0: fixed.  values_dev[D] -> smoothed_dev[D] (fp64);
 * lambda_used_dev[n_probs] (fp64, may be NULL).  Builds the plan first if needed.  Asynchronous
 * once the plan exists. */
mc_status mc_smooth(mc_ctx* ctx, const double* values_dev, double lambda, double* smoothed_dev,
                    double* lambda_used_dev, void* cuda_stream);

/* ---- NEXT f1: the continuous optimum on the smoothed surface ------------------ */

/* Fits (and caches in the ctx) every problem's TPS coefficients through values_dev[D] with lambda
 * (< 0: GCV, as mc_smooth): w on the GPU from the plan, beta on the host.  Synchronises. */
mc_status mc_tps_fit(mc_ctx* ctx, const double* values_dev, double lambda, void* cuda_stream);

/* Evaluates the cached TPS surface of `problem` at q points x_host[q*d] (x = alpha_{1..d}/alpha0,
 * d = n-1): f_host[q] and, if non-NULL, grad_host[q*d].  Host only. */
mc_status mc_tps_eval(const mc_ctx* ctx, int32_t problem, const double* x_host, int64_t q, double* f_host,
                      double* grad_host);

/* Per problem: maximises the TPS surface (mc_tps_fit with lambda) by box-constrained limited-memory
 * quasi-Newton (projected L-BFGS, memory 10) started from the fitted design with the largest P~ over
 * the box spanned by the fitted designs; re-solves alpha_n from Formula 2 (GPU, fp64).  Writes
 * alpha_out_host[n_probs*n], value_out_host[n_probs] (P~ at the optimum) and status_out_host[n_probs]:
 * 0 = ok, 1 = the optimum's alpha_n is infeasible (alpha_n = NaN), 2 = no surface (n = 1 or too few
 * designs: the best evaluated design is returned).  Synchronises. */
mc_status mc_refine(mc_ctx* ctx, const double* values_dev, double lambda, double* alpha_out_host,
                    double* value_out_host, int32_t* status_out_host, void* cuda_stream);

/* ---- NEXT f2: TPS over the r-lattice ---------------------------------------------- */

typedef struct mc_surface mc_surface;

/* Thin-plate spline (DESIGN.md §2.9 kernels, affine null space) through N points x_host[N*d]
 * (1 <= d <= 3, N >= d + 2) with values y_host[N]: P:234 fits "TPS of optimal power as functions of r".
 * lambda < 0: GCV over the §2.9 grid (influence-matrix trace); *lambda_used receives it.  Host fp64
 * dense solve.  MC_ERR_NUMERIC if the sites are degenerate. */
mc_status mc_surface_fit(const double* x_host, int64_t N, int32_t d, const double* y_host, double lambda,
                         mc_surface** out, double* lambda_used);
mc_status mc_surface_eval(const mc_surface* s, const double* x_host, int64_t q, double* f_host, double* grad_host);
/* Maximum over the sites' bounding box by the same projected L-BFGS as mc_refine, started from the
 * best site ("find optimal solution of r on the fitted TPS using the same procedure"). */
mc_status mc_surface_max(const mc_surface* s, double* x_out_host, double* f_out_host);
void mc_surface_destroy(mc_surface* s);

/* ---- a9 for dense regular grids (configuration C4, R23) ------- */

/* Separable Gaussian (Nadaraya-Watson) kernel smoother of a regular design grid:
 * smoothed_dev = S_r values_dev S_a^T, values_dev[nr*na] row-major (row i: coordinate xr_host[i], column j:
 * xa_host[j]; both strictly increasing, 2 <= nr, na <= 4096), S_x the row-normalised weights
 * exp(-(x_i - x_k)^2 / (2 h_x^2)).  hr, ha > 0: those bandwidths; otherwise both are chosen jointly by GCV
 * over h = 2^(j/2) x (mean grid step), j = -2..8 (first minimiser, r bandwidth outer).  h_used_host[2]
 * (may be NULL) receives (hr, ha).  fp64, device pointers in/out (in-place allowed), caller's stream;
 * synchronises (the GCV choice is made on the host).  MC_ERR_INVALID on bad sizes/coordinates. */
mc_status mc_grid_smooth(const double* values_dev, int32_t nr, int32_t na, const double* xr_host,
                         const double* xa_host, double hr, double ha, double* smoothed_dev, double* h_used_host,
                         void* cuda_stream);

/* ---- a10: argmax --------------------------------------------------------------- */

/* Per problem: the design with the largest value (lowest index on ties; NaN never wins) ->
 * idx_dev[n_probs] (int64, global design index), val_dev[n_probs].  If best_idx_host is non-NULL
 * also returns the overall argmax (and its value in *best_val_host) and synchronises. */
mc_status mc_argmax(mc_ctx* ctx, const double* values_dev, int64_t* idx_dev, double* val_dev,
                    int64_t* best_idx_host, double* best_val_host, void* cuda_stream);

/* ---- introspection / test hooks --------------------------------------------------------- */

int64_t mc_num_designs(const mc_ctx* ctx);
int32_t mc_num_problems(const mc_ctx* ctx);
/* Stream words per RECORD: COND records are sample pairs (2j, 2j+1) of U = 2p + 2 floor(n/2)
 * uniforms (p shared Box-Muller pairs, then each sample's SOV uniforms), IND records single samples of
 * U = 2 ceil((p+n)/2) uniforms; the U 23-bit uniforms are packed into 2 ceil(23 U / 64) words.  -1 for a
 * null ctx. */
int32_t mc_words_per_record(const mc_ctx* ctx);

/* K3 (test hook): Philox words exactly as the kernels generate them.  out_dev[i] = word word_dev[i] of
 * the stream (id_dev[i], tag) for `seed` (lane w mod 4 of the block with counter
 * (q_lo, q_hi, id, tag), q = w / 4).  tag: 0 independent draws (id = design), 1 common random numbers
 * (id = problem), 2 / 3 the crossed estimator's outer / inner streams.  form: 0 the fused and CRN kernels'
 * steady-state block (round 1 hoisted, constant-bank round keys), 1 the fused kernel's masked-path block
 * (tag 0 only), 2 the plain ten-round block of the crossed kernel.  count entries; MC_ERR_INVALID for a
 * bad form.  Asynchronous. */
mc_status mc_philox_dump(uint64_t seed, uint32_t tag, int32_t form, const uint32_t* id_dev, const uint64_t* word_dev,
                         int64_t count, uint32_t* out_dev, void* cuda_stream);

/* Per-draw record of (design_dev[i], sample_dev[i]) computed by the same device code as the fused
 * kernel (the steady-state Philox form; COND: the packed two-sample record code of K1):
 * out_dev[i*stride ...] = normals (p prior, then n null for IND), b[n], u; stride = p + 2n + 1
 * (IND) or p + n + 1 (COND), fp32.  Asynchronous. */
mc_status mc_draw_dump(mc_ctx* ctx, const int64_t* design_dev, const uint64_t* sample_dev,
                       int64_t count, float* out_dev, void* cuda_stream);
int32_t mc_draw_dump_stride(const mc_ctx* ctx);

/* Number of CUDA kernel launches issued by this ctx's calls since creation (bench gpu_launches). */
int64_t mc_kernel_launches(const mc_ctx* ctx);

const char* mc_last_error(void);
const char* mc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MC_DESIGN_H */
