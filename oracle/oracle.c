/*
 * oracle.c — the CPU ORACLE for arXiv 2005.10494's Monte-Carlo design objective.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2005_10494_b200/,
 * include/, the CUDA library) may include, link or call this file.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg use it.
 * It shares no code, header, table or constant generator with the CUDA path.
 *
 * Plain, single-threaded, fp64, written to be checked against PAPER.md by eye.
 * Citations: P:n = /root/reference/PAPER.md line n (not available at run time;
 * the citations are for the reader).  Readings of the paper are listed in DESIGN.md §3.
 *
 * What it computes, step by step (DESIGN.md §2 gives the contract both sides follow):
 *   Formula 1 (A.1 P:417-424)  Sigma0[k][l] = sqrt(r_l/r_k), k<l
 *   Formula 10              Delta ~ N(theta, Sigma_p), Sigma_p = diag(sigma) Sigma0 diag(sigma)
 *   Formula 3                 X | Delta ~ N(c*Delta, Sigma0), c_i = sqrt(r_i I3)
 *   Formula 4/5   P(alpha) = 1 - E_Delta[ Phi_Sigma0(z - c*Delta) ]
 *   Formula 6/7             inner indicator  1[ exists i: X_i > z_i - c_i Delta_i ]  (IND)
 *   Genz separation of variables        one-sample unbiased estimate of Phi_Sigma0 (COND; reading R6)
 *   Formula 2                 FWER = 1 - Phi_Sigma0(z_1..z_n)
 *   Sec. 2.3                    m^(n-1) alpha grid, alpha_n solved, N3 random valid points
 *
 * Parity unpinned: none (every function has a pin in tests/test_oracle_*.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAXN 10

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy
 * as 1, 2, 3", SC'11).  Pinned by the Random123 known-answer vectors in
 * tests/golden/philox4x32_10_kat.txt.  Reading R9: the paper's
 * Algorithms 1-2 are missing images, so the generator is ours.   */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Word w of design d's stream: block q = w/4 with counter
 * (q_lo, q_hi, d, 0) and key (seed_lo, seed_hi); the word is lane w mod 4.   */
uint32_t or_word_tagged(uint64_t seed, uint32_t id, uint32_t tag, uint64_t w)
{
    uint64_t q = w / 4;
    uint32_t ctr[4] = { (uint32_t)q, (uint32_t)(q >> 32), id, tag };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t out[4];
    or_philox4x32_10(ctr, key, out);
    return out[w % 4];
}

/* Stream tags: tag 0 = independent draws per design (id = design index), tag 1 = common
 * random numbers per problem (id = problem index; NEXT f3).  The draw functions below take (id, tag). */
uint32_t or_word(uint64_t seed, uint32_t design, uint64_t w)
{
    uint64_t q = w / 4;
    uint32_t ctr[4] = { (uint32_t)q, (uint32_t)(q >> 32), design, 0u };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t out[4];
    or_philox4x32_10(ctr, key, out);
    return out[w % 4];
}

/* Uniforms from a 23-bit field k.                          */
static double u_radius(uint32_t k) { return 1.0 - (double)k / 8388608.0; }   /* (0,1] */
static double u_angle(uint32_t k)  { return (double)k / 8388608.0; }         /* [0,1) */
static double u_open(uint32_t k)   { return ((double)k + 0.5) / 8388608.0; } /* (0,1) */

/* Records (round 2): a record of U uniforms starts at word w0.  If 2 ceil(23 U / 64) < U
 * (U >= 8) the record is PACKED into W = 2 ceil(23 U / 64) words and uniform i is the 23-bit field at bit
 * offset 23 i of the record's bit string, in which bit b is bit (b mod 32) of word w0 + floor(b / 32);
 * otherwise W = U and uniform i is the low 23 bits of word w0 + i.                                      */
static int record_packed(int uniforms) { return 2 * ((23 * uniforms + 63) / 64) < uniforms; }

static uint32_t record_field(uint64_t seed, uint32_t id, uint32_t tag, uint64_t w0, int U, int i)
{
    if (!record_packed(U)) return or_word_tagged(seed, id, tag, w0 + (uint64_t)i) & 0x7FFFFFu;
    const uint64_t bit = 23u * (uint64_t)i;
    const uint64_t j = bit / 32;
    const int sh = (int)(bit % 32);
    uint64_t v = or_word_tagged(seed, id, tag, w0 + j);
    if (sh + 23 > 32) v |= (uint64_t)or_word_tagged(seed, id, tag, w0 + j + 1) << 32;
    return (uint32_t)((v >> sh) & 0x7FFFFFu);
}

int or_record_words(int uniforms) { return record_packed(uniforms) ? 2 * ((23 * uniforms + 63) / 64) : uniforms; }

uint32_t or_record_field(uint64_t seed, uint32_t id, uint32_t tag, uint64_t w0, int uniforms, int i)
{
    return record_field(seed, id, tag, w0, uniforms, i);
}

/* ------------------------------------------------------------------------- */
/* Standard normal CDF and quantile.                                          */
double or_Phi(double x) { return 0.5 * erfc(-x / sqrt(2.0)); }

/* Wichura, "Algorithm AS 241: The percentage points of the normal
 * distribution", Applied Statistics 37 (1988) 477-484 (PPND16).  Pinned
 * against scipy.special.ndtri in tests/test_oracle_math.py.                  */
double or_Phi_inv(double p)
{
    if (p <= 0.0) return -INFINITY;
    if (p >= 1.0) return INFINITY;
    double q = p - 0.5, r, val;
    if (fabs(q) <= 0.425) {
        r = 0.180625 - q * q;
        val = q * (((((((2.5090809287301226727e+3 * r + 3.3430575583588128105e+4) * r
                        + 6.7265770927008700853e+4) * r + 4.5921953931549871457e+4) * r
                        + 1.3731693765509461125e+4) * r + 1.9715909503065514427e+3) * r
                        + 1.3314166789178437745e+2) * r + 3.3871328727963666080e+0)
                / (((((((5.2264952788528545610e+3 * r + 2.8729085735721942674e+4) * r
                        + 3.9307895800092710610e+4) * r + 2.1213794301586595867e+4) * r
                        + 5.3941960214247511077e+3) * r + 6.8718700749205790830e+2) * r
                        + 4.2313330701600911252e+1) * r + 1.0);
        return val;
    }
    r = (q < 0.0) ? p : 1.0 - p;
    r = sqrt(-log(r));
    if (r <= 5.0) {
        r -= 1.6;
        val = (((((((7.74545014278341407640e-4 * r + 2.27238449892691845833e-2) * r
                    + 2.41780725177450611770e-1) * r + 1.27045825245236838258e+0) * r
                    + 3.64784832476320460504e+0) * r + 5.76949722146069140550e+0) * r
                    + 4.63033784615654529590e+0) * r + 1.42343711074968357734e+0)
            / (((((((1.05075007164441684324e-9 * r + 5.47593808499534494600e-4) * r
                    + 1.51986665636164571966e-2) * r + 1.48103976427480074590e-1) * r
                    + 6.89767334985100004550e-1) * r + 1.67638483018380384940e+0) * r
                    + 2.05319162663775882187e+0) * r + 1.0);
    } else {
        r -= 5.0;
        val = (((((((2.01033439929228813265e-7 * r + 2.71155556874348757815e-5) * r
                    + 1.24266094738807843860e-3) * r + 2.65321895265761230930e-2) * r
                    + 2.96560571828504891230e-1) * r + 1.78482653991729133580e+0) * r
                    + 5.46378491116411436990e+0) * r + 6.65790464350110377720e+0)
            / (((((((2.04426310338993978564e-15 * r + 1.42151175831644588870e-7) * r
                    + 1.84631831751005468180e-5) * r + 7.86869131145613259100e-4) * r
                    + 1.48753612908506148525e-2) * r + 1.36929880922735805310e-1) * r
                    + 5.99832206555887937690e-1) * r + 1.0);
    }
    return (q < 0.0) ? -val : val;
}

/* Threshold Z_{1-alpha}; alpha = 0 means "test never rejects" -> +inf (reading R13). */
double or_threshold(double alpha)
{
    if (alpha <= 0.0) return INFINITY;
    return or_Phi_inv(1.0 - alpha);
}

/* ------------------------------------------------------------------------- */
/* Dense linear algebra: textbook Cholesky A = L L^T (row-major n x n).
 * Returns 0 on success, (k+1) if the k-th pivot is not positive.            */
int or_cholesky(int n, const double *A, double *L)
{
    memset(L, 0, sizeof(double) * n * n);
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j <= i; ++j) {
            double s = A[i * n + j];
            for (int k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
            if (i == j) {
                if (!(s > 0.0)) return i + 1;
                L[i * n + i] = sqrt(s);
            } else {
                L[i * n + j] = s / L[j * n + j];
            }
        }
    }
    return 0;
}

/* Formula 1 / Appendix A.1: Sigma0[k][l] = sqrt(r_l / r_k) for k <= l (r_1 = 1). */
void or_null_corr(int n, const double *r, double *S)
{
    for (int k = 0; k < n; ++k)
        for (int l = 0; l < n; ++l) {
            int a = k < l ? k : l, b = k < l ? l : k;
            S[k * n + l] = sqrt(r[b] / r[a]);
        }
}

/* ------------------------------------------------------------------------- */
/* One draw (design d, sample s) of the per-draw utility.
 *   n, p   populations, prior dimensions (p = n for the Formula-10 prior)
 *   r[n]   subpopulation fractions; i3 information units
 *   theta[p], Lp[p*p] prior mean and lower Cholesky factor (row-major) of Sigma_p
 *   z[n]   thresholds Z_{1-alpha_i} (+inf allowed)
 *   est    0 = COND (Genz SOV), 1 = IND (Formula 6/7 indicator)
 * Outputs (may be NULL): eps[p] prior normals, delta[n], b[n], w_null[n] (IND) .
 * Returns u in [0,1]: the success probability (COND) or indicator (IND).    */
/* Uniforms per record (records are sample pairs (2j, 2j+1)): COND shares p Box-Muller pairs (2p uniforms)
 * between the two samples, followed by each sample's n/2 SOV uniforms; IND gives each sample its own
 * ceil((p+n)/2) pairs, sample 2j's first.                                                            */
int or_record_uniforms(int n, int p, int est)
{
    if (est == 0) return 2 * p + 2 * (n / 2);
    return 4 * ((p + n + 1) / 2);
}

/* Box-Muller: pair j uses record uniforms 2(j0 + j) (radius) and 2(j0 + j) + 1 (angle) of
 * the U-uniform record starting at word w0. */
static void bm_normals_rec(uint64_t seed, uint32_t design, uint32_t tag, uint64_t w0, int U, int j0, int nnorm,
                           double *normals)
{
    for (int j = 0; 2 * j < nnorm; ++j) {
        double R = sqrt(-2.0 * log(u_radius(record_field(seed, design, tag, w0, U, 2 * (j0 + j)))));
        double a = 2.0 * M_PI * u_angle(record_field(seed, design, tag, w0, U, 2 * (j0 + j) + 1));
        normals[2 * j] = R * cos(a);
        normals[2 * j + 1] = R * sin(a);
    }
}

/* The crossed estimator's streams (tags 2, 3) keep one uniform per word: pair j uses words w0 + 2j and
 * w0 + 2j + 1, the 23-bit field being the word's low 23 bits.                                        */
static void bm_normals(uint64_t seed, uint32_t design, uint32_t tag, uint64_t w0, int nnorm, double *normals)
{
    for (int j = 0; 2 * j < nnorm; ++j) {
        double R = sqrt(-2.0 * log(u_radius(or_word_tagged(seed, design, tag, w0 + 2 * j) & 0x7FFFFFu)));
        double a = 2.0 * M_PI * u_angle(or_word_tagged(seed, design, tag, w0 + 2 * j + 1) & 0x7FFFFFu);
        normals[2 * j] = R * cos(a);
        normals[2 * j + 1] = R * sin(a);
    }
}

/* The normals of sample s; writes the record's first word and the record index of the sample's first
 * SOV uniform.
 * Samples come in records of two, (2j, 2j+1), record j starting at word j W (W = or_record_words(U)).
 * COND (U = 2p + 2(n/2)): uniforms [0, 2p) are p Box-Muller pairs giving 2p normals, sample 2j takes
 * normals [0, p) and sample 2j+1 normals [p, 2p); then sample 2j's n/2 SOV uniforms, then sample 2j+1's.
 * IND (U = 4 ceil((p+n)/2)): sample 2j + h takes pairs [h c, (h+1) c), c = ceil((p+n)/2): p prior normals
 * then n null normals.                                                                               */
static void sample_normals(int n, int p, int est, uint64_t seed, uint32_t design, uint32_t tag, uint64_t s,
                           double *normals, uint64_t *rec_w0, int *sov_u0)
{
    const int U = or_record_uniforms(n, p, est);
    const uint64_t W = (uint64_t)or_record_words(U);
    *rec_w0 = (s / 2) * W;
    const int h = (int)(s % 2);
    if (est == 1) {
        bm_normals_rec(seed, design, tag, *rec_w0, U, h * ((p + n + 1) / 2), p + n, normals);
        *sov_u0 = U;
        return;
    }
    double rec[4 * OR_MAXN + 4];
    bm_normals_rec(seed, design, tag, *rec_w0, U, 0, 2 * p, rec);
    for (int k = 0; k < p; ++k) normals[k] = rec[h * p + k];
    *sov_u0 = 2 * p + h * (n / 2);
}

/* Utility of one draw given the thresholds b of Phi_Sigma0 (Formulas 4-7):
 * IND uses the null normals w[0..n); COND reads its SOV uniforms at record uniforms u0 + a of the
 * rec_u-uniform record starting at word rw0. */
static double utility_from_b(int n, const double *r, const double *b, const double *w, int est,
                             uint64_t seed, uint32_t design, uint32_t tag, uint64_t rw0, int rec_u, int u0,
                             double *wnull_out)
{
    double S0[OR_MAXN * OR_MAXN], L0[OR_MAXN * OR_MAXN];
    or_null_corr(n, r, S0);
    if (or_cholesky(n, S0, L0) != 0) return NAN;

    if (est == 1) {
        /* Formula 6/7 with one independent null draw per sample (reading R1):
         * x = L0 W ~ N(0, Sigma0); success iff some X_i exceeds its threshold.   */
        int reject = 0;
        for (int i = 0; i < n; ++i) {
            double x = 0.0;
            for (int k = 0; k <= i; ++k) x += L0[i * n + k] * w[k];
            if (wnull_out) wnull_out[i] = x;
            if (x > b[i]) reject = 1;
        }
        return reject ? 1.0 : 0.0;
    }
    /* COND: Genz separation of variables (SOV) for Phi_Sigma0(b) in the variable order
     * pi = (populations 2, 4, 6, ..., then 1, 3, 5, ...).  With the permuted
     * correlation S' = Sigma0[pi][pi] = L' L'^T, Y iid N(0,1), X_pi = L' Y:
     *   e_a = P(X_pi(a) <= b_pi(a) | y_1..y_{a-1}) = Phi((b_pi(a) - sum_{j<a} L'_aj y_j) / L'_aa),
     *   y_a = Phi^{-1}(v_a e_a),  and prod_a e_a is an unbiased estimate of Phi_Sigma0(b).
     * Only the first n/2 (even-population) stages draw a uniform v_a: A.1 makes X a Markov chain,
     * so every odd population is independent of the other odd ones given the even ones, i.e.
     * L'_aj = 0 for j >= n/2 (checked below) and those y_j are never used.               */
    const int neven = n / 2;
    int ord[OR_MAXN], k = 0;
    for (int i = 1; i < n; i += 2) ord[k++] = i;     /* 0-based index of population 2, 4, ... */
    for (int i = 0; i < n; i += 2) ord[k++] = i;     /* populations 1, 3, ... */
    double Sp[OR_MAXN * OR_MAXN], Lq[OR_MAXN * OR_MAXN];
    for (int a = 0; a < n; ++a)
        for (int c = 0; c < n; ++c) Sp[a * n + c] = S0[ord[a] * n + ord[c]];
    if (or_cholesky(n, Sp, Lq) != 0) return NAN;
    double y[OR_MAXN], prod = 1.0;
    for (int a = 0; a < n; ++a) {
        double m = 0.0;
        for (int j = 0; j < a; ++j) {
            if (j >= neven) {
                if (fabs(Lq[a * n + j]) > 1e-12) return NAN;   /* the Markov zero of A.1 */
                continue;
            }
            m += Lq[a * n + j] * y[j];
        }
        double e = or_Phi((b[ord[a]] - m) / Lq[a * n + a]);
        prod *= e;
        if (prod == 0.0) break;                        /* u = 1 exactly; later stages are irrelevant */
        if (a < neven) {
            double v = u_open(record_field(seed, design, tag, rw0, rec_u, u0 + a));
            y[a] = or_Phi_inv(v * e);
        }
    }
    return 1.0 - prod;
}


double or_draw(int n, int p, const double *r, double i3, const double *theta, const double *Lp,
               const double *z, int est, uint64_t seed, uint32_t design, uint32_t tag, uint64_t s,
               double *eps_out, double *delta_out, double *b_out, double *wnull_out)
{
    double normals[2 * OR_MAXN + 2];
    uint64_t rw0;
    int u0;
    sample_normals(n, p, est, seed, design, tag, s, normals, &rw0, &u0);
    /* Formula 10: Delta = theta + Lp * eps. */
    double delta[OR_MAXN], b[OR_MAXN];
    for (int i = 0; i < n; ++i) {
        double acc = theta[i];
        for (int k = 0; k <= i && k < p; ++k) acc += Lp[i * p + k] * normals[k];
        delta[i] = acc;
    }
    /* Formulas 3-5: thresholds of Phi_Sigma0 are z_i - sqrt(r_i I3) Delta_i. */
    for (int i = 0; i < n; ++i) b[i] = z[i] - sqrt(r[i] * i3) * delta[i];
    if (eps_out) for (int k = 0; k < p; ++k) eps_out[k] = normals[k];
    if (delta_out) for (int i = 0; i < n; ++i) delta_out[i] = delta[i];
    if (b_out) for (int i = 0; i < n; ++i) b_out[i] = b[i];
    return utility_from_b(n, r, b, normals + p, est, seed, design, tag, rw0, or_record_uniforms(n, p, est), u0,
                          wnull_out);
}

/* C4 strata prior (a synthetic extension inside the Formula-3 model, not in the paper).
 * n = 2 (overall population and a biomarker-positive subset of fraction r2), five independent normal
 * components per draw, sp[10] = (mean, sd) of: logit prevalence pi, effect in responders delta+,
 * effect in non-responders delta-, log variance inflation v, logit dropout d.
 *   I_eff = I3 (1 - d) / v;  responders are the top-pi biomarker fraction:
 *   q+ = min(1, pi / r2), q- = max(0, (pi - r2) / (1 - r2));
 *   Delta_2 = q+ delta+ + (1 - q+) delta-,  Delta_neg = q- delta+ + (1 - q-) delta-,
 *   Delta_1 = r2 Delta_2 + (1 - r2) Delta_neg;  mu_i = sqrt(r_i I_eff) Delta_i;  b = z - mu.      */
double or_draw_strata(double r2, double i3, const double *sp, const double *z, int est, uint64_t seed,
                      uint32_t design, uint32_t tag, uint64_t s, double *eps_out, double *delta_out, double *b_out,
                      double *wnull_out)
{
    const int n = 2, p = 5;
    const double r[2] = { 1.0, r2 };
    double normals[2 * OR_MAXN + 2];
    uint64_t rw0;
    int u0;
    sample_normals(n, p, est, seed, design, tag, s, normals, &rw0, &u0);
    const double pi = 1.0 / (1.0 + exp(-(sp[0] + sp[1] * normals[0])));
    const double dp = sp[2] + sp[3] * normals[1];
    const double dm = sp[4] + sp[5] * normals[2];
    const double v = exp(sp[6] + sp[7] * normals[3]);
    const double d = 1.0 / (1.0 + exp(-(sp[8] + sp[9] * normals[4])));
    const double ieff = i3 * (1.0 - d) / v;
    const double qp = fmin(1.0, pi / r2);
    const double qm = fmax(0.0, (pi - r2) / (1.0 - r2));
    const double d2 = qp * dp + (1.0 - qp) * dm;
    const double dneg = qm * dp + (1.0 - qm) * dm;
    const double d1 = r2 * d2 + (1.0 - r2) * dneg;
    double b[2];
    b[0] = z[0] - sqrt(r[0] * ieff) * d1;
    b[1] = z[1] - sqrt(r[1] * ieff) * d2;
    if (eps_out) for (int k = 0; k < p; ++k) eps_out[k] = normals[k];
    if (delta_out) { delta_out[0] = d1; delta_out[1] = d2; }
    if (b_out) { b_out[0] = b[0]; b_out[1] = b[1]; }
    return utility_from_b(n, r, b, normals + p, est, seed, design, tag, rw0, or_record_uniforms(n, p, est), u0,
                          wnull_out);
}

void or_design_sums_strata(double r2, double i3, const double *sp, const double *z, int est, uint64_t seed,
                           uint32_t design, uint32_t tag, uint64_t s0, uint64_t count, int64_t *sums)
{
    int64_t a1 = 0, a2 = 0;
    for (uint64_t s = s0; s < s0 + count; ++s) {
        double u = or_draw_strata(r2, i3, sp, z, est, seed, design, tag, s, NULL, NULL, NULL, NULL);
        a1 += (int64_t)nearbyint(ldexp(u, 23));
        a2 += (int64_t)nearbyint(ldexp(u * u, 23));
    }
    sums[0] += a1;
    sums[1] += a2;
}

/* Per-design sums over samples [s0, s0+count): each draw's u
 * and u^2 are rounded (half-to-even) to the 2^-23 grid and added as integers.  */
void or_design_sums(int n, int p, const double *r, double i3, const double *theta, const double *Lp,
                    const double *z, int est, uint64_t seed, uint32_t design, uint32_t tag,
                    uint64_t s0, uint64_t count, int64_t *sums)
{
    int64_t a1 = 0, a2 = 0;
    for (uint64_t s = s0; s < s0 + count; ++s) {
        double u = or_draw(n, p, r, i3, theta, Lp, z, est, seed, design, tag, s, NULL, NULL, NULL, NULL);
        a1 += (int64_t)nearbyint(ldexp(u, 23));
        a2 += (int64_t)nearbyint(ldexp(u * u, 23));
    }
    sums[0] += a1;
    sums[1] += a2;
}

/* ------------------------------------------------------------------------- */
/* Gauss-Legendre rule on [-1,1]: nodes and weights are SUPPLIED by the caller
 * (oracle.py passes numpy.polynomial.legendre.leggauss(20), a library routine),
 * so this file computes no quadrature rule of its own.                       */
enum { OR_GL_MAX = 64 };
static int or_gl_n = 0;
static double or_gl_x[OR_GL_MAX], or_gl_w[OR_GL_MAX];

int or_set_gauss_legendre(int G, const double *x, const double *w)
{
    if (G < 2 || G > OR_GL_MAX) return 1;
    for (int i = 0; i < G; ++i) { or_gl_x[i] = x[i]; or_gl_w[i] = w[i]; }
    or_gl_n = G;
    return 0;
}

/* Composite Gauss-Legendre nodes on [a, b] with panels no wider than h.
 * Returns the node count, or -1 if the nodes would not fit in cap.           */
static int panel_nodes(double a, double b, double h, double *xs, double *ws, int cap)
{
    const int G = or_gl_n;
    if (!(b > a)) return 0;
    int P = (int)ceil((b - a) / h);
    if ((long)P * G > cap) return -1;
    double len = (b - a) / P;
    int m = 0;
    for (int k = 0; k < P; ++k) {
        double lo = a + k * len;
        for (int g = 0; g < G; ++g) {
            xs[m] = lo + 0.5 * len * (or_gl_x[g] + 1.0);
            ws[m] = 0.5 * len * or_gl_w[g];
            ++m;
        }
    }
    return m;
}

static double phi_pdf(double x) { return exp(-0.5 * x * x) / sqrt(2.0 * M_PI); }

/* Phi_Sigma0(b) = P(X_i <= b_i, i = 1..n) for the Formula-1 correlation.
 * Appendix A.1 makes corr(X_k, X_l) = sqrt(r_l/r_k) = prod_{j=k}^{l-1} rho_j with
 * rho_j = sqrt(r_{j+1}/r_j): X is a Gaussian Markov chain X_{j+1} = rho_j X_j + s_j W,
 * s_j = sqrt(1 - rho_j^2).  The orthant is the chain's iterated integral
 *   Phi = int_{-inf}^{b_1} phi(x_1) h_1(x_1) dx_1,
 *   h_k(x) = int_{-inf}^{b_{k+1}} phi((y - rho_k x)/s_k)/s_k h_{k+1}(y) dy,
 *   h_{n-1}(x) = Phi((b_n - rho_{n-1} x)/s_{n-1}),
 * evaluated with composite Gauss-Legendre (the supplied G-point rule) on [-10, min(b_k, 10)]
 * (mass outside < 1e-23) with panels no wider than the narrowest conditional sd s_j.
 * Returns NAN if no rule was supplied or a level would need more than CAP nodes.
 * (Level storage is allocated per call: the oracle is single-threaded per process.)      */
double or_mvn_orthant(int n, const double *r, const double *b)
{
    if (n == 1) return or_Phi(b[0]);
    if (or_gl_n == 0) return NAN;
    double rho[OR_MAXN], sd[OR_MAXN], smin = 1.0;
    for (int k = 0; k + 1 < n; ++k) {
        rho[k] = sqrt(r[k + 1] / r[k]);
        sd[k] = sqrt(1.0 - r[k + 1] / r[k]);
        if (sd[k] < smin) smin = sd[k];
    }
    const double LO = -10.0, HI = 10.0;
    double h = smin;
    enum { CAP = 1000000 };
    const int need = or_gl_n * (int)ceil((HI - LO) / h);
    if (need > CAP) return NAN;
    double *xs[OR_MAXN], *ws[OR_MAXN], *hv[OR_MAXN];
    double *buf = (double *)malloc(sizeof(double) * 3 * (size_t)need * (n - 1));
    if (!buf) return NAN;
    int m[OR_MAXN] = { 0 };
    for (int k = 0; k + 1 < n; ++k) {
        xs[k] = buf + (size_t)need * (3 * k);
        ws[k] = xs[k] + need;
        hv[k] = ws[k] + need;
        double up = b[k] < HI ? b[k] : HI;
        if (up <= LO) { free(buf); return 0.0; }
        m[k] = panel_nodes(LO, up, h, xs[k], ws[k], need);
    }
    /* level n-1 (0-based n-2): closed-form last conditional */
    int L = n - 2;
    for (int j = 0; j < m[L]; ++j)
        hv[L][j] = isinf(b[n - 1]) ? 1.0 : or_Phi((b[n - 1] - rho[L] * xs[L][j]) / sd[L]);
    for (int k = L - 1; k >= 0; --k) {
        for (int i = 0; i < m[k]; ++i) {
            double acc = 0.0;
            for (int j = 0; j < m[k + 1]; ++j)
                acc += ws[k + 1][j] * phi_pdf((xs[k + 1][j] - rho[k] * xs[k][i]) / sd[k]) / sd[k] * hv[k + 1][j];
            hv[k][i] = acc;
        }
    }
    double acc = 0.0;
    for (int j = 0; j < m[0]; ++j) acc += ws[0][j] * phi_pdf(xs[0][j]) * hv[0][j];
    free(buf);
    return acc;
}

/* Formula 2: FWER(alpha) = 1 - Phi_Sigma0(Z_{1-alpha_1}, ..., Z_{1-alpha_n}). */
double or_fwer(int n, const double *r, const double *alpha)
{
    double z[OR_MAXN];
    for (int i = 0; i < n; ++i) z[i] = or_threshold(alpha[i]);
    return 1.0 - or_mvn_orthant(n, r, z);
}

/* Sec. 2.1 re-parametrisation: solve FWER(alpha_1..alpha_{n-1}, a) = alpha0 for
 * a in [0, alpha0] by bisection (FWER is increasing in a).  Returns 1 and writes *an
 * when feasible; 0 when FWER(.., 0) > alpha0 (reading R12: the point is invalid);
 * -1 when the orthant quadrature is unavailable (or_mvn_orthant returned NAN).          */
int or_solve_alpha_n(int n, const double *r, double alpha0, const double *partial, double tol, double *an)
{
    double a[OR_MAXN];
    for (int i = 0; i + 1 < n; ++i) a[i] = partial[i];
    if (n == 1) { *an = alpha0; return 1; }
    a[n - 1] = 0.0;
    /* FWER(.., 0) decides feasibility up to quadrature rounding: |err| < 1e-12 (R12). */
    double f0 = or_fwer(n, r, a) - alpha0;
    if (isnan(f0)) return -1;                      /* quadrature unavailable / under-resolved */
    if (f0 > 1e-12) return 0;
    if (f0 >= -1e-12) { *an = 0.0; return 1; }
    double lo = 0.0, hi = alpha0;
    while (hi - lo > tol) {
        double mid = 0.5 * (lo + hi);
        a[n - 1] = mid;
        if (or_fwer(n, r, a) - alpha0 > 0.0) hi = mid; else lo = mid;
    }
    *an = 0.5 * (lo + hi);
    return 1;
}

/* Sec. 2.3: the m^(n-1) half-offset grid alpha_j = (k_j + 1/2) alpha0 / m on
 * (0, alpha0)^(n-1) (reading R8/R10), first coordinate slowest.  Writes every grid
 * point's feasibility flag and solved alpha_n.  Returns the number of grid points, or -1
 * if the orthant quadrature is unavailable for r.                                      */
int64_t or_alpha_grid(int n, const double *r, double alpha0, int m, double tol,
                      double *alpha_out /* [m^(n-1) * n] */, uint8_t *valid_out)
{
    int64_t G = 1;
    for (int i = 0; i + 1 < n; ++i) G *= m;
    for (int64_t g = 0; g < G; ++g) {
        double part[OR_MAXN];
        int64_t rem = g;
        for (int i = n - 2; i >= 0; --i) { part[i] = ((double)(rem % m) + 0.5) * alpha0 / m; rem /= m; }
        double an = 0.0;
        int ok = or_solve_alpha_n(n, r, alpha0, part, tol, &an);
        if (ok < 0) return -1;                         /* quadrature unavailable */
        for (int i = 0; i + 1 < n; ++i) alpha_out[g * n + i] = part[i];
        alpha_out[g * n + n - 1] = ok ? an : NAN;
        valid_out[g] = (uint8_t)ok;
    }
    return G;
}

/* Seeded N3-subset of V valid points (reading R11): partial Fisher-Yates over
 * idx = [0, V) with word i of the Philox stream key (seed_lo ^ 0x00C0FFEE, seed_hi),
 * counter (i/4, 0, 0, 0xC0FFEE): j = i + floor(word * (V - i) / 2^32).  The chosen
 * indices are returned in ascending order.                                    */
static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

void or_subset(int64_t V, int64_t n3, uint64_t seed, int64_t *out)
{
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (V > 0 ? V : 1));
    for (int64_t i = 0; i < V; ++i) idx[i] = i;
    uint32_t key[2] = { (uint32_t)seed ^ 0x00C0FFEEu, (uint32_t)(seed >> 32) };
    for (int64_t i = 0; i < n3; ++i) {
        uint32_t ctr[4] = { (uint32_t)(i / 4), (uint32_t)((uint64_t)i >> 34), 0u, 0x00C0FFEEu };
        uint32_t o[4];
        or_philox4x32_10(ctr, key, o);
        uint64_t word = o[i % 4];
        int64_t j = i + (int64_t)((word * (uint64_t)(V - i)) >> 32);
        int64_t t = idx[i]; idx[i] = idx[j]; idx[j] = t;
    }
    for (int64_t i = 0; i < n3; ++i) out[i] = idx[i];
    qsort(out, (size_t)n3, sizeof(int64_t), cmp_i64);
    free(idx);
}

/* NEXT f3 (ii): Formula 7 literally: every outer prior draw Delta^(k) (stream (design, tag 2),
 * 2ceil(p/2) words per draw) paired with every inner null draw x^(l) (stream (design, tag 3),
 * 2ceil(n/2) words per draw).  sums += (sum_k c_k, sum_k c_k^2), c_k = #{l : exists i x_i^(l) > b_i^(k)}. */
void or_design_sums_crossed(int n, const double *r, double i3, const double *theta, const double *Lp,
                            const double *z, uint64_t seed, uint32_t design, uint64_t n1, uint64_t n2, int64_t *sums)
{
    const int p = n, uo = 2 * ((p + 1) / 2), ui = 2 * ((n + 1) / 2);
    double S0[OR_MAXN * OR_MAXN], L0[OR_MAXN * OR_MAXN];
    or_null_corr(n, r, S0);
    if (or_cholesky(n, S0, L0) != 0) return;
    double *X = (double *)malloc(sizeof(double) * (size_t)(n2 > 0 ? n2 : 1) * n);
    for (uint64_t l = 0; l < n2; ++l) {
        double w[2 * OR_MAXN + 2];
        bm_normals(seed, design, 3u, l * (uint64_t)ui, n, w);
        for (int i = 0; i < n; ++i) {
            double x = 0.0;
            for (int k = 0; k <= i; ++k) x += L0[i * n + k] * w[k];
            X[l * n + i] = x;
        }
    }
    int64_t s1 = 0, s2 = 0;
    for (uint64_t k = 0; k < n1; ++k) {
        double eps[2 * OR_MAXN + 2], b[OR_MAXN];
        bm_normals(seed, design, 2u, k * (uint64_t)uo, p, eps);
        for (int i = 0; i < n; ++i) {
            double dl = theta[i];
            for (int c = 0; c <= i; ++c) dl += Lp[i * p + c] * eps[c];
            b[i] = z[i] - sqrt(r[i] * i3) * dl;
        }
        int64_t ck = 0;
        for (uint64_t l = 0; l < n2; ++l) {
            int rej = 0;
            for (int i = 0; i < n; ++i) if (X[l * n + i] > b[i]) rej = 1;
            ck += rej;
        }
        s1 += ck;
        s2 += ck * ck;
    }
    free(X);
    sums[0] += s1;
    sums[1] += s2;
}
