// mc_device.cuh — device arithmetic of the fused Monte-Carlo kernel (sm_100a, fp32 + integer).
//
// Implements DESIGN.md §2.2-2.7 (the contract the independent oracle also implements):
//   Philox4x32-10 word stream keyed (design, sample)          §2.2
//   23-bit uniforms, Box-Muller on MUFU.{LG2,SQRT,SIN,COS}     §2.3
//   prior draw Delta = theta + L_p eps  (Formula 10) §2.4, folded into b = zc - M eps
//   utility u: COND (SOV normal CDFs) or IND (Formula 6/7)     §2.5, §2.6
//   exact 2^-23 fixed-point accumulation                       §2.7
#pragma once
#include <cstdint>

namespace mcd {

constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }

// Geometry of the word stream for N populations, estimator EST (0 COND, 1 IND) and prior MODEL
// (0: Gaussian, prior dimension P = N; 1: the C4 strata prior, P = 5, N = 2).  The stream of a design
// is cut into RECORDS of R = 2 consecutive samples: COND (the pair shares P Box-Muller
// pairs: 2P normals, then NE SOV uniforms per sample), IND (NPS pairs per sample, sample 0 first).  A record's U
// uniforms are 23-bit fields: PACKED into WR = 2 ceil(23 U / 64) words when that is fewer than U (uniform
// i = bits [23 i, 23 i + 23) of the record's little-endian bit string; U >= 8), else one per word (its low
// 23 bits).  n = 3 COND packs 8 uniforms into 6 words per sample pair: 1.5 Philox blocks instead of 2.
template <int N, int EST, int MODEL = 0>
struct Geo {
  static constexpr int P = MODEL == 1 ? 5 : N;
  static constexpr int NNORM = (EST == 0) ? P : P + N;          // normals per sample
  static constexpr int NE = N / 2;           // COND: even populations (sampled), 0-based index 2k+1
  static constexpr int NO = (N + 1) / 2;     // COND: odd populations (analytic), 0-based index 2j
  static constexpr int R = 2;                                     // samples per record (a pair)
  static constexpr int NPS = (NNORM + 1) / 2;                     // IND: Box-Muller pairs per sample
  static constexpr int NPAIR = (EST == 0) ? P : 2 * NPS;          // Box-Muller pairs per record
  static constexpr int SOFF = (EST == 0) ? P : 2 * NPS;           // sample h's normals start at h SOFF
  static constexpr int U = (EST == 0) ? 2 * P + 2 * NE : 2 * NPAIR;    // 23-bit uniforms per record
  static constexpr bool PACKED = 2 * ((23 * U + 63) / 64) < U;    // packing saves words (U >= 8)
  static constexpr int WR = PACKED ? 2 * ((23 * U + 63) / 64) : U;   // words per record
  static constexpr int LR = 4 / cgcd(WR, 4);                      // records per Philox-aligned step
  static constexpr int L = R * LR;                                // samples per step
  static constexpr int BLOCKS = LR * WR / 4;                      // Philox blocks per step
  static constexpr int NM = N * (N + 1) / 2;                      // packed lower-triangular M
  static constexpr int DUMP = NNORM + N + 1;                      // floats per dumped draw
  // first word of sample s (s a multiple of R) and of its record
  static __host__ __device__ constexpr uint64_t word_of(uint64_t s) { return s / R * (uint64_t)WR; }
};

// ---------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11).  Counter (q_lo, q_hi, design, 0), key (seed_lo, seed_hi).
// The ten round keys (k0 + r W0, k1 + r W1), r = 0..9, precomputed on the host and passed by value
// as a kernel parameter: the rounds then read them straight from the constant bank (no key schedule
// in the loop).
struct RoundKeys { uint32_t k0[10], k1[10]; };

__host__ __device__ inline RoundKeys round_keys(uint64_t seed) {
  RoundKeys rk;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    rk.k0[r] = k0;
    rk.k1[r] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return rk;
}

// 32x32 -> 64-bit product as ONE IMAD.WIDE.U32 (ptxas otherwise often splits it into IMAD.HI + IMAD).
__device__ __forceinline__ void mulhilo(uint32_t a, uint32_t m, uint32_t& hi, uint32_t& lo) {
  uint64_t p;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(m));
  lo = (uint32_t)p;
  hi = (uint32_t)(p >> 32);
}

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                             uint32_t k0, uint32_t k1) {
  uint32_t lo0, hi0, lo1, hi1;
  mulhilo(c0, 0xD2511F53u, hi0, lo0);
  mulhilo(c2, 0xCD9E8D57u, hi1, lo1);
  c0 = hi1 ^ c1 ^ k0;
  c1 = lo1;
  c2 = hi0 ^ c3 ^ k1;
  c3 = lo0;
}

// Same block with the precomputed round keys (the fused kernel's form).
__device__ __forceinline__ void philox_block_rk(uint64_t q, uint32_t lo1d, uint32_t hi1d, const RoundKeys& rk,
                                                uint32_t out[4]) {
  const uint32_t q0 = (uint32_t)q, q1 = (uint32_t)(q >> 32);
  uint32_t hq, lq;
  mulhilo(q0, 0xD2511F53u, hq, lq);
  uint32_t c0 = hi1d ^ q1 ^ rk.k0[0];
  uint32_t c1 = lo1d;
  uint32_t c2 = hq ^ rk.k1[0];
  uint32_t c3 = lq;
#pragma unroll
  for (int r = 1; r < 10; ++r) philox_round(c0, c1, c2, c3, rk.k0[r], rk.k1[r]);
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// Block for counter (q_lo, q_hi, design, 0) when the caller holds the round-1 word
// c0 = hi(M1 * design) ^ q_hi ^ k0 fixed (q_hi constant over a thread's run): one IMAD.WIDE and one
// LOP3 in round 1 instead of two each.
// k1r1 = k1 ^ c3 of round 1 (c3 = the stream tag: 0 independent, 1 common random numbers).
__device__ __forceinline__ void philox_block_lo(uint32_t q0, uint32_t c0r1, uint32_t lo1d, uint32_t k1r1,
                                                const RoundKeys& rk, uint32_t out[4]) {
  uint32_t hq, lq;
  mulhilo(q0, 0xD2511F53u, hq, lq);
  uint32_t c0 = c0r1;
  uint32_t c1 = lo1d;
  uint32_t c2 = hq ^ k1r1;
  uint32_t c3 = lq;
#pragma unroll
  for (int r = 1; r < 10; ++r) philox_round(c0, c1, c2, c3, rk.k0[r], rk.k1[r]);
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// Word w of the stream (id, tag): counter (q_lo, q_hi, id, tag) — plain 10-round form (test hooks).
__device__ __forceinline__ uint32_t philox_word_tagged(uint64_t seed, uint32_t id, uint32_t tag, uint64_t w) {
  uint32_t c0 = (uint32_t)(w >> 2), c1 = (uint32_t)(w >> 34), c2 = id, c3 = tag;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    philox_round(c0, c1, c2, c3, k0, k1);
  }
  const uint32_t o[4] = {c0, c1, c2, c3};
  return o[w & 3];
}

// ---------------------------------------------------------------------------------------------
// Fast fp32 primitives on the SFU (MUFU) pipe.
__device__ __forceinline__ float lg2_approx(float x) { float y; asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2_approx(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcp_approx(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float sqrt_approx(float x) { float y; asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float sin_approx(float x) { float y; asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float cos_approx(float x) { float y; asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

// 1 + k 2^-23 in [1, 2) from the low 23 bits k of a Philox word as ONE LOP3
// ((w & 0x7FFFFF) | one): `one` = 0x3F800000 held in a register by the caller (ptxas cannot encode two
// immediates in one LOP3).
__device__ __forceinline__ float word_to_f12(uint32_t w, uint32_t one) {
  uint32_t r;
  asm("lop3.b32 %0, %1, 0x007FFFFF, %2, 0xEA;" : "=r"(r) : "r"(w), "r"(one));
  return __uint_as_float(r);
}
// Record uniform i as 1 + k 2^-23, k = the 23-bit field at bit offset 23 i of the record words w[] (PACKED)
// or the low 23 bits of word i: one LOP3, plus one SHF (shift or funnel shift across two
// words) for a packed field unless 23 i is a multiple of 32.  i is a compile-time constant at every call site (unrolled loops), so the word
// indices and shifts fold.
template <bool PACKED>
__device__ __forceinline__ float unif_f12(const uint32_t* w, int i, uint32_t one) {
  if constexpr (!PACKED) return word_to_f12(w[i], one);
  const int b = 23 * i, j = b >> 5, sh = b & 31;
  const uint32_t f = sh == 0 ? w[j] : (sh <= 9 ? (w[j] >> sh) : __funnelshift_r(w[j], w[j + 1], sh));
  return word_to_f12(f, one);
}
__device__ __forceinline__ uint32_t one_bits_reg() {
  uint32_t r;
  asm volatile("mov.b32 %0, 0x3F800000;" : "=r"(r));
  return r;
}

// Box-Muller scale: R = sqrt(-2 ln u) = BM_K sqrt(-log2 u), BM_K = sqrt(2 ln 2).  The kernel draws the
// scaled normals eps / BM_K and folds BM_K into the per-problem factors (see problem_record()).
constexpr float BM_K = 1.17741002251547469f;

// The kernel's Box-Muller from the two uniforms as 1 + k 2^-23 (fr, fa): returns (n0, n1) / BM_K.
// sqrt(|log2 u_r|) replaces the clamp at 0 (log2 of u_r <= 1 can come back ~1e-7 positive from
// MUFU.LG2); the angle 2 pi (u_a - 1/2) is one FFMA.
__device__ __forceinline__ void box_muller_f12(float fr, float fa, float& n0, float& n1) {
  const float ur = 2.0f - fr;
  const float mr = -sqrt_approx(fabsf(lg2_approx(ur)));
  const float x = fmaf(fa, 6.28318530718f, -9.42477796077f);
  n0 = mr * cos_approx(x);
  n1 = mr * sin_approx(x);
}
// ... from two whole words (the crossed estimator's streams keep one uniform per word)
__device__ __forceinline__ void box_muller_scaled(uint32_t wr, uint32_t wa, uint32_t one, float& n0, float& n1) {
  box_muller_f12(word_to_f12(wr, one), word_to_f12(wa, one), n0, n1);
}

// Upper normal tail q = Phi(-x), x >= 0, as ONE power of two: q = 2^E(m), m = min(|a|, PHI_CLAMP), E a
// degree-9 polynomial in m that includes the -a^2 term (tools/fit_normal_tail_ex2.py: relative error 9.0e-7
// in exact arithmetic, 1.8e-6 in fp32 for x <= 4).  The argument arrives PRE-SCALED,
// a = x sqrt(log2(e)/2) (the COND record folds the factor into M, the thresholds and the stage
// coefficients: mc_api.cu PHI_SCALE), so E ~ -a^2.  Beyond the clamp (x > 5.887) q is held at
// q(5.887) = 2.0e-9 (reading R25): ten stages add at most 2.0e-8, below half the per-draw 2^-23
// fixed-point step, so alpha = 0 (z = +inf, a = +inf) gives u = 0 exactly for every n <= 10.  One MUFU (EX2), no reciprocal: round 1's
// Numerical-Recipes form t = 1/(1 + kappa x), q = t 2^(P(t) - a^2) needed RCP + EX2 per call.
// Returns q and e = 1 - q (= Phi(x)) without cancellation for either sign of a.
#ifndef MC_PHI_DEG
#define MC_PHI_DEG 9      // 11: the degree-11 fit on m <= 5 (3.6e-8 exact), -4 % draws/s (profiles/r02/tune_pk2.jsonl)
#endif
#if MC_PHI_DEG == 9
// degree 9 on m <= 5 (x <= 5.887, q(clamp) = 2.0e-9): relative error 9.0e-7 exact, 1.8e-6 fp32 (x <= 4)
constexpr float PHI_CLAMP = 5.0f;
#define MC_PHI_POLY(HORNER, m)                                                                              \
  HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(                                         \
      2.4093271849031533e-07f, m, -5.50882381484465e-06f), m, 4.659686919954287e-05f), m,                   \
      -0.0001033207823907455f), m, -0.0013127185110967503f), m, 0.014977484435093462f), m,                   \
      -0.08674957729065969f), m, -0.6362018435487484f), m, -1.355378895260889f), m, -0.9999986975583613f)
#else
constexpr float PHI_CLAMP = 5.0f;
#define MC_PHI_POLY(HORNER, m)                                       \
  HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER( \
      1.3214344735792895e-08f, m, -4.290973434515816e-07f), m, 6.177874180542052e-06f), m,                   \
      -5.145014405324849e-05f), m, 0.0002655422273086682f), m, -0.0007692117070775829f), m,                    \
      -1.9095885481130195e-05f), m, 0.013417788461371934f), m, -0.08565676580912412f), m,                      \
      -0.6365931830340086f), m, -1.355324411309415f), m, -0.9999999477305315f)
#endif
__device__ __forceinline__ float horner1(float p, float x, float c) { return fmaf(p, x, c); }

__device__ __forceinline__ void normal_tail(float a, float& q, float& e) {
  const float m = fminf(fabsf(a), PHI_CLAMP);
  const float qp = ex2_approx(MC_PHI_POLY(horner1, m));   // Phi(-|x|)
  const float qc = 1.0f - qp;                              // Phi(|x|)
  const bool pos = a >= 0.0f;
  q = pos ? qp : qc;
  e = pos ? qc : qp;
}

// Standard normal quantile Phi^{-1}(p) given p and its complement pc = 1 - p (both computed accurately by
// the caller): Phi^{-1}(p) = g(t) (p - pc) with t = w/8 - 1, w = -ln(4 p pc) in [0, 16]
// (p in [2.8e-8, 1 - 2.8e-8]), g ONE degree-12 polynomial in t (tools/fit_erfinv_w.py: relative error
// 1.3e-6 in exact arithmetic, 2.3e-6 in fp32) — no square root, no per-coefficient selects and no branch.
// t = lg2(p pc) (-ln2/8) + (-ln4/8 - 1) is one FFMA after MUFU.LG2.  Beyond that range t is clamped to 1
// (w = 16, reading R24): in the SOV this only happens when v e_k < 2.8e-8 (the upper side cannot clamp:
// 1 - v >= 2^-24), and the resulting change of u is at most e_k on an event of probability
// <= 2.8e-8 / e_k, i.e. a bias of at most 2.8e-8 per even stage.  Round 1 used a degree-12 polynomial
// in sqrt(w + 2) (one MUFU.SQRT more per call) and before that a deep-tail branch (-4.8 % draws/s).
#ifndef MC_QUANT_DEG
#define MC_QUANT_DEG 12   // 14: relative error 6.0e-8 exact, one packed FFMA more per call
#endif
#if MC_QUANT_DEG == 12
// degree 12: relative error 1.3e-6 exact, 2.3e-6 fp32
#define MC_QUANTILE_POLY(HORNER, t)                                                                               \
  HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(                         \
      0.013822934060579422f, t, 0.01174856432856336f), t, -0.07083904242963865f), t, 0.0036023348788869554f), t, \
      0.10475706180380204f), t, -0.08248599065262685f), t, 0.0347135537264593f), t, -0.01678848886490599f), t,   \
      -0.046555255159994154f), t, 0.17713202118124255f), t, -0.45794967801334f), t, 1.995276138502238f), t,      \
      3.7638474592654703f)
#else
#define MC_QUANTILE_POLY(HORNER, t)                                                                               \
  HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(HORNER(           \
      0.01019474611084561f, t, -0.012522037903250294f), t, -0.029537615373728402f), t, 0.05105979421834458f), t, \
      0.001191401517323608f), t, -0.0434556915527025f), t, 0.04556025718938638f), t, -0.05578006817451819f), t,  \
      0.059710341538845794f), t, -0.024018910794271674f), t, -0.05160295363704608f), t, 0.17794569832657112f), t, \
      -0.45756438521357723f), t, 1.9952513929012803f), t, 3.7638425973256995f)
#endif
constexpr float QT_A = -0.08664339756999316f;    // -ln2 / 8
constexpr float QT_B = -1.1732867951399863f;     // -ln4 / 8 - 1

__device__ __forceinline__ float normal_quantile_fast(float p, float pc) {
  // p pc may flush to 0 (lg2 -> -inf, t -> +inf): the clamp holds
  const float t = fminf(fmaf(lg2_approx(p * pc), QT_A, QT_B), 1.0f);
  return MC_QUANTILE_POLY(horner1, t) * (p - pc);
}

// ---------------------------------------------------------------------------------------------
// Per-problem parameters in registers (loaded once per tile; uniform across the block).
//
// COND evaluates the SOV in the order (populations 2, 4, ..., then 1, 3, ...): by the
// Markov structure of A.1 the even populations form a chain X_{2k+2} | X_{2k} ~ N(mu x, sd^2) and each
// odd population is conditionally independent of the rest given its even neighbours (a Gaussian
// bridge).  The device record folds the conditional standard deviations into the rows of M and zc
// (mc_api.cu problem_record()), so every stage argument is one or two FFMAs:
//   even k:  a = b'_{2k+1} - er_k x_{k-1},  x_k = emu_k x_{k-1} + esd_k Phi^{-1}(v_k e_k)
//   odd  j:  a = b'_{2j} - oa_j x_{j-1} - ob_j x_j
// IND uses the natural Markov recursion (rho, s) with b' = b / BM_K.
template <int N>
struct ProbRegs {
  static constexpr int NE = N / 2 > 0 ? N / 2 : 1, NO = (N + 1) / 2, NR = N > 1 ? N - 1 : 1;
  float M[N * (N + 1) / 2];   // packed lower triangular (row i: M[i(i+1)/2 + j])
  float rho[NR], sd[NR];      // IND
  float er[NE], emu[NE], esd[NE], oa[NO], ob[NO];   // COND
};

// One draw from its U words w[0..U): returns u in [0,1].  If DBG, writes the (unscaled) normals,
// b and u; bsc[i] (the row scales) and BM_K undo the folding for the dump.
// C4 strata prior parameters (MODEL 1; mc_api.cu problem_record(): sds pre-multiplied by BM_K).
struct StrataRegs {
  float pm, ps, dpm, dps, dmm, dms, lvm, lvs, ldm, lds;   // (mean, sd) of the five components
  float i3, inv_r2, inv_1mr2, r2, sqrt_r2, rs0, rs1;      // I3, 1/r2, 1/(1-r2), r2, sqrt(r2), row scales
};

// b = z - mu of the C4 strata model (oracle.c or_draw_strata) from the five scaled
// normals: I_eff = I3 (1-d)/v; q+ = min(1, pi/r2), q- = max(0, (pi - r2)/(1 - r2));
// Delta_2 = delta- + q+ (delta+ - delta-), Delta_neg = delta- + q- (delta+ - delta-),
// Delta_1 = Delta_neg + r2 (Delta_2 - Delta_neg); mu_1 = sqrt(I_eff) Delta_1, mu_2 = sqrt(r2 I_eff) Delta_2.
__device__ __forceinline__ void strata_b(const float* nrm, const float* zc, const StrataRegs& s, float* b) {
  constexpr float L2E = 1.44269504088896341f;
  const float pi = rcp_approx(1.0f + ex2_approx(-L2E * fmaf(s.ps, nrm[0], s.pm)));
  const float dp = fmaf(s.dps, nrm[1], s.dpm);
  const float dm = fmaf(s.dms, nrm[2], s.dmm);
  const float inv_v = ex2_approx(-L2E * fmaf(s.lvs, nrm[3], s.lvm));
  const float omd = rcp_approx(1.0f + ex2_approx(L2E * fmaf(s.lds, nrm[4], s.ldm)));   // 1 - d
  const float si = sqrt_approx(s.i3 * omd * inv_v);
  const float qp = fminf(1.0f, pi * s.inv_r2);
  const float qm = fmaxf(0.0f, (pi - s.r2) * s.inv_1mr2);
  const float dd = dp - dm;
  const float d2 = fmaf(qp, dd, dm);
  const float dneg = fmaf(qm, dd, dm);
  const float d1 = fmaf(s.r2, d2 - dneg, dneg);
  b[0] = fmaf(-si * s.rs0, d1, zc[0]);
  b[1] = fmaf(-si * s.sqrt_r2 * s.rs1, d2, zc[1]);
}

// The design-independent part of one draw (shared by every design under common random numbers,
// NEXT f3): the prior term v with b = zc - v, the IND null vector X, and the SOV uniforms.
template <int N, int EST, int MODEL = 0>
struct Shared {
  float v[N];
  float x[EST == 1 ? N : 1];                                   // IND: X = L0 W (scaled)
  float vu[Geo<N, EST, MODEL>::NE > 0 ? Geo<N, EST, MODEL>::NE : 1];   // COND: SOV uniforms v_k
};

// Box-Muller over the record's NPAIR word pairs: normals 2j, 2j+1 from words 2j (radius), 2j+1 (angle).
template <int N, int EST, int MODEL>
__device__ __forceinline__ void record_normals(const uint32_t* w, uint32_t one, float* nrm) {
  using G = Geo<N, EST, MODEL>;
#pragma unroll
  for (int j = 0; j < G::NPAIR; ++j)
    box_muller_f12(unif_f12<G::PACKED>(w, 2 * j, one), unif_f12<G::PACKED>(w, 2 * j + 1, one), nrm[2 * j], nrm[2 * j + 1]);
}

// Sample h of a record: its normals start at nrm + h SOFF (COND: h P; IND: h 2 NPS) and its SOV uniforms
// (COND) at record uniform 2P + h NE.
template <int N, int EST, int MODEL>
__device__ __forceinline__ void shared_of_sample(const float* nrm, const uint32_t* w, int h, uint32_t one,
                                                 const ProbRegs<N>& pr, const StrataRegs* sr, Shared<N, EST, MODEL>& sh) {
  using G = Geo<N, EST, MODEL>;
  const float* e = nrm + h * G::SOFF;
  if constexpr (MODEL == 1) {
    static_assert(N == 2, "the C4 strata model has n = 2");
    const float zero[2] = {0.0f, 0.0f};
    float bb[2];
    strata_b(e, zero, *sr, bb);
    sh.v[0] = -bb[0];
    sh.v[1] = -bb[1];
  } else {
    // c_i Delta_i - c_i theta_i = sum_{j<=i} (c_i L_p,ij) eps_j   (Formulas 3-5, 10)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      float acc = 0.0f;
#pragma unroll
      for (int j = 0; j <= i; ++j) acc = fmaf(pr.M[i * (i + 1) / 2 + j], e[j], acc);
      sh.v[i] = acc;
    }
  }
  if constexpr (EST == 1) {
    // Formula 6/7: the null draw X = L0 W by the Markov recursion
    float x = e[G::P];
    sh.x[0] = x;
#pragma unroll
    for (int i = 1; i < N; ++i) {
      x = fmaf(pr.rho[i - 1], x, pr.sd[i - 1] * e[G::P + i]);
      sh.x[i] = x;
    }
  } else {
#pragma unroll
    for (int k = 0; k < G::NE; ++k)   // (k+1/2) 2^-23
      sh.vu[k] = unif_f12<G::PACKED>(w, 2 * G::P + h * G::NE + k, one) - 0.99999994039535522f;
  }
}

// IND indicator 1[exists i: x_i > b_i] as ONE predicate chain (FSETP, then FSETP.OR per further
// population) and one select: ptxas otherwise materialises a select per population.
template <int N>
__device__ __forceinline__ float ind_indicator(const float* x, const float* b) {
  float u;
  if constexpr (N == 1) {
    asm("{ .reg .pred p; setp.gt.f32 p, %1, %2; selp.f32 %0, 0f3F800000, 0f00000000, p; }"
        : "=f"(u) : "f"(x[0]), "f"(b[0]));
  } else if constexpr (N == 2) {
    asm("{ .reg .pred p; setp.gt.f32 p, %1, %2; setp.gt.or.f32 p, %3, %4, p;"
        " selp.f32 %0, 0f3F800000, 0f00000000, p; }"
        : "=f"(u) : "f"(x[0]), "f"(b[0]), "f"(x[1]), "f"(b[1]));
  } else if constexpr (N == 3) {
    asm("{ .reg .pred p; setp.gt.f32 p, %1, %2; setp.gt.or.f32 p, %3, %4, p; setp.gt.or.f32 p, %5, %6, p;"
        " selp.f32 %0, 0f3F800000, 0f00000000, p; }"
        : "=f"(u) : "f"(x[0]), "f"(b[0]), "f"(x[1]), "f"(b[1]), "f"(x[2]), "f"(b[2]));
  } else {
    bool rej = x[0] > b[0];
#pragma unroll
    for (int i = 1; i < N; ++i) rej = rej | (x[i] > b[i]);
    u = rej ? 1.0f : 0.0f;
  }
  return u;
}

// cnt += 1[exists i: x_i > b_i] (the IND / Formula 7 rejection indicator) as ONE predicate chain (FSETP,
// FSETP.OR ...) on the ALU pipe and one predicated FADD on the FMA pipe (the crossed and CRN kernels)
template <int N>
__device__ __forceinline__ void ind_count(const float* x, const float* b, float& cnt) {
  static_assert(N >= 1 && N <= 4, "ind_count compares at most 4 populations (the crossed and CRN kernels' range)");
  if constexpr (N == 1) {
    asm("{ .reg .pred p; setp.gt.f32 p, %1, %2; @p add.f32 %0, %0, 0f3F800000; }"
        : "+f"(cnt) : "f"(x[0]), "f"(b[0]));
  } else if constexpr (N == 2) {
    asm("{ .reg .pred p; setp.gt.f32 p, %1, %2; setp.gt.or.f32 p, %3, %4, p; @p add.f32 %0, %0, 0f3F800000; }"
        : "+f"(cnt) : "f"(x[0]), "f"(b[0]), "f"(x[1]), "f"(b[1]));
  } else if constexpr (N == 3) {
    asm("{ .reg .pred p; setp.gt.f32 p, %1, %2; setp.gt.or.f32 p, %3, %4, p; setp.gt.or.f32 p, %5, %6, p;"
        " @p add.f32 %0, %0, 0f3F800000; }"
        : "+f"(cnt) : "f"(x[0]), "f"(b[0]), "f"(x[1]), "f"(b[1]), "f"(x[2]), "f"(b[2]));
  } else {
    asm("{ .reg .pred p; setp.gt.f32 p, %1, %2; setp.gt.or.f32 p, %3, %4, p; setp.gt.or.f32 p, %5, %6, p;"
        " setp.gt.or.f32 p, %7, %8, p; @p add.f32 %0, %0, 0f3F800000; }"
        : "+f"(cnt) : "f"(x[0]), "f"(b[0]), "f"(x[1]), "f"(b[1]), "f"(x[2]), "f"(b[2]), "f"(x[3]), "f"(b[3]));
  }
}

// The design-dependent part: the utility u in [0, 1] from the thresholds b (= zc - v).
template <int N, int EST, int MODEL>
__device__ __forceinline__ float utility_of_b(const float* b, const Shared<N, EST, MODEL>& sh, const ProbRegs<N>& pr) {
  using G = Geo<N, EST, MODEL>;
  float u = 0.0f;
  if constexpr (EST == 1) {
    // success iff some X_i > b_i
    u = ind_indicator<N>(sh.x, b);
  } else {
    // COND: u = 1 - prod e accumulated as u <- u + (1 - u) q (q = 1 - e: no cancellation).
    float x[G::NE > 0 ? G::NE : 1];
    float q, e;
#pragma unroll
    for (int k = 0; k < G::NE; ++k) {
      const float a = k == 0 ? b[1] : fmaf(-pr.er[k], x[k - 1], b[2 * k + 1]);
      normal_tail(a, q, e);
      u = k == 0 ? q : fmaf(1.0f - u, q, u);
      const float v = sh.vu[k];
      const float vc = 1.0f - v;                                            // exact
      const float y = normal_quantile_fast(v * e, fmaf(v, q, vc));
      x[k] = k == 0 ? y : fmaf(pr.esd[k], y, pr.emu[k] * x[k - 1]);
    }
#pragma unroll
    for (int j = 0; j < G::NO; ++j) {
      float a = b[2 * j];
      if (2 * j >= 1) a = fmaf(-pr.oa[j], x[j - 1], a);
      if (2 * j + 1 < N) a = fmaf(-pr.ob[j], x[j], a);
      normal_tail(a, q, e);
      u = (G::NE == 0 && j == 0) ? q : fmaf(1.0f - u, q, u);
    }
  }
  return u;
}

// ---------------------------------------------------------------------------------------------
// Packed-pair COND path (sm_100a FFMA2/FMUL2/FADD2, `fma.rn.f32x2`).  A COND record holds R = 2
// samples that run the identical instruction sequence on different data, so every FP32 operation of
// the pair is ONE packed instruction: each lane is an IEEE fp32 op with round-to-nearest, exactly
// what the scalar fmaf/mul/add computes, so the arithmetic per sample is unchanged (only ptxas's
// contraction choices differ where the scalar path wrote a*b+c as two ops).  MUFU work (LG2, SQRT,
// SIN, COS, RCP, EX2) and the selects stay scalar per lane.  The kernel is issue-bound,
// so halving the FP32 instruction count is the lever.
#ifndef MC_F32X2
#define MC_F32X2 1
#endif
typedef unsigned long long f2x;   // (lo = sample 0, hi = sample 1)
__device__ __forceinline__ f2x pk2(float lo, float hi) {
  f2x r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r;
}
__device__ __forceinline__ f2x bc2(float c) { return pk2(c, c); }
__device__ __forceinline__ void up2(f2x r, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
  f2x d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
  f2x d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
  f2x d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}

// normal_tail() for a pair: q = Phi(-x) and e = Phi(x) per lane, the same polynomial and operation order.
__device__ __forceinline__ f2x horner2(f2x p, f2x x, float c) { return fma2(p, x, bc2(c)); }
__device__ __forceinline__ f2x horner2(float p, f2x x, float c) { return fma2(bc2(p), x, bc2(c)); }

__device__ __forceinline__ void normal_tail2(f2x a, f2x& q, f2x& e) {
  float a0, a1;
  up2(a, a0, a1);
  const f2x m = pk2(fminf(fabsf(a0), PHI_CLAMP), fminf(fabsf(a1), PHI_CLAMP));
  float E0, E1;
  up2(MC_PHI_POLY(horner2, m), E0, E1);
  const f2x qp = pk2(ex2_approx(E0), ex2_approx(E1));   // Phi(-|x|)
  const f2x qc = fma2(qp, bc2(-1.0f), bc2(1.0f));        // Phi(|x|)
  float qp0, qp1, qc0, qc1;
  up2(qp, qp0, qp1);
  up2(qc, qc0, qc1);
  const bool pos0 = a0 >= 0.0f, pos1 = a1 >= 0.0f;
  q = pk2(pos0 ? qp0 : qc0, pos1 ? qp1 : qc1);
  e = pk2(pos0 ? qc0 : qp0, pos1 ? qc1 : qp1);
}

// normal_quantile_fast() for a pair (same polynomial, same clamp, reading R24).
__device__ __forceinline__ f2x normal_quantile_fast2(f2x p, f2x pc) {
  float m0, m1;
  up2(mul2(p, pc), m0, m1);
  float t0, t1;
  up2(fma2(pk2(lg2_approx(m0), lg2_approx(m1)), bc2(QT_A), bc2(QT_B)), t0, t1);
  const f2x t = pk2(fminf(t0, 1.0f), fminf(t1, 1.0f));
  return mul2(MC_QUANTILE_POLY(horner2, t), fma2(pc, bc2(-1.0f), p));   // g (p - pc)
}

// Lane-split forms: the same per-lane operations as normal_tail2 / normal_quantile_fast2 (bit-identical
// results) issued as scalar FFMAs.  A packed FFMA2 occupies BOTH the fmaheavy and fmalite datapaths for
// two cycles, while a scalar FFMA takes one of them; IMAD.WIDE (Philox) needs fmaheavy for four cycles.
// Moving part of the polynomial work to scalar FFMAs lets the scheduler run it on fmalite while fmaheavy
// is busy with Philox products (profiles/r02/pipe_model.md).
#ifndef MC_SCALAR_PHI_EVEN
#define MC_SCALAR_PHI_EVEN 0
#endif
#ifndef MC_SCALAR_PHI_ODD
#define MC_SCALAR_PHI_ODD 0
#endif
#ifndef MC_SCALAR_QUANTILE
#define MC_SCALAR_QUANTILE 0
#endif
__device__ __forceinline__ void normal_tail2s(f2x a, f2x& q, f2x& e) {
  float a0, a1, q0, q1, e0, e1;
  up2(a, a0, a1);
  normal_tail(a0, q0, e0);
  normal_tail(a1, q1, e1);
  q = pk2(q0, q1);
  e = pk2(e0, e1);
}
__device__ __forceinline__ f2x normal_quantile_fast2s(f2x p, f2x pc) {
  float p0, p1, c0, c1;
  up2(p, p0, p1);
  up2(pc, c0, c1);
  return pk2(normal_quantile_fast(p0, c0), normal_quantile_fast(p1, c1));
}
template <bool SCALAR>
__device__ __forceinline__ void normal_tail2x(f2x a, f2x& q, f2x& e) {
  if constexpr (SCALAR) normal_tail2s(a, q, e);
  else normal_tail2(a, q, e);
}

// utility_of_b<N, 0, MODEL> for two lanes at once: thresholds b[i] and SOV uniforms vu[k] packed
// (two samples of a record, or two designs sharing a sample under common random numbers).
template <int N>
__device__ __forceinline__ f2x utility_cond_x2(const f2x* b, const f2x* vu, const ProbRegs<N>& pr) {
  constexpr int NE = N / 2, NO = (N + 1) / 2;
  f2x uu = 0ull, q, e;
  f2x x[NE > 0 ? NE : 1];
#pragma unroll
  for (int k = 0; k < NE; ++k) {
    const f2x a = k == 0 ? b[1] : fma2(bc2(-pr.er[k]), x[k > 0 ? k - 1 : 0], b[2 * k + 1]);
    normal_tail2x<MC_SCALAR_PHI_EVEN>(a, q, e);
    uu = k == 0 ? q : fma2(fma2(uu, bc2(-1.0f), bc2(1.0f)), q, uu);
    const f2x v = vu[k];
    const f2x vc = fma2(v, bc2(-1.0f), bc2(1.0f));                            // exact
    const f2x y = MC_SCALAR_QUANTILE ? normal_quantile_fast2s(mul2(v, e), fma2(v, q, vc))
                                     : normal_quantile_fast2(mul2(v, e), fma2(v, q, vc));
    x[k] = k == 0 ? y : fma2(bc2(pr.esd[k]), y, mul2(bc2(pr.emu[k]), x[k > 0 ? k - 1 : 0]));
  }
#pragma unroll
  for (int j = 0; j < NO; ++j) {
    f2x a = b[2 * j];
    if (2 * j >= 1) a = fma2(bc2(-pr.oa[j]), x[j > 0 ? j - 1 : 0], a);
    if (2 * j + 1 < N) a = fma2(bc2(-pr.ob[j]), x[j < NE ? j : 0], a);
    normal_tail2x<MC_SCALAR_PHI_ODD>(a, q, e);
    uu = (NE == 0 && j == 0) ? q : fma2(fma2(uu, bc2(-1.0f), bc2(1.0f)), q, uu);
  }
  return uu;
}

// Both utilities of a COND record (MODEL 0), packed: sample 0 in the low lane, sample 1 in the high lane.
// Same words, same normals (pairs consumed in word order, cos first; sample h's normals at nrm + hP),
// same stage order as utility_of_b<N, 0, 0>.  This is the fused kernel's COND code; with DBG (the
// mc_draw_dump test hook) it also writes, per sample h, its unscaled normals, b and u to dbg + h DUMP.
template <int N, bool DBG = false>
__device__ __forceinline__ void record_utility_cond_x2(const uint32_t* w, uint32_t one, const float* zc,
                                                       const ProbRegs<N>& pr, float* u, float* dbg = nullptr,
                                                       const float* bsc = nullptr) {
  using G = Geo<N, 0, 0>;
  constexpr int P = G::P, NE = G::NE;
  // Box-Muller (box_muller_scaled) with the radius and angle FFMAs of two word pairs packed
  float mr[P], cs[P], sn[P];
#pragma unroll
  for (int j = 0; j < P; j += 2) {
    float ur[2], xa[2];
    if (j + 1 < P) {
      up2(fma2(pk2(unif_f12<G::PACKED>(w, 2 * j, one), unif_f12<G::PACKED>(w, 2 * j + 2, one)), bc2(-1.0f), bc2(2.0f)),
          ur[0], ur[1]);
      up2(fma2(pk2(unif_f12<G::PACKED>(w, 2 * j + 1, one), unif_f12<G::PACKED>(w, 2 * j + 3, one)), bc2(6.28318530718f),
               bc2(-9.42477796077f)), xa[0], xa[1]);
    } else {
      ur[0] = 2.0f - unif_f12<G::PACKED>(w, 2 * j, one);
      xa[0] = fmaf(unif_f12<G::PACKED>(w, 2 * j + 1, one), 6.28318530718f, -9.42477796077f);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (j + h < P) {
        mr[j + h] = -sqrt_approx(fabsf(lg2_approx(ur[h])));
        cs[j + h] = cos_approx(xa[h]);
        sn[j + h] = sin_approx(xa[h]);
      }
    }
  }
  // packed normals E[j] = (eps_j of sample 0, eps_j of sample 1) = (nrm[j], nrm[P + j])
  f2x E[P];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const int m0 = j, m1 = P + j;
    E[j] = mul2(pk2(mr[m0 / 2], mr[m1 / 2]), pk2(m0 % 2 ? sn[m0 / 2] : cs[m0 / 2], m1 % 2 ? sn[m1 / 2] : cs[m1 / 2]));
  }
  // b = zc - M eps
  f2x b[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    f2x acc = bc2(zc[i]);
#pragma unroll
    for (int j = 0; j <= i; ++j) acc = fma2(bc2(-pr.M[i * (i + 1) / 2 + j]), E[j], acc);
    b[i] = acc;
  }
  f2x vu[NE > 0 ? NE : 1];
#pragma unroll
  for (int k = 0; k < NE; ++k)   // the SOV uniforms (k+1/2) 2^-23 of both samples
    vu[k] = add2(pk2(unif_f12<G::PACKED>(w, 2 * P + k, one), unif_f12<G::PACKED>(w, 2 * P + NE + k, one)),
                 bc2(-0.99999994039535522f));
  up2(utility_cond_x2<N>(b, vu, pr), u[0], u[1]);
  if constexpr (DBG) {
    constexpr int DUMP = G::DUMP;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      float e0, e1;
      up2(E[j], e0, e1);
      dbg[j] = e0 * BM_K;
      dbg[DUMP + j] = e1 * BM_K;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      float b0, b1;
      up2(b[i], b0, b1);
      dbg[P + i] = b0 / bsc[i];
      dbg[DUMP + P + i] = b1 / bsc[i];
    }
    dbg[P + N] = u[0];
    dbg[DUMP + P + N] = u[1];
  }
}

// Independent draws: the R utilities of one record, b formed directly from zc (FFMA chains seeded
// with zc, no separate v).  If DBG, writes per sample the (unscaled) normals, b and u; bsc[i] (the
// row scales) and BM_K undo the folding for the dump.
template <int N, int EST, bool DBG, int MODEL = 0>
__device__ __forceinline__ void record_utility(const uint32_t* w, uint32_t one, const float* zc, const ProbRegs<N>& pr,
                                               const StrataRegs* sr, float* u, float* dbg = nullptr,
                                               const float* bsc = nullptr) {
  using G = Geo<N, EST, MODEL>;
#if MC_F32X2
  // COND: the packed pair.  The DBG instantiation (mc_draw_dump) runs this same code and dumps from it.
  if constexpr (EST == 0 && MODEL == 0) {
    record_utility_cond_x2<N, DBG>(w, one, zc, pr, u, dbg, bsc);
    return;
  }
  if constexpr (EST == 0 && MODEL == 1) {   // C4 strata prior: b per sample, the SOV packed
    float nrm[2 * G::NPAIR];
    record_normals<N, EST, MODEL>(w, one, nrm);
    Shared<N, EST, MODEL> sh0, sh1;
    shared_of_sample<N, EST, MODEL>(nrm, w, 0, one, pr, sr, sh0);
    shared_of_sample<N, EST, MODEL>(nrm, w, 1, one, pr, sr, sh1);
    f2x b[N], vu[G::NE > 0 ? G::NE : 1];
#pragma unroll
    for (int i = 0; i < N; ++i) b[i] = pk2(zc[i] - sh0.v[i], zc[i] - sh1.v[i]);
#pragma unroll
    for (int k = 0; k < G::NE; ++k) vu[k] = pk2(sh0.vu[k], sh1.vu[k]);
    up2(utility_cond_x2<N>(b, vu, pr), u[0], u[1]);
    if constexpr (DBG) {
#pragma unroll
      for (int k = 0; k < 2 * G::P; ++k) dbg[(k / G::P) * G::DUMP + k % G::P] = nrm[k] * BM_K;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        float b0, b1;
        up2(b[i], b0, b1);
        dbg[G::P + i] = b0 / bsc[i];
        dbg[G::DUMP + G::P + i] = b1 / bsc[i];
      }
      dbg[G::P + N] = u[0];
      dbg[G::DUMP + G::P + N] = u[1];
    }
    return;
  }
#endif
  float nrm[2 * G::NPAIR];
  record_normals<N, EST, MODEL>(w, one, nrm);
#pragma unroll
  for (int h = 0; h < G::R; ++h) {
    Shared<N, EST, MODEL> sh;
    float b[N];
    const float* e = nrm + h * G::SOFF;
    if constexpr (MODEL == 1) {
      shared_of_sample<N, EST, MODEL>(nrm, w, h, one, pr, sr, sh);
#pragma unroll
      for (int i = 0; i < N; ++i) b[i] = zc[i] - sh.v[i];
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        float acc = zc[i];
#pragma unroll
        for (int j = 0; j <= i; ++j) acc = fmaf(-pr.M[i * (i + 1) / 2 + j], e[j], acc);
        b[i] = acc;
      }
      if constexpr (EST == 1) {
        float x = e[G::P];
        sh.x[0] = x;
#pragma unroll
        for (int i = 1; i < N; ++i) {
          x = fmaf(pr.rho[i - 1], x, pr.sd[i - 1] * e[G::P + i]);
          sh.x[i] = x;
        }
      } else {
#pragma unroll
        for (int k = 0; k < G::NE; ++k) sh.vu[k] = unif_f12<G::PACKED>(w, 2 * G::P + h * G::NE + k, one) - 0.99999994039535522f;
      }
    }
    u[h] = utility_of_b<N, EST, MODEL>(b, sh, pr);
    if constexpr (DBG) {
      float* o = dbg + h * G::DUMP;
#pragma unroll
      for (int k = 0; k < G::P; ++k) o[k] = e[k] * BM_K;
#pragma unroll
      for (int k = G::P; k < G::NNORM; ++k) o[k] = e[k] * BM_K;   // IND null normals
#pragma unroll
      for (int i = 0; i < N; ++i) o[G::NNORM + i] = b[i] / bsc[i];
      o[G::NNORM + N] = u[h];
    }
  }
}

}  // namespace mcd
