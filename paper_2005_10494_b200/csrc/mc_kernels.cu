// mc_kernels.cu — K1 fused Monte-Carlo kernel, K2 finalize, K3 Philox dump, draw dump, K6 argmax.
//
// K1 (rows a2-a6 of DESIGN.md §1): one warp per warp tile (design, 32 x 128 samples), hardware-balanced.
// Each thread owns 128 consecutive samples of one design, generates their Philox words in
// registers (records of R samples, WR words, LR records per aligned step), evaluates u, and accumulates the exact
// 2^-23 fixed-point sums in 32-bit registers; a 64-bit warp shuffle reduction then issues one 64-bit
// atomicAdd pair per warp tile (no block barrier).  Integer sums make the result independent of the
// launch shape.
#include <cuda_runtime.h>

#include <cfloat>
#include <math_constants.h>
#include <cstdint>
#include <vector>
#include <algorithm>

#include "mc_device.cuh"
#include "mc_internal.h"

namespace mci {

using namespace mcd;

template <int N>
__device__ __forceinline__ void load_problem(const float* __restrict__ rec, ProbRegs<N>& pr) {
#pragma unroll
  for (int k = 0; k < N * (N + 1) / 2; ++k) pr.M[k] = __ldg(rec + OFF_M + k);
#pragma unroll
  for (int k = 0; k < N - 1; ++k) {
    pr.rho[k] = __ldg(rec + OFF_RHO + k);
    pr.sd[k] = __ldg(rec + OFF_SD + k);
  }
#pragma unroll
  for (int k = 0; k < N / 2; ++k) {
    pr.er[k] = __ldg(rec + OFF_ER + k);
    pr.emu[k] = __ldg(rec + OFF_EMU + k);
    pr.esd[k] = __ldg(rec + OFF_ESD + k);
  }
#pragma unroll
  for (int k = 0; k < (N + 1) / 2; ++k) {
    pr.oa[k] = __ldg(rec + OFF_OA + k);
    pr.ob[k] = __ldg(rec + OFF_OB + k);
  }
}

__device__ __forceinline__ void load_strata(const float* __restrict__ rec, StrataRegs& sr) {
  const float* r = rec + OFF_STR;
  sr.pm = __ldg(r + 0); sr.ps = __ldg(r + 1); sr.dpm = __ldg(r + 2); sr.dps = __ldg(r + 3);
  sr.dmm = __ldg(r + 4); sr.dms = __ldg(r + 5); sr.lvm = __ldg(r + 6); sr.lvs = __ldg(r + 7);
  sr.ldm = __ldg(r + 8); sr.lds = __ldg(r + 9); sr.i3 = __ldg(r + 10); sr.inv_r2 = __ldg(r + 11);
  sr.inv_1mr2 = __ldg(r + 12); sr.r2 = __ldg(r + 13); sr.sqrt_r2 = __ldg(r + 14); sr.rs0 = __ldg(r + 15);
  sr.rs1 = __ldg(r + 16);
}

// fixed-point accumulation of one draw: q(x) = round-half-even(2^23 x) for x in [0,1] is the
// mantissa of the fp32 sum x + 1 (one FADD / FFMA + one IADD3).  IND: u in {0, 1}, u^2 = u, so only
// the first sum is accumulated (the second is copied at the end).
template <int EST>
__device__ __forceinline__ void accumulate(float u, uint32_t& a1, uint32_t& a2) {
  a1 += __float_as_uint(u + 1.0f) - 0x3F800000u;
  if constexpr (EST == 0) a2 += __float_as_uint(fmaf(u, u, 1.0f)) - 0x3F800000u;
}
// Steady-state form: the raw bit patterns are summed modulo 2^32 and the constant 0x3F800000 per draw
// is removed once per run (finish_biased); exact because the true sum stays below 2^31.
// (COND only: the IND indicator already folds into one select per draw.)
// IND: u in {0, 1} is counted in an fp32 register (exact up to 2^24 >> 128 draws) and converted once.
template <int EST>
__device__ __forceinline__ void accumulate_biased(float u, uint32_t& a1, uint32_t& a2, float& cnt) {
  if constexpr (EST == 0) {
    a1 += __float_as_uint(u + 1.0f);
    a2 += __float_as_uint(fmaf(u, u, 1.0f));
  } else {
    cnt += u;
  }
}
template <int EST>
__device__ __forceinline__ void finish_biased(uint32_t draws, uint32_t& a1, uint32_t& a2, float cnt) {
  if constexpr (EST == 0) {
    a1 -= draws * 0x3F800000u;
    a2 -= draws * 0x3F800000u;
  } else {
    a1 += (uint32_t)cnt << 23;
  }
}

#ifndef MC_STEP_UNROLL
#define MC_STEP_UNROLL 1
#endif
#ifndef MC_PIPELINE_PHILOX
#define MC_PIPELINE_PHILOX 0   // 1: generate step t+1's Philox blocks while step t is evaluated
#endif
#ifndef MC_STEP_UNROLL_COND
#define MC_STEP_UNROLL_COND MC_STEP_UNROLL
#endif
constexpr int kStepUnroll = MC_STEP_UNROLL;   // steady-loop unroll (pragma arguments are not macro-expanded)
constexpr int kStepUnrollCond = MC_STEP_UNROLL_COND;
template <int N, int EST, bool MASKED, int MODEL>
__device__ __forceinline__ void run_samples(uint64_t s_begin, uint64_t B, uint64_t E, uint32_t lo1d, uint32_t hi1d,
                                            const RoundKeys& rk, const float* zc, const ProbRegs<N>& pr,
                                            const StrataRegs& sr, uint32_t& a1, uint32_t& a2) {
  using G = Geo<N, EST, MODEL>;
  constexpr int STEPS = SAMPLES_PER_THREAD / G::L;
  static_assert(SAMPLES_PER_THREAD % G::L == 0, "L must divide the per-thread run");
  uint64_t q = G::word_of(s_begin) / 4;   // first Philox block of this thread's run
  const uint32_t one = one_bits_reg();
  if constexpr (!MASKED) {
    // steady state: the run's Philox counters q .. q + STEPS*BLOCKS share q_hi unless the low word wraps
    constexpr uint32_t NBLK = (uint32_t)(STEPS * G::BLOCKS);
    const uint32_t q0 = (uint32_t)q;
    if (q0 <= 0xFFFFFFFFu - NBLK) {
      const uint32_t c0r1 = hi1d ^ (uint32_t)(q >> 32) ^ rk.k0[0];
      uint32_t ql = q0;
      float cnt = 0.0f;
      auto eval_step = [&](const uint32_t* w) {
#pragma unroll
        for (int r = 0; r < G::LR; ++r) {
          float u[G::R];
          record_utility<N, EST, false, MODEL>(&w[r * G::WR], one, zc, pr, &sr, u);
#if MC_F32X2
          if constexpr (EST == 0) {   // the pair's u + 1 and u u + 1 as one FADD2 and one FFMA2
            const f2x uu = pk2(u[0], u[1]);
            float s0, s1, t0, t1;
            up2(add2(uu, bc2(1.0f)), s0, s1);
            up2(fma2(uu, uu, bc2(1.0f)), t0, t1);
            a1 += __float_as_uint(s0) + __float_as_uint(s1);
            a2 += __float_as_uint(t0) + __float_as_uint(t1);
          } else
#endif
          {
#pragma unroll
            for (int h = 0; h < G::R; ++h) accumulate_biased<EST>(u[h], a1, a2, cnt);
          }
        }
      };
#if MC_PIPELINE_PHILOX
      // software-pipelined: the next step's Philox blocks (IMAD.WIDE / LOP3) are generated in the same
      // basic block as this step's Box-Muller / normal-CDF chains, so the scheduler can interleave them
      uint32_t wn[G::BLOCKS * 4];
#pragma unroll
      for (int b = 0; b < G::BLOCKS; ++b) philox_block_lo(ql + b, c0r1, lo1d, rk.k1[0], rk, &wn[4 * b]);
      ql += G::BLOCKS;
#pragma unroll 1
      for (int st = 0; st < STEPS - 1; ++st) {
        uint32_t w[G::BLOCKS * 4];
#pragma unroll
        for (int k = 0; k < G::BLOCKS * 4; ++k) w[k] = wn[k];
#pragma unroll
        for (int b = 0; b < G::BLOCKS; ++b) philox_block_lo(ql + b, c0r1, lo1d, rk.k1[0], rk, &wn[4 * b]);
        ql += G::BLOCKS;
        eval_step(w);
      }
      eval_step(wn);
#else
#pragma unroll(EST == 0 ? kStepUnrollCond : kStepUnroll)
      for (int st = 0; st < STEPS; ++st) {
        uint32_t w[G::BLOCKS * 4];
#pragma unroll
        for (int b = 0; b < G::BLOCKS; ++b) philox_block_lo(ql + b, c0r1, lo1d, rk.k1[0], rk, &w[4 * b]);
        ql += G::BLOCKS;
        eval_step(w);
      }
#endif
      finish_biased<EST>(SAMPLES_PER_THREAD, a1, a2, cnt);
      if constexpr (EST == 1) a2 = a1;
      return;
    }
  }
#pragma unroll 1
  for (int st = 0; st < STEPS; ++st) {
    const uint64_t s0 = s_begin + (uint64_t)st * G::L;
    if (MASKED && s0 >= E) break;
    uint32_t w[G::BLOCKS * 4];
#pragma unroll
    for (int b = 0; b < G::BLOCKS; ++b) philox_block_rk(q + b, lo1d, hi1d, rk, &w[4 * b]);
    q += G::BLOCKS;
#pragma unroll
    for (int r = 0; r < G::LR; ++r) {
      float u[G::R];
      record_utility<N, EST, false, MODEL>(&w[r * G::WR], one, zc, pr, &sr, u);
#pragma unroll
      for (int h = 0; h < G::R; ++h) {
        if (MASKED) {
          const uint64_t s = s0 + r * G::R + h;
          u[h] = (s >= B && s < E) ? u[h] : 0.0f;
        }
        accumulate<EST>(u[h], a1, a2);
      }
    }
  }
  if constexpr (EST == 1) a2 = a1;
}

// Work unit = one WARP tile: (design, 32 x SAMPLES_PER_THREAD consecutive samples).  Warps are
// independent (no block barrier): each reduces its tile with 64-bit shuffles and lane 0 issues one
// 64-bit atomicAdd pair.  Default launch: one tile per warp (a grid_blocks > 0 launch strides over the tiles).
#ifndef MC_MIN_BLOCKS_C4
#define MC_MIN_BLOCKS_C4 4   // C4 strata kernel: 4 resident blocks/SM, -6 % kernel time vs 2 (profiles/r02/tto_c4.jsonl;
#endif                       // round 1's time-to-optimal "anomaly" is host-side jitter: 0.42-1.45 s in both builds)
constexpr int min_blocks(int n, int est, int model) {
  return model == 1 ? MC_MIN_BLOCKS_C4 : (n <= 3 ? (est == 0 ? MIN_BLOCKS_COND : MIN_BLOCKS_IND) : (n <= 5 ? 2 : 1));
}

template <int N, int EST, int MODEL>
__global__ void __launch_bounds__(MAX_BLOCK, min_blocks(N, EST, MODEL)) mc_fused_kernel(
    const float* __restrict__ prob, const float* __restrict__ zc_all, const int32_t* __restrict__ pod, int64_t d0,
    uint64_t B, uint64_t E, uint64_t Balign, int64_t tiles_per_design, int64_t total_tiles, const RoundKeys rk,
    unsigned long long* __restrict__ sums) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  constexpr uint64_t tile_samples = 32ull * SAMPLES_PER_THREAD;
  for (int64_t tile = gw; tile < total_tiles; tile += nw) {
    const int64_t d = d0 + tile / tiles_per_design;
    const int64_t chunk = tile % tiles_per_design;
    const float* rec = prob + (int64_t)__ldg(pod + d) * PROB_STRIDE;
    ProbRegs<N> pr;
    load_problem<N>(rec, pr);
    StrataRegs sr;
    if constexpr (MODEL == 1) load_strata(rec, sr);
    float zc[N];
#pragma unroll
    for (int i = 0; i < N; ++i) zc[i] = __ldg(zc_all + d * N + i);
    const uint32_t dd = (uint32_t)d;
    const uint32_t lo1d = 0xCD9E8D57u * dd, hi1d = __umulhi(0xCD9E8D57u, dd);
    const uint64_t s_begin = Balign + (uint64_t)chunk * tile_samples + (uint64_t)lane * SAMPLES_PER_THREAD;
    uint32_t a1 = 0, a2 = 0;
    if (s_begin >= B && s_begin + SAMPLES_PER_THREAD <= E)
      run_samples<N, EST, false, MODEL>(s_begin, B, E, lo1d, hi1d, rk, zc, pr, sr, a1, a2);
    else if (s_begin < E)
      run_samples<N, EST, true, MODEL>(s_begin, B, E, lo1d, hi1d, rk, zc, pr, sr, a1, a2);
    unsigned long long v1 = a1, v2 = a2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v1 += __shfl_xor_sync(0xffffffffu, v1, o);
      v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    }
    if (lane == 0) {
      atomicAdd(sums + 2 * d, v1);
      atomicAdd(sums + 2 * d + 1, v2);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// NEXT f3: common random numbers.  The stream is keyed (problem, sample) with tag 1 (counter
// (q_lo, q_hi, problem, 1)); every design of the problem sees the same draws, so the design-
// independent part of a draw (Philox, Box-Muller, the prior term, the IND null vector, the SOV
// uniforms) is computed once and reused for a block of CRN_KD designs held in registers.
// designs per CRN warp tile and min resident blocks (measured on B200, tools/tune_crn.sh): COND 16 / 1 (packed FP32 design pairs: 3.65e11/s vs 3.60e11 with 12, 3.45e11 with 8; scalar 12: 3.34e11),
// IND 32 / 1 (IND: one shared y = X + v per sample, 3 compares + 1 predicated FADD per design: 2.74e12/s)
#ifndef MC_CRN_KD_COND
#define MC_CRN_KD_COND 16
#endif
#ifndef MC_CRN_KD_IND
#define MC_CRN_KD_IND 32
#endif
#ifndef MC_CRN_MINB_COND
#define MC_CRN_MINB_COND 1
#endif
#ifndef MC_CRN_MINB_IND
#define MC_CRN_MINB_IND 1
#endif
template <int EST> constexpr int crn_kd() { return EST == 0 ? MC_CRN_KD_COND : MC_CRN_KD_IND; }

template <int N, int EST, int MODEL, bool MASKED, int KD>
__device__ __forceinline__ void crn_samples(uint64_t s_begin, uint64_t B, uint64_t E, uint32_t pid, const RoundKeys& rk,
                                            const float (&zc)[KD][N], const ProbRegs<N>& pr, const StrataRegs& sr,
                                            uint32_t (&a1)[KD], uint32_t (&a2)[KD]) {
  using G = Geo<N, EST, MODEL>;
  constexpr int STEPS = SAMPLES_PER_THREAD / G::L;
  const uint32_t one = one_bits_reg();
  const uint32_t lo1d = 0xCD9E8D57u * pid, hi1d = __umulhi(0xCD9E8D57u, pid);
  uint64_t q = G::word_of(s_begin) / 4;
  const uint32_t k1r1 = rk.k1[0] ^ 1u;   // counter word 3 = tag 1
  float cf[EST == 1 ? KD : 1];            // IND steady state: fp32 counts per design
#pragma unroll
  for (int k = 0; k < (EST == 1 ? KD : 1); ++k) cf[k] = 0.0f;
#pragma unroll 1
  for (int st = 0; st < STEPS; ++st) {
    const uint64_t s0 = s_begin + (uint64_t)st * G::L;
    if (MASKED && s0 >= E) break;
    uint32_t w[G::BLOCKS * 4];
#pragma unroll
    for (int b = 0; b < G::BLOCKS; ++b) {
      const uint64_t qb = q + b;
      philox_block_lo((uint32_t)qb, hi1d ^ (uint32_t)(qb >> 32) ^ rk.k0[0], lo1d, k1r1, rk, &w[4 * b]);
    }
    q += G::BLOCKS;
#pragma unroll
    for (int r = 0; r < G::LR; ++r) {
      const uint32_t* wr = &w[r * G::WR];
      float nrm[2 * G::NPAIR];
      record_normals<N, EST, MODEL>(wr, one, nrm);
#pragma unroll
      for (int h = 0; h < G::R; ++h) {
        Shared<N, EST, MODEL> sh;
        shared_of_sample<N, EST, MODEL>(nrm, wr, h, one, pr, &sr, sh);
        bool valid = true;
        if (MASKED) {
          const uint64_t s = s0 + r * G::R + h;
          valid = s >= B && s < E;
        }
        if constexpr (EST == 1 && !MASKED && MODEL == 0) {
          // IND, steady state: X_i > zc_i - v_i  <=>  X_i + v_i > zc_i; y = X + v is shared by the KD designs,
          // so each (design, sample) costs n compares in one predicate chain and one predicated FADD
          float y[N];
#pragma unroll
          for (int i = 0; i < N; ++i) y[i] = sh.x[i] + sh.v[i];
#pragma unroll
          for (int k = 0; k < KD; ++k) ind_count<N>(y, zc[k], cf[k]);
        } else if constexpr (EST == 0 && MC_F32X2 && KD % 2 == 0) {
          // COND: two designs of the block per packed lane pair (same sample, same SOV uniforms)
          f2x nv[N], vu[G::NE > 0 ? G::NE : 1];
#pragma unroll
          for (int i = 0; i < N; ++i) nv[i] = bc2(-sh.v[i]);
#pragma unroll
          for (int k = 0; k < G::NE; ++k) vu[k] = bc2(sh.vu[k]);
#pragma unroll
          for (int k = 0; k < KD; k += 2) {
            f2x b[N];
#pragma unroll
            for (int i = 0; i < N; ++i) b[i] = add2(pk2(zc[k][i], zc[k + 1][i]), nv[i]);
            float u0, u1;
            up2(utility_cond_x2<N>(b, vu, pr), u0, u1);
            if (MASKED) {
              u0 = valid ? u0 : 0.0f;
              u1 = valid ? u1 : 0.0f;
            }
            accumulate<EST>(u0, a1[k], a2[k]);
            accumulate<EST>(u1, a1[k + 1], a2[k + 1]);
          }
        } else {
#pragma unroll
          for (int k = 0; k < KD; ++k) {
            float b[N];
#pragma unroll
            for (int i = 0; i < N; ++i) b[i] = zc[k][i] - sh.v[i];
            float u = utility_of_b<N, EST, MODEL>(b, sh, pr);
            if (MASKED) u = valid ? u : 0.0f;
            accumulate<EST>(u, a1[k], a2[k]);
          }
        }
      }
    }
  }
  if constexpr (EST == 1 && !MASKED && MODEL == 0)
#pragma unroll
    for (int k = 0; k < KD; ++k) a1[k] += (uint32_t)cf[k] << 23;   // counts <= 128: exact in fp32
  if constexpr (EST == 1)
#pragma unroll
    for (int k = 0; k < KD; ++k) a2[k] = a1[k];
}

// Work unit = warp tile (design block of <= KD designs of one problem, 32 x SAMPLES_PER_THREAD samples).
template <int N, int EST, int MODEL>
__global__ void __launch_bounds__(MAX_BLOCK, EST == 0 ? MC_CRN_MINB_COND : MC_CRN_MINB_IND) mc_crn_kernel(
    const float* __restrict__ prob, const float* __restrict__ zc_all, const int32_t* __restrict__ blk_first,
    const int32_t* __restrict__ blk_count, const int32_t* __restrict__ blk_prob, uint64_t B, uint64_t E,
    uint64_t Balign, int64_t tiles_per_block, int64_t total_tiles, const RoundKeys rk,
    unsigned long long* __restrict__ sums) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  constexpr uint64_t tile_samples = 32ull * SAMPLES_PER_THREAD;
  for (int64_t tile = gw; tile < total_tiles; tile += nw) {
    const int64_t j = tile / tiles_per_block;
    const int64_t chunk = tile % tiles_per_block;
    const int p = __ldg(blk_prob + j);
    const int64_t d0 = __ldg(blk_first + j);
    const int cnt = __ldg(blk_count + j);
    const float* rec = prob + (int64_t)p * PROB_STRIDE;
    ProbRegs<N> pr;
    load_problem<N>(rec, pr);
    StrataRegs sr;
    if constexpr (MODEL == 1) load_strata(rec, sr);
    constexpr int KD = crn_kd<EST>();
    float zc[KD][N];
#pragma unroll
    for (int k = 0; k < KD; ++k)
#pragma unroll
      for (int i = 0; i < N; ++i) zc[k][i] = k < cnt ? __ldg(zc_all + (d0 + k) * N + i) : __int_as_float(0x7f800000);
    const uint64_t s_begin = Balign + (uint64_t)chunk * tile_samples + (uint64_t)lane * SAMPLES_PER_THREAD;
    uint32_t a1[KD], a2[KD];
#pragma unroll
    for (int k = 0; k < KD; ++k) a1[k] = a2[k] = 0u;
    if (s_begin >= B && s_begin + SAMPLES_PER_THREAD <= E)
      crn_samples<N, EST, MODEL, false, KD>(s_begin, B, E, (uint32_t)p, rk, zc, pr, sr, a1, a2);
    else if (s_begin < E)
      crn_samples<N, EST, MODEL, true, KD>(s_begin, B, E, (uint32_t)p, rk, zc, pr, sr, a1, a2);
#pragma unroll
    for (int k = 0; k < KD; ++k) {
      unsigned long long v1 = a1[k], v2 = a2[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        v2 += __shfl_xor_sync(0xffffffffu, v2, o);
      }
      if (lane == 0 && k < cnt) {
        atomicAdd(sums + 2 * (d0 + k), v1);
        atomicAdd(sums + 2 * (d0 + k) + 1, v2);
      }
    }
  }
}

template <int N, int EST, int MODEL = 0>
static cudaError_t launch_crn_t(mc_ctx* c, int64_t d0, int64_t dcount, uint64_t B, uint64_t E, cudaStream_t st,
                                int64_t* sums) {
  using G = Geo<N, EST, MODEL>;
  // design blocks of <= CRN_KD consecutive designs that never straddle a problem (cached per range)
  constexpr int KD = crn_kd<EST>();
  if (c->crn_d0 != d0 || c->crn_dc != dcount || c->crn_kd != KD || !c->d_crn) {
    std::vector<int32_t> first, count, pb;
    for (int k = 0; k < c->n_probs; ++k) {
      const int64_t b = std::max<int64_t>(c->prob_begin[k], d0), e = std::min<int64_t>(c->prob_begin[k + 1], d0 + dcount);
      for (int64_t x = b; x < e; x += KD) {
        first.push_back((int32_t)x);
        count.push_back((int32_t)std::min<int64_t>(KD, e - x));
        pb.push_back(k);
      }
    }
    cudaFree(c->d_crn);
    c->d_crn = nullptr;
    c->crn_blocks = (int64_t)first.size();
    if (c->crn_blocks == 0) return cudaSuccess;
    cudaError_t e = cudaMalloc(&c->d_crn, sizeof(int32_t) * 3 * c->crn_blocks);
    if (e != cudaSuccess) return e;
    std::vector<int32_t> all(first);
    all.insert(all.end(), count.begin(), count.end());
    all.insert(all.end(), pb.begin(), pb.end());
    e = cudaMemcpy(c->d_crn, all.data(), sizeof(int32_t) * all.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    c->crn_d0 = d0;
    c->crn_dc = dcount;
    c->crn_kd = KD;
  }
  const int threads = c->block_threads;
  const uint64_t tile = 32ull * SAMPLES_PER_THREAD;
  const uint64_t Balign = B - (B % G::L);
  const int64_t tpb = (int64_t)((E - Balign + tile - 1) / tile);
  const int64_t total = tpb * c->crn_blocks;
  // one warp tile per warp by default, as for the fused kernel (+2.5% measured over a persistent grid)
  const int64_t wpb = threads / 32;
  int64_t grid64 = c->grid_blocks > 0 ? c->grid_blocks : (total + wpb - 1) / wpb;
  if (grid64 * wpb > total) grid64 = (total + wpb - 1) / wpb;
  const int grid = (int)std::min<int64_t>(grid64, 0x7FFFFFFF);
  if (grid <= 0) return cudaSuccess;
  const int32_t* bf = c->d_crn;
  mc_crn_kernel<N, EST, MODEL><<<grid, threads, 0, st>>>(c->d_prob, c->d_zc, bf, bf + c->crn_blocks,
                                                         bf + 2 * c->crn_blocks, B, E, Balign, tpb, total,
                                                         round_keys(c->seed), reinterpret_cast<unsigned long long*>(sums));
  c->launches += 1;
  return cudaGetLastError();
}

template <int N, int EST, int MODEL = 0>
static cudaError_t launch_fused_t(mc_ctx* c, int64_t d0, int64_t dcount, uint64_t B, uint64_t E, cudaStream_t st,
                                  int64_t* sums) {
  using G = Geo<N, EST, MODEL>;
  const int threads = c->block_threads;
  const uint64_t tile = 32ull * SAMPLES_PER_THREAD;   // one warp tile
  const uint64_t Balign = B - (B % G::L);
  const int64_t tpd = (int64_t)((E - Balign + tile - 1) / tile);
  const int64_t total = tpd * dcount;
  // default: one warp tile per warp and the hardware block scheduler balances the load (tiles differ
  // in cost: partial last tiles, the rare inverse-CDF tail); measured +5.6% over a persistent grid of
  // #SMs x resident blocks with static striding (profiles/r01/tune_grid.txt).  grid_blocks > 0 gives a
  // persistent grid that strides over the tiles.
  const int64_t warps_needed = total, wpb = threads / 32;
  int64_t grid64 = c->grid_blocks > 0 ? c->grid_blocks : (warps_needed + wpb - 1) / wpb;
  if (grid64 * wpb > warps_needed) grid64 = (warps_needed + wpb - 1) / wpb;
  const int grid = (int)std::min<int64_t>(grid64, 0x7FFFFFFF);
  if (grid <= 0) return cudaSuccess;
  mc_fused_kernel<N, EST, MODEL><<<grid, threads, 0, st>>>(c->d_prob, c->d_zc, c->d_pod, d0, B, E, Balign, tpd,
                                                           total, round_keys(c->seed),
                                                           reinterpret_cast<unsigned long long*>(sums));
  c->launches += 1;
  return cudaGetLastError();
}

#define MC_DISPATCH_N(FN, ...)                                                  \
  switch (c->n) {                                                               \
    case 1: e = FN<1, EST>(__VA_ARGS__); break;                                 \
    case 2: e = FN<2, EST>(__VA_ARGS__); break;                                 \
    case 3: e = FN<3, EST>(__VA_ARGS__); break;                                 \
    case 4: e = FN<4, EST>(__VA_ARGS__); break;                                 \
    case 5: e = FN<5, EST>(__VA_ARGS__); break;                                 \
    case 6: e = FN<6, EST>(__VA_ARGS__); break;                                 \
    case 7: e = FN<7, EST>(__VA_ARGS__); break;                                 \
    case 8: e = FN<8, EST>(__VA_ARGS__); break;                                 \
    case 9: e = FN<9, EST>(__VA_ARGS__); break;                                 \
    case 10: e = FN<10, EST>(__VA_ARGS__); break;                               \
    default: set_error("n out of range"); return MC_ERR_INVALID;                \
  }

template <int EST>
static mc_status launch_fused_est(mc_ctx* c, int64_t d0, int64_t dcount, uint64_t B, uint64_t E, cudaStream_t st,
                                  int64_t* sums) {
  cudaError_t e = cudaSuccess;
  if (c->sampling == 1) {
    if (c->model == 1) e = launch_crn_t<2, EST, 1>(c, d0, dcount, B, E, st, sums);
    else if (c->n == 1) e = launch_crn_t<1, EST>(c, d0, dcount, B, E, st, sums);
    else if (c->n == 2) e = launch_crn_t<2, EST>(c, d0, dcount, B, E, st, sums);
    else if (c->n == 3) e = launch_crn_t<3, EST>(c, d0, dcount, B, E, st, sums);
    else { set_error("common random numbers are built for n <= 3"); return MC_ERR_INVALID; }
    if (e != cudaSuccess) return cuda_fail(e, "mc_crn_kernel launch");
    return MC_OK;
  }
  if (c->model == 1) {
    e = launch_fused_t<2, EST, 1>(c, d0, dcount, B, E, st, sums);
    if (e != cudaSuccess) return cuda_fail(e, "mc_fused_kernel launch");
    return MC_OK;
  }
  MC_DISPATCH_N(launch_fused_t, c, d0, dcount, B, E, st, sums);
  if (e != cudaSuccess) return cuda_fail(e, "mc_fused_kernel launch");
  return MC_OK;
}

mc_status launch_fused(mc_ctx* c, int64_t d0, int64_t dcount, uint64_t B, uint64_t E, cudaStream_t st, int64_t* sums) {
  if (dcount <= 0 || E <= B) return MC_OK;
  return c->est == 0 ? launch_fused_est<0>(c, d0, dcount, B, E, st, sums)
                     : launch_fused_est<1>(c, d0, dcount, B, E, st, sums);
}

int words_per_record(int n, int est, int model) {
  // Geo<N,EST,MODEL>::WR without instantiating every N: U 23-bit uniforms in 2 ceil(23 U / 64) words if
  // that is fewer than U, else one word each
  const int p = model == 1 ? 5 : n;
  const int U = est == 0 ? 2 * p + 2 * (n / 2) : 4 * ((p + n + 1) / 2);
  const int W = 2 * ((23 * U + 63) / 64);
  return W < U ? W : U;
}
int draw_dump_stride(int n, int est, int model) {
  const int p = model == 1 ? 5 : n;
  return (est == 0 ? p : p + n) + n + 1;
}

// ---------------------------------------------------------------------------------------------
// Design thresholds (row a1): zc_i = Z_{1-alpha_i} - c_i theta_i in fp64 -> fp32; alpha = 0 -> +inf.
__global__ void k_zc(const double* __restrict__ alpha, const int32_t* __restrict__ pod, const double* __restrict__ ctheta,
                     int n, int64_t D, float* __restrict__ zc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= D * n) return;
  const int64_t d = t / n;
  const int i = (int)(t % n);
  const double a = alpha[t];
  const double z = a <= 0.0 ? CUDART_INF : -normcdfinv(a);   // Z_{1-a} = -Phi^{-1}(a)
  const double* ct = ctheta + ((int64_t)pod[d] * n + i) * 2;  // (c_i theta_i, row scale)
  zc[t] = (float)((z - ct[0]) * ct[1]);
}

mc_status launch_zc(mc_ctx* c, cudaStream_t st) {
  const int64_t T = c->D * c->n;
  if (T == 0) return MC_OK;
  k_zc<<<(unsigned)((T + 255) / 256), 256, 0, st>>>(c->d_alpha, c->d_pod, c->d_ctheta, c->n, c->D, c->d_zc);
  c->launches += 1;
  MC_CUDA(cudaGetLastError());
  return MC_OK;
}

// ---------------------------------------------------------------------------------------------
// K2: finalize (row a8), fp64.
__global__ void k_finalize(const long long* __restrict__ sums, int64_t D, double N, double* __restrict__ mean,
                           double* __restrict__ var) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= D) return;
  const double scale = 1.0 / (N * 8388608.0);
  const double m = (double)sums[2 * d] * scale;
  const double m2 = (double)sums[2 * d + 1] * scale;
  mean[d] = m;
  if (var) var[d] = N > 1.0 ? (m2 - m * m) * N / (N - 1.0) : 0.0;
}

mc_status launch_finalize(mc_ctx* c, const int64_t* sums, uint64_t N, double* mean, double* var, cudaStream_t st) {
  if (c->D == 0) return MC_OK;
  const int threads = 256;
  const int64_t blocks = (c->D + threads - 1) / threads;
  k_finalize<<<(unsigned)blocks, threads, 0, st>>>(reinterpret_cast<const long long*>(sums), c->D, (double)N, mean, var);
  c->launches += 1;
  MC_CUDA(cudaGetLastError());
  return MC_OK;
}

// ---------------------------------------------------------------------------------------------
// K3: Philox words (test hook) in the forms the kernels generate them.  Word w of stream (id, tag) is
// lane w mod 4 of the block with counter (q_lo, q_hi, id, tag), q = w / 4, key (seed_lo, seed_hi):
//   form 0: philox_block_lo — the fused and CRN kernels' steady state (round keys from the constant
//           bank, round 1 with the design product hoisted and c0 = hi(M1 id) ^ q_hi ^ k0 held fixed);
//   form 1: philox_block_rk — the fused kernel's masked (partial-tile / counter-wrap) path (tag 0 only);
//   form 2: philox_word_tagged — the plain 10-round form of the crossed kernel.
__device__ __forceinline__ uint32_t word_form(uint64_t seed, const RoundKeys& rk, uint32_t id, uint32_t tag, int form,
                                              uint64_t w) {
  const uint64_t q = w >> 2;
  const uint32_t lo1d = 0xCD9E8D57u * id, hi1d = __umulhi(0xCD9E8D57u, id);
  uint32_t o[4];
  if (form == 0)
    philox_block_lo((uint32_t)q, hi1d ^ (uint32_t)(q >> 32) ^ rk.k0[0], lo1d, rk.k1[0] ^ tag, rk, o);
  else if (form == 1)
    philox_block_rk(q, lo1d, hi1d, rk, o);
  else
    return philox_word_tagged(seed, id, tag, w);
  return o[w & 3];
}

__global__ void k_philox_dump(uint64_t seed, const RoundKeys rk, uint32_t tag, int form, const uint32_t* __restrict__ id,
                              const uint64_t* __restrict__ word, int64_t count, uint32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < count) out[i] = word_form(seed, rk, id[i], tag, form, word[i]);
}

mc_status launch_philox_dump(uint64_t seed, uint32_t tag, int form, const uint32_t* id, const uint64_t* word,
                             int64_t count, uint32_t* out, cudaStream_t st) {
  if (form < 0 || form > 2 || (form == 1 && tag != 0)) {
    set_error("mc_philox_dump: form must be 0, 1 (tag 0 only) or 2");
    return MC_ERR_INVALID;
  }
  if (count <= 0) return MC_OK;
  k_philox_dump<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(seed, round_keys(seed), tag, form, id, word, count, out);
  MC_CUDA(cudaGetLastError());
  return MC_OK;
}

// Per-draw dump through the fused kernel's record_utility (test hook): the words of the sample's record
// in the steady-state form (philox_block_lo), then the same record code as K1 (COND: the packed pair).
template <int N, int EST, int MODEL, bool CRN>
__global__ void k_draw_dump(const float* __restrict__ prob, const float* __restrict__ zc_all,
                            const int32_t* __restrict__ pod, uint64_t seed, const RoundKeys rk,
                            const int64_t* __restrict__ design, const uint64_t* __restrict__ sample, int64_t count,
                            float* __restrict__ out) {
  using G = Geo<N, EST, MODEL>;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int64_t d = design[i];
  ProbRegs<N> pr;
  load_problem<N>(prob + (int64_t)pod[d] * PROB_STRIDE, pr);
  StrataRegs sr;
  if constexpr (MODEL == 1) load_strata(prob + (int64_t)pod[d] * PROB_STRIDE, sr);
  float zc[N];
  for (int k = 0; k < N; ++k) zc[k] = zc_all[d * N + k];
  // the whole record of the sample, then its half h
  uint32_t w[G::WR];
  const uint64_t base = G::word_of(sample[i] - sample[i] % G::R);
  const int h = (int)(sample[i] % G::R);
  for (int k = 0; k < G::WR; ++k)
    w[k] = word_form(seed, rk, CRN ? (uint32_t)pod[d] : (uint32_t)d, CRN ? 1u : 0u, 0, base + k);
  float bsc[N];
  for (int k = 0; k < N; ++k) bsc[k] = prob[(int64_t)pod[d] * PROB_STRIDE + OFF_BSC + k];
  float u[G::R], dbg[G::R * G::DUMP];
  record_utility<N, EST, true, MODEL>(w, one_bits_reg(), zc, pr, &sr, u, dbg, bsc);
  for (int k = 0; k < G::DUMP; ++k) out[i * G::DUMP + k] = dbg[h * G::DUMP + k];
}

template <int N, int EST, int MODEL = 0>
static cudaError_t launch_dump_t(mc_ctx* c, const int64_t* design, const uint64_t* sample, int64_t count, float* out,
                                 cudaStream_t st) {
  const RoundKeys rk = round_keys(c->seed);
  if (c->sampling == 1)
    k_draw_dump<N, EST, MODEL, true><<<(unsigned)((count + 127) / 128), 128, 0, st>>>(
        c->d_prob, c->d_zc, c->d_pod, c->seed, rk, design, sample, count, out);
  else
    k_draw_dump<N, EST, MODEL, false><<<(unsigned)((count + 127) / 128), 128, 0, st>>>(
        c->d_prob, c->d_zc, c->d_pod, c->seed, rk, design, sample, count, out);
  return cudaGetLastError();
}

template <int EST>
static mc_status launch_dump_est(mc_ctx* c, const int64_t* design, const uint64_t* sample, int64_t count, float* out,
                                 cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  if (c->model == 1) {
    e = launch_dump_t<2, EST, 1>(c, design, sample, count, out, st);
    if (e != cudaSuccess) return cuda_fail(e, "k_draw_dump launch");
    return MC_OK;
  }
  MC_DISPATCH_N(launch_dump_t, c, design, sample, count, out, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_draw_dump launch");
  return MC_OK;
}

mc_status launch_draw_dump(mc_ctx* c, const int64_t* design, const uint64_t* sample, int64_t count, float* out,
                           cudaStream_t st) {
  if (count <= 0) return MC_OK;
  return c->est == 0 ? launch_dump_est<0>(c, design, sample, count, out, st)
                     : launch_dump_est<1>(c, design, sample, count, out, st);
}

// ---------------------------------------------------------------------------------------------
// K6: segmented argmax (row a10): one block per problem, lexicographic (max value, min index).
__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi) {
  if (v != v) return false;                 // NaN never wins
  if (bv != bv) return true;
  return v > bv || (v == bv && i < bi);
}

__global__ void k_segmented_argmax(const double* __restrict__ values, const int64_t* __restrict__ begin,
                                   int64_t* __restrict__ idx, double* __restrict__ val) {
  __shared__ double sv[32];
  __shared__ long long si[32];
  const int p = blockIdx.x;
  const int64_t b = begin[p], e = begin[p + 1];
  double bv = __longlong_as_double(0xFFF8000000000000ull);   // NaN = empty
  int64_t bi = -1;
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
    const double v = values[i];
    if (better(v, i, bv, bi)) { bv = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, (long long)bi, o);
    if (oi >= 0 && (bi < 0 || better(ov, oi, bv, bi))) { bv = ov; bi = oi; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sv[warp] = bv; si[warp] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (si[k] >= 0 && (bi < 0 || better(sv[k], si[k], bv, bi))) { bv = sv[k]; bi = si[k]; }
    idx[p] = bi;
    val[p] = bv;
  }
}

mc_status launch_argmax(mc_ctx* c, const double* values, int64_t* idx, double* val, cudaStream_t st) {
  if (c->n_probs == 0) return MC_OK;
  k_segmented_argmax<<<c->n_probs, 256, 0, st>>>(values, c->d_prob_begin, idx, val);
  c->launches += 1;
  MC_CUDA(cudaGetLastError());
  return MC_OK;
}

}  // namespace mci
