// pipemix.cu — issue/pipe model of the fused K1 kernel's instruction mix on sm_100a (round 2).
//
// Measures warp-instructions per clock per SM for single instruction classes and for fixed mixes
// (independent chains, 8 per thread, 8 warps per block, max resident blocks), so the per-draw demand
// model of DESIGN.md §4 can name the binding pipe:
//   FFMA2 (fma.rn.f32x2), FFMA (scalar, immediate), IMAD.WIDE.U32 (64-bit accumulate), LOP3, MUFU.EX2,
//   and the pairs FFMA2+IMAD.WIDE, FFMA2+MUFU, IMAD.WIDE+MUFU, IMAD.WIDE+LOP3, FFMA+IMAD.WIDE.
// Output: one JSON object; "wi_per_clk_sm" counts warp-instructions of every class in the mix.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 2048;
constexpr int CH = 8;

__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__device__ __forceinline__ void op_ffma2(unsigned long long& x) {
  asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(0x3F7FF0003F7FF000ull), "l"(0x3F0000003F000000ull));
}
__device__ __forceinline__ void op_ffma(float& x) { asm volatile("fma.rn.f32 %0, %0, 0f3F7FF000, 0f3F000000;" : "+f"(x)); }
__device__ __forceinline__ void op_imadw(unsigned long long& x) {
  asm volatile("{ .reg .u32 lo, hi; mov.b64 {lo, hi}, %0; xor.b32 lo, lo, hi; mul.wide.u32 %0, lo, 0xD2511F53; }" : "+l"(x));
}
__device__ __forceinline__ void op_lop3(uint32_t& x, uint32_t y) {
  asm volatile("lop3.b32 %0, %0, %1, 0x9E3779B9, 0x96;" : "+r"(x) : "r"(y));
}
__device__ __forceinline__ void op_ex2(float& x) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x)); }
__device__ __forceinline__ void op_ffma_r(float& x, float y, float z) { asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(y), "f"(z)); }
__device__ __forceinline__ void op_imad(uint32_t& x, uint32_t y) { asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(x) : "r"(y)); }
__device__ __forceinline__ void op_fmul2(unsigned long long& x) { asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(0x3F7FF0003F7FF000ull)); }
__device__ __forceinline__ void op_fadd2(unsigned long long& x) { asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(0x3F7FF0003F7FF000ull)); }
__device__ __forceinline__ void op_dfma(double& x, double y) { asm volatile("fma.rn.f64 %0, %0, %1, 0d3FE0000000000000;" : "+d"(x) : "d"(y)); }
__device__ __forceinline__ void op_f2d(double& x, float& y) { asm volatile("{ .reg .f64 t; cvt.f64.f32 t, %1; add.f64 %0, %0, t; }" : "+d"(x) : "f"(y)); }
__device__ __forceinline__ void op_d2f(float& y, double x) { asm volatile("{ .reg .f32 t; cvt.rn.f32.f64 t, %1; add.f32 %0, %0, t; }" : "+f"(y) : "d"(x)); }
__device__ __forceinline__ void op_cvt_fd(float& y) { asm volatile("{ .reg .f64 t; cvt.f64.f32 t, %0; cvt.rn.f32.f64 %0, t; }" : "+f"(y)); }
__device__ __forceinline__ void op_fmnmx(float& x, float y) { asm volatile("min.f32 %0, %0, %1;" : "+f"(x) : "f"(y)); }

// MIX selects the per-chain body; counts[] = warp-instructions per chain per body of each class
template <int MIX>
__global__ void __launch_bounds__(256) mix_kernel(float* out, uint64_t* clk) {
  unsigned long long a[CH], b[CH];
  double dd[CH];
  float f[CH], g[CH];
  uint32_t u[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    a[c] = 0x3F8000003F800000ull + threadIdx.x + c; b[c] = threadIdx.x * 77ull + c;
    dd[c] = 0.5 + c * 1e-3 + threadIdx.x * 1e-7;
    f[c] = 1.0f + c * 1e-3f + threadIdx.x * 1e-6f; g[c] = 0.5f + c * 1e-3f + threadIdx.x * 1e-7f; u[c] = threadIdx.x * 2654435761u + c;
  }
  uint64_t c0 = clock64(), t0 = gtime();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MIX == 0) { op_ffma2(a[c]); op_ffma2(a[c]); }
      else if (MIX == 1) { op_ffma(f[c]); op_ffma(f[c]); }
      else if (MIX == 2) { op_imadw(b[c]); op_imadw(b[c]); }
      else if (MIX == 3) { op_lop3(u[c], u[(c + 1) % CH]); op_lop3(u[c], u[(c + 2) % CH]); }
      else if (MIX == 4) { op_ex2(f[c]); op_ex2(g[c]); }
      else if (MIX == 5) { op_ffma2(a[c]); op_imadw(b[c]); }                         // 1:1
      else if (MIX == 6) { op_ffma2(a[c]); op_ffma2(a[c]); op_ffma2(a[c]); op_ex2(f[c]); }   // 3:1
      else if (MIX == 7) { op_imadw(b[c]); op_ex2(f[c]); }                           // 1:1
      else if (MIX == 8) { op_imadw(b[c]); op_lop3(u[c], u[(c + 1) % CH]); }       // 1:1
      else if (MIX == 9) { op_ffma(f[c]); op_imadw(b[c]); }                          // 1:1
      else if (MIX == 10) { op_ffma2(a[c]); op_lop3(u[c], u[(c + 1) % CH]); }      // 1:1
      else if (MIX == 11) { op_ex2(f[c]); op_lop3(u[c], u[(c + 1) % CH]); }        // 1:1
      else if (MIX == 12) { op_ffma2(a[c]); op_ffma2(a[c]); op_imadw(b[c]); op_lop3(u[c], u[(c + 1) % CH]); }  // 2:1:1
      else if (MIX == 13) { op_ffma2(a[c]); op_imadw(b[c]); op_ex2(f[c]); op_lop3(u[c], u[(c + 1) % CH]); }   // 1:1:1:1
      else if (MIX == 14) { op_ffma_r(f[c], g[c], g[(c + 1) % CH]); op_ffma_r(f[c], g[(c + 2) % CH], g[c]); }
      else if (MIX == 15) { op_imad(u[c], u[(c + 1) % CH]); op_imad(u[c], u[(c + 3) % CH]); }
      else if (MIX == 16) { op_fmul2(a[c]); op_fmul2(a[c]); }
      else if (MIX == 17) { op_fadd2(a[c]); op_fadd2(a[c]); }
      else if (MIX == 18) { op_ffma2(a[c]); op_ffma_r(f[c], g[c], g[(c + 1) % CH]); }       // 1:1
      else if (MIX == 19) { op_ffma_r(f[c], g[c], g[(c + 1) % CH]); op_imadw(b[c]); }      // 1:1
      else if (MIX == 20) { op_ffma2(a[c]); op_imad(u[c], u[(c + 1) % CH]); }                               // 1:1
      else if (MIX == 21) { op_imadw(b[c]); op_imad(u[c], u[(c + 1) % CH]); }                               // 1:1
      else if (MIX == 22) { op_fmnmx(f[c], f[(c + 1) % CH]); op_fmnmx(g[c], f[(c + 2) % CH]); }
      else if (MIX == 23) { op_ffma2(a[c]); op_ffma2(a[c]); op_imadw(b[c]); }             // 2:1
      else if (MIX == 24) { op_dfma(dd[c], dd[(c + 1) % CH]); op_dfma(dd[c], dd[(c + 2) % CH]); }
      else if (MIX == 25) { op_dfma(dd[c], dd[(c + 1) % CH]); op_ffma2(a[c]); }                // 1:1
      else if (MIX == 26) { op_dfma(dd[c], dd[(c + 1) % CH]); op_imadw(b[c]); }                // 1:1
      else if (MIX == 27) { op_cvt_fd(f[c]); }                                                   // F2F x2
      else if (MIX == 28) { op_dfma(dd[c], dd[(c + 1) % CH]); op_lop3(u[c], u[(c + 1) % CH]); }  // 1:1
    }
  }
  uint64_t c1 = clock64(), t1 = gtime();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += (float)dd[c] + f[c] + g[c] + (float)u[c] + (float)(a[c] ^ (a[c] >> 32)) + (float)(b[c] ^ (b[c] >> 29));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
}

template <int MIX>
int run(const char* name, int per_body, int nsm, float* out, uint64_t* clk, bool last) {
  int bps = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, mix_kernel<MIX>, 256, 0));
  const int grid = nsm * bps;
  mix_kernel<MIX><<<grid, 256>>>(out, clk);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix_kernel<MIX><<<grid, 256>>>(out, clk);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  uint64_t h[2]; CK(cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost));
  const double mhz = (double)h[0] / (double)h[1] * 1e3;
  const double winstr = (double)grid * 8 * ITERS * CH * per_body;   // warp-instructions (8 warps/block)
  const double per_clk_sm = winstr / (ms * 1e-3) / (mhz * 1e6) / nsm;
  printf("  \"%s\": {\"wi_per_clk_sm\": %.3f, \"sm_mhz\": %.0f, \"blocks_per_sm\": %d, \"ms\": %.3f}%s\n", name,
         per_clk_sm, mhz, bps, ms, last ? "" : ",");
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  const int nsm = p.multiProcessorCount;
  float* out; uint64_t* clk;
  CK(cudaMalloc(&out, sizeof(float) * nsm * 32 * 256));
  CK(cudaMalloc(&clk, 16));
  printf("{\n  \"gpu\": \"%s\", \"sms\": %d,\n", p.name, nsm);
  run<0>("ffma2", 2, nsm, out, clk, false);
  run<1>("ffma_imm", 2, nsm, out, clk, false);
  run<2>("imad_wide", 2, nsm, out, clk, false);
  run<3>("lop3", 2, nsm, out, clk, false);
  run<4>("mufu_ex2", 2, nsm, out, clk, false);
  run<5>("ffma2+imad_wide_1:1", 2, nsm, out, clk, false);
  run<6>("ffma2+ex2_3:1", 4, nsm, out, clk, false);
  run<7>("imad_wide+ex2_1:1", 2, nsm, out, clk, false);
  run<8>("imad_wide+lop3_1:1", 2, nsm, out, clk, false);
  run<9>("ffma+imad_wide_1:1", 2, nsm, out, clk, false);
  run<10>("ffma2+lop3_1:1", 2, nsm, out, clk, false);
  run<11>("ex2+lop3_1:1", 2, nsm, out, clk, false);
  run<12>("ffma2+imad_wide+lop3_2:1:1", 4, nsm, out, clk, false);
  run<13>("ffma2+imad_wide+ex2+lop3_1:1:1:1", 4, nsm, out, clk, false);
  run<14>("ffma_reg", 2, nsm, out, clk, false);
  run<15>("imad32", 2, nsm, out, clk, false);
  run<16>("fmul2", 2, nsm, out, clk, false);
  run<17>("fadd2", 2, nsm, out, clk, false);
  run<18>("ffma2+ffma_1:1", 2, nsm, out, clk, false);
  run<19>("ffma+imad_wide_1:1(reg)", 2, nsm, out, clk, false);
  run<20>("ffma2+imad32_1:1", 2, nsm, out, clk, false);
  run<21>("imad_wide+imad32_1:1", 2, nsm, out, clk, false);
  run<22>("fmnmx", 2, nsm, out, clk, false);
  run<23>("ffma2+imad_wide_2:1", 3, nsm, out, clk, false);
  run<24>("dfma", 2, nsm, out, clk, false);
  run<25>("dfma+ffma2_1:1", 2, nsm, out, clk, false);
  run<26>("dfma+imad_wide_1:1", 2, nsm, out, clk, false);
  run<27>("f2f_f64_f32+f2f_f32_f64", 2, nsm, out, clk, false);
  run<28>("dfma+lop3_1:1", 2, nsm, out, clk, true);
  printf("}\n");
  return 0;
}
