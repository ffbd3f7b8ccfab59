// Pipe-rate microbenchmark for sm_100a.
// Measures sustained lane-ops/s of the pipes the Monte-Carlo kernel uses
// (FFMA, FMUL-imm, IMAD.WIDE.U32, LOP3, IADD3, MUFU.{EX2,LG2,RCP,SIN,RSQ,SQRT}, I2F)
// and the SM clock seen under that load (clock64 cycles / globaltimer ns).
// Output: one JSON object on stdout; bench/DESIGN use it for the ALU roofline.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

template <int OP>
__global__ void __launch_bounds__(256) pipe_kernel(float* out, uint64_t* clk, float seed) {
  float f[CH]; uint32_t u[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { f[c] = seed + threadIdx.x * 1e-3f + c; u[c] = threadIdx.x * 2654435761u + c; }
  uint64_t c0 = clock64(), t0 = gtime();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (OP == 0) { f[c] = fmaf(f[c], f[(c + 1) % CH], 0.999f * f[(c+2)%CH]); }                 // FFMA 3-reg
        else if (OP == 1) { f[c] = fmaf(f[c], 0.9999f, 0.5f); }                                      // FFMA imm
        else if (OP == 2) { uint64_t w = (uint64_t)u[c] * 0xD2511F53u; u[c] = (uint32_t)(w >> 32) ^ (uint32_t)w; } // IMAD.WIDE + LOP3
        else if (OP == 3) { u[c] = u[c] ^ u[(c + 1) % CH] ^ 0x9E3779B9u; }                           // LOP3
        else if (OP == 4) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[c])); }              // MUFU.EX2
        else if (OP == 5) { asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(f[c])); }              // MUFU.LG2
        else if (OP == 6) { float t = f[c] + 1.0f; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(f[c]) : "f"(t)); } // MUFU.RCP (+FADD)
        else if (OP == 7) { asm volatile("sin.approx.ftz.f32 %0, %0;" : "+f"(f[c])); }              // MUFU.SIN
        else if (OP == 8) { asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(f[c])); }            // MUFU.RSQ
        else if (OP == 9) { asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(f[c])); }             // MUFU.SQRT
        else if (OP == 10) { f[c] = __uint_as_float((u[c] & 0x007FFFFFu) | 0x3F800000u) + f[c]; u[c] += 0x01000193u; } // LOP3+FADD+IADD
        else if (OP == 11) { f[c] = f[c] + (float)(u[c] >> 9); u[c] += 7u; }                        // I2F path
        else if (OP == 12) { u[c] = u[c] + u[(c + 1) % CH] + 0x9E3779B9u; }                          // IADD3
        else if (OP == 13) { uint32_t lo = u[c] * 0xCD9E8D57u; uint32_t hi = __umulhi(u[c], 0xCD9E8D57u); u[c] = hi ^ lo ^ 0x1234u; } // mul.hi + mul.lo
      }
    }
  }
  uint64_t c1 = clock64(), t1 = gtime();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += f[c] + (float)u[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
}

template <int OP>
int run(const char* name, int nsm, float* out, uint64_t* clk, bool last) {
  int bps = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, pipe_kernel<OP>, 256, 0));
  int grid = nsm * bps;
  pipe_kernel<OP><<<grid, 256>>>(out, clk, 1.0f);  // warm
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  pipe_kernel<OP><<<grid, 256>>>(out, clk, 1.0f);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  uint64_t h[2]; CK(cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost));
  double ops = (double)grid * 256 * ITERS * 8 * CH;  // inner ops (one "op" per chain update)
  double mhz = (double)h[0] / (double)h[1] * 1e3;
  printf("  \"%s\": {\"ops_per_s\": %.4e, \"ops_per_clk_per_sm\": %.2f, \"sm_mhz\": %.0f, \"blocks_per_sm\": %d, \"ms\": %.3f}%s\n",
         name, ops / (ms * 1e-3), ops / (ms * 1e-3) / (mhz * 1e6) / nsm, mhz, bps, ms, last ? "" : ",");
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int nsm = p.multiProcessorCount;
  float* out; uint64_t* clk;
  CK(cudaMalloc(&out, sizeof(float) * nsm * 32 * 256));
  CK(cudaMalloc(&clk, 16));
  printf("{\n  \"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\",\n", p.name, nsm, p.major, p.minor);
  run<0>("ffma_3reg", nsm, out, clk, false);
  run<1>("ffma_imm", nsm, out, clk, false);
  run<2>("imad_wide_plus_lop3", nsm, out, clk, false);
  run<3>("lop3", nsm, out, clk, false);
  run<4>("mufu_ex2", nsm, out, clk, false);
  run<5>("mufu_lg2", nsm, out, clk, false);
  run<6>("mufu_rcp", nsm, out, clk, false);
  run<7>("mufu_sin", nsm, out, clk, false);
  run<8>("mufu_rsq", nsm, out, clk, false);
  run<9>("mufu_sqrt", nsm, out, clk, false);
  run<10>("lop3_fadd_iadd", nsm, out, clk, false);
  run<11>("shr_i2f_fadd_iadd", nsm, out, clk, false);
  run<12>("iadd3", nsm, out, clk, false);
  run<13>("mulhi_mullo_lop3", nsm, out, clk, true);
  printf("}\n");
  return 0;
}
