// imadw_probe.cu — which sm_100a pipe executes IMAD.WIDE.U32 in Philox-like code (round 2 probe).
// Variants of a 64-bit product chain; run under ncu with sm__inst_executed_pipe_fmaheavy.sum etc.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int ITERS = 2048, CH = 8;

template <int V>
__global__ void __launch_bounds__(256) probe(uint32_t* out, uint32_t k) {
  uint32_t lo[CH], hi[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { lo[c] = threadIdx.x * 2654435761u + c; hi[c] = threadIdx.x ^ (c * 77u); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint64_t p;
      if (V == 0) {        // product of the LOW half, both halves used via XOR next step (Philox-like)
        asm volatile("mul.wide.u32 %0, %1, 0xD2511F53;" : "=l"(p) : "r"(lo[c]));
        lo[c] = (uint32_t)p ^ k; hi[c] ^= (uint32_t)(p >> 32);
      } else if (V == 1) { // product of the low half; only the high half used
        asm volatile("mul.wide.u32 %0, %1, 0xD2511F53;" : "=l"(p) : "r"(lo[c]));
        lo[c] = (uint32_t)(p >> 32);
      } else if (V == 2) { // mul.hi + mul.lo
        uint32_t h, l;
        asm volatile("mul.hi.u32 %0, %2, 0xD2511F53; mul.lo.u32 %1, %2, 0xD2511F53;" : "=r"(h), "=r"(l) : "r"(lo[c]));
        lo[c] = l ^ k; hi[c] ^= h;
      } else if (V == 3) { // Philox round on (lo, hi) pairs: c0' = hi(M*c2) ^ c1 ^ k; exactly the kernel pattern
        asm volatile("mul.wide.u32 %0, %1, 0xCD9E8D57;" : "=l"(p) : "r"(lo[c]));
        const uint32_t n0 = (uint32_t)(p >> 32) ^ hi[c] ^ k;
        hi[c] = (uint32_t)p;
        lo[c] = n0;
      } else if (V == 4) { // product with a register multiplier
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(lo[c]), "r"(k));
        lo[c] = (uint32_t)p ^ (uint32_t)(p >> 32);
      } else if (V == 5) { // mad.wide with 64-bit addend
        uint64_t a = ((uint64_t)hi[c] << 32) | lo[c];
        asm volatile("mad.wide.u32 %0, %1, 0xD2511F53, %2;" : "=l"(p) : "r"(lo[c]), "l"(a));
        lo[c] = (uint32_t)p; hi[c] = (uint32_t)(p >> 32);
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += lo[c] ^ hi[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
void run(int nsm, uint32_t* out) {
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, probe<V>, 256, 0);
  probe<V><<<nsm * bps, 256>>>(out, 0x9E3779B9u);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<V><<<nsm * bps, 256>>>(out, 0x9E3779B9u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("variant %d: %.3f ms (%d blocks/SM)\n", V, ms, bps);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  uint32_t* out; cudaMalloc(&out, sizeof(uint32_t) * p.multiProcessorCount * 32 * 256);
  run<0>(p.multiProcessorCount, out); run<1>(p.multiProcessorCount, out); run<2>(p.multiProcessorCount, out);
  run<3>(p.multiProcessorCount, out); run<4>(p.multiProcessorCount, out); run<5>(p.multiProcessorCount, out);
  return 0;
}
