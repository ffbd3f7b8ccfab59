// Does cuSOLVER Dsyevd overlap across streams/threads?  (tuning probe for the TPS plan builder)
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/syevd_overlap tools/syevd_overlap.cu -lcusolver
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

__global__ void fill(double* A, int n, int seed) {
  int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  unsigned h = (unsigned)(i < j ? i * 7919 + j : j * 7919 + i) * 2654435761u + seed;
  A[(size_t)i * n + j] = (double)(h % 100000) / 100000.0 + (i == j ? n : 0);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1997;
  for (int lanes : {1, 2, 4, 8}) {
    const int per = 4;
    std::vector<std::thread> th;
    auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < lanes; ++t)
      th.emplace_back([=] {
        cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        cusolverDnHandle_t h; cusolverDnCreate(&h); cusolverDnSetStream(h, st);
        double *A, *W, *work; int* info; int lw = 0;
        cudaMalloc(&A, sizeof(double) * n * n); cudaMalloc(&W, sizeof(double) * n); cudaMalloc(&info, sizeof(int));
        cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, &lw);
        cudaMalloc(&work, sizeof(double) * lw);
        for (int r = 0; r < per; ++r) {
          fill<<<dim3((n + 255) / 256, n), 256, 0, st>>>(A, n, t * 100 + r);
          cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, work, lw, info);
        }
        cudaStreamSynchronize(st);
        cudaFree(A); cudaFree(W); cudaFree(work); cudaFree(info);
        cusolverDnDestroy(h); cudaStreamDestroy(st);
      });
    for (auto& x : th) x.join();
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("{\"n\": %d, \"lanes\": %d, \"problems\": %d, \"s\": %.3f, \"ms_per_problem\": %.2f}\n", n, lanes,
           lanes * per, s, 1e3 * s / (lanes * per));
  }
  return 0;
}
