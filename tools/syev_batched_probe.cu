// Probe: cusolverDnXsyevBatched vs cusolverDnDsyevd for the TPS plan's n ~ 2000 eigenproblems.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/p tools/syev_batched_probe.cu -lcusolver
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void fill(double* A, int n, int seed) {
  int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  unsigned h = (unsigned)(i < j ? i * 7919 + j : j * 7919 + i) * 2654435761u + seed;
  A[(size_t)i * n + j] = (double)(h % 100000) / 100000.0 + (i == j ? n : 0);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1997;
  const int batch = argc > 2 ? atoi(argv[2]) : 8;
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  cusolverDnParams_t prm; cusolverDnCreateParams(&prm);
  double *A, *W; int* info;
  cudaMalloc(&A, sizeof(double) * n * n * batch); cudaMalloc(&W, sizeof(double) * n * batch);
  cudaMalloc(&info, sizeof(int) * batch);
  for (int b = 0; b < batch; ++b) fill<<<dim3((n + 255) / 256, n), 256>>>(A + (size_t)b * n * n, n, b);
  size_t wd = 0, wh = 0;
  cusolverStatus_t s = cusolverDnXsyevBatched_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                                         CUDA_R_64F, A, n, CUDA_R_64F, W, CUDA_R_64F, &wd, &wh, batch);
  printf("bufferSize status %d dev %zu host %zu\n", (int)s, wd, wh);
  void* bd = nullptr; void* bh = malloc(wh > 0 ? wh : 1);
  cudaMalloc(&bd, wd > 0 ? wd : 1);
  cudaDeviceSynchronize();
  for (int rep = 0; rep < 2; ++rep) {
    for (int b = 0; b < batch; ++b) fill<<<dim3((n + 255) / 256, n), 256>>>(A + (size_t)b * n * n, n, b);
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    s = cusolverDnXsyevBatched(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n,
                               CUDA_R_64F, W, CUDA_R_64F, bd, wd, bh, wh, info, batch);
    cudaError_t e = cudaDeviceSynchronize();
    double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("{\"api\": \"XsyevBatched\", \"n\": %d, \"batch\": %d, \"status\": %d, \"cuda\": %d, \"ms_per_matrix\": %.2f}\n",
           n, batch, (int)s, (int)e, 1e3 * t / batch);
  }
  // reference: Dsyevd one by one
  int lw = 0;
  cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, &lw);
  double* work; cudaMalloc(&work, sizeof(double) * lw);
  for (int b = 0; b < batch; ++b) fill<<<dim3((n + 255) / 256, n), 256>>>(A + (size_t)b * n * n, n, b);
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int b = 0; b < batch; ++b)
    cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A + (size_t)b * n * n, n, W + b * n, work, lw, info);
  cudaDeviceSynchronize();
  double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("{\"api\": \"Dsyevd\", \"n\": %d, \"batch\": %d, \"ms_per_matrix\": %.2f}\n", n, batch, 1e3 * t / batch);
  return 0;
}
