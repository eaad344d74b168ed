// Standalone timing harness for a generated (pattern-specialised) factor kernel.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include KERNEL_FILE
int main(int argc, char** argv) {
  const int K = 65536, nnzA = NNZA, n = NDIM;
  std::vector<double> A(nnzA), eps(K), d(n);
  FILE* f = fopen(argv[1], "rb"); fread(A.data(), 8, nnzA, f); fread(d.data(), 8, n, f); fread(eps.data(), 8, K, f); fclose(f);
  double *dA, *de, *dd, *dV; int* dst;
  cudaMalloc(&dA, 8 * nnzA); cudaMalloc(&de, 8 * K); cudaMalloc(&dd, 8 * n);
  cudaMalloc(&dV, (size_t)8 * NNZLU * K); cudaMalloc(&dst, 4 * K);
  cudaMemcpy(dA, A.data(), 8 * nnzA, cudaMemcpyHostToDevice);
  cudaMemcpy(de, eps.data(), 8 * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dd, d.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int threads : {64, 128}) {
    for (int it = 0; it < 3; ++it) factor_gen<<<K / threads, threads>>>(dA, de, dd, 1e-300, dV, dst, K);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) factor_gen<<<K / threads, threads>>>(dA, de, dd, 1e-300, dV, dst, K);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("threads=%d factor_gen: %.3f ms per launch, %.1f GB/s (write %.2f GB)  err=%s\n", threads, ms / 10,
           (double)8 * NNZLU * K / (ms / 10 * 1e-3) / 1e9, 8.0 * NNZLU * K / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<double> V((size_t)NNZLU * 64);
  cudaMemcpy(V.data(), dV, 8 * V.size(), cudaMemcpyDeviceToHost);
  f = fopen(argv[2], "wb"); fwrite(V.data(), 8, V.size(), f); fclose(f);
  return 0;
}
