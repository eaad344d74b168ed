// Device probe: properties, FP64 FMA throughput/latency, smem FP64 load throughput.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
    x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void dfma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __fma_rn(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lds_tput(double* out, int iters) {
  extern __shared__ double s[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  int base = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = 0; i < iters; ++i) {
    int o = ((i * 4 + w) & 31) * 128;
    acc0 += s[o + base]; acc1 += s[o + 32 + base]; acc2 += s[o + 64 + base]; acc3 += s[o + 96 + base];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("name=%s sms=%d cc=%d.%d l2=%d smem_per_sm=%zu smem_optin=%zu regs_per_sm=%d clock_khz=%d memclk_khz=%d busw=%d\n",
         p.name, p.multiProcessorCount, p.major, p.minor, p.l2CacheSize, p.sharedMemPerMultiprocessor,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  double* out; long long* cyc; cudaMalloc(&out, 1 << 26); cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 1 << 16; int blocks = p.multiProcessorCount * 8, threads = 256;
  dfma_tput<<<blocks, threads>>>(out, 1024, 1.0000001, 1e-9);
  cudaEventRecord(e0); dfma_tput<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
  cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 8 * iters * (double)blocks * threads;
  printf("dfma_tput: %.2f TFLOP/s fp64 (%.3f ms)\n", fl / ms / 1e9, ms);
  dfma_lat<<<1, 32>>>(out, cyc, 4096, 1.0000001, 1e-9);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dfma_lat: %.2f cycles per dependent DFMA\n", c / 4096.0);
  cudaFuncSetAttribute(lds_tput, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  lds_tput<<<blocks, threads, 32768>>>(out, 1024);
  cudaEventRecord(e0); lds_tput<<<blocks, threads, 32768>>>(out, iters); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  double by = 8.0 * 4 * iters * (double)blocks * threads;
  printf("lds64_tput: %.2f TB/s chip, %.1f B/clk/SM at %d MHz\n", by / ms / 1e9, by / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3), p.clockRate / 1000);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
