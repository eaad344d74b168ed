// Shared-memory bandwidth probe: warp-wide LDS.64 / LDS.128 / STS.64 per SM clock.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(unsigned long long* out, int iters, long long* cyc) {
  extern __shared__ double s[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long acc = 0;
  int o = (w * 256) & 8191;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < 16; ++u) acc ^= __double_as_longlong(s[((o + u * 32) & 8191) + lane]);
    } else if (MODE == 1) {
      const double2* s2 = reinterpret_cast<const double2*>(s);
#pragma unroll
      for (int u = 0; u < 16; ++u) { double2 v = s2[((o / 2 + u * 32) & 4095) + lane]; acc ^= __double_as_longlong(v.x) ^ __double_as_longlong(v.y); }
    } else {
#pragma unroll
      for (int u = 0; u < 16; ++u) s[((o + u * 32) & 8191) + lane] = (double)(i + u);
    }
    o = (o + 512 + (int)(acc & 1)) & 8191;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + (MODE == 2 ? __double_as_longlong(s[lane]) : 0);
}
int main() {
  unsigned long long* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 16);
  int sms = 148, iters = 4096;
  for (int threads : {256, 1024}) {
    for (int mode = 0; mode < 3; ++mode) {
      auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      f<<<sms, threads, 65536>>>(out, 16, cyc);
      f<<<sms, threads, 65536>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double bytes = (double)threads / 32 * iters * 16 * (mode == 1 ? 512.0 : 256.0);
      printf("mode=%s threads=%d: %.1f B/clk/SM (%.2f warp-instr/clk)\n", mode == 0 ? "LDS.64" : mode == 1 ? "LDS.128" : "STS.64",
             threads, bytes / c, (double)threads / 32 * iters * 16 / c);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
