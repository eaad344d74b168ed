// FP64 peaks on B200 (sm_100a): DFMA (CUDA cores) and DMMA.8x8x4 (mma.sync f64 tensor
// path) throughput, and the accumulation semantics of one m8n8k4 f64 MMA
// (d = c + sum_{k<4} a_k b_k): compared with sequential fma chains in both orders and
// with the exactly rounded sum (double-double reference).  Output feeds profiles/.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = __fma_rn(x[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_tput(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// one m8n8k4 per warp: A (8x4 row), B (4x8 col), C (8x8).  Lane t holds A[t/4][t%4],
// B[t%4][t/4], C[t/4][2(t%4)], C[t/4][2(t%4)+1] (PTX fragment layout for m8n8k4 f64).
__global__ void dmma_once(const double* A, const double* B, const double* C, double* D) {
  int t = threadIdx.x;
  double a = A[(t / 4) * 4 + t % 4], b = B[(t % 4) * 8 + t / 4];
  double c0 = C[(t / 4) * 8 + 2 * (t % 4)], c1 = C[(t / 4) * 8 + 2 * (t % 4) + 1];
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  D[(t / 4) * 8 + 2 * (t % 4)] = c0;
  D[(t / 4) * 8 + 2 * (t % 4) + 1] = c1;
}

static double fma_fwd(const double* a, const double* b, double c) {
  for (int k = 0; k < 4; ++k) c = fma(a[k], b[k], c);
  return c;
}
static double fma_bwd(const double* a, const double* b, double c) {
  for (int k = 3; k >= 0; --k) c = fma(a[k], b[k], c);
  return c;
}
static double exact_round(const double* a, const double* b, double c) {
  __float128 s = c;
  for (int k = 0; k < 4; ++k) s += (__float128)a[k] * (__float128)b[k];
  return (double)s;
}

int main(int argc, char** argv) {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int iters = 1 << 14;
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (2048 / tpb);
    dfma_tput<<<blocks, tpb>>>(out, 64, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_tput<<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)blocks * tpb;
    printf("dfma_tput tpb=%d: %.2f TFLOP/s fp64\n", tpb, fl / ms / 1e9);
    dmma_tput<<<blocks, tpb>>>(out, 64);
    cudaEventRecord(e0); dmma_tput<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fm = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (tpb / 32);
    printf("dmma_tput tpb=%d: %.2f TFLOP/s fp64 (m8n8k4)\n", tpb, fm / ms / 1e9);
  }
  // semantics
  double *A, *B, *C, *D;
  cudaMallocManaged(&A, 32 * 8); cudaMallocManaged(&B, 32 * 8); cudaMallocManaged(&C, 64 * 8);
  cudaMallocManaged(&D, 64 * 8);
  srand(1);
  long n_fwd = 0, n_bwd = 0, n_exact = 0, n_tot = 0;
  for (int trial = 0; trial < 4000; ++trial) {
    for (int i = 0; i < 32; ++i) {
      double r = (rand() / (double)RAND_MAX - 0.5);
      A[i] = ldexp(r, rand() % 40 - 20);
      B[i] = (rand() / (double)RAND_MAX - 0.5) * (1 + rand() % 3);
    }
    for (int i = 0; i < 64; ++i) C[i] = ldexp(rand() / (double)RAND_MAX - 0.5, rand() % 40 - 20);
    dmma_once<<<1, 32>>>(A, B, C, D);
    cudaDeviceSynchronize();
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) {
        double a[4], b[4];
        for (int k = 0; k < 4; ++k) { a[k] = A[r * 4 + k]; b[k] = B[k * 8 + c]; }
        double d = D[r * 8 + c];
        n_tot++;
        n_fwd += d == fma_fwd(a, b, C[r * 8 + c]);
        n_bwd += d == fma_bwd(a, b, C[r * 8 + c]);
        n_exact += d == exact_round(a, b, C[r * 8 + c]);
      }
  }
  printf("dmma semantics over %ld outputs: equal to sequential fma k=0..3: %ld; k=3..0: %ld; "
         "exactly rounded sum: %ld\n", n_tot, n_fwd, n_bwd, n_exact);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
