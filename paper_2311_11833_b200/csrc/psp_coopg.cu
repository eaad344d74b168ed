// Level-scheduled kernels for large systems (n = 3600 / 18000,
// K = 1024 / 512): one CTA per perturbed system, the parallelism inside the system used
// instead of one thread per lane (K lanes leave the batch kernels with K / 32 warps on 148
// SMs).  Same elimination-tree level schedule as the cooperative small-batch kernels
// (psp_plan.cpp build_coop: a contribution of pivot p to an entry runs at the running
// maximum of the levels of that entry's contributors in ascending pivot order), so every
// entry still receives its updates in the canonical order (R11): bitwise the batch
// kernels and the oracle.  The difference: the factor image does not fit shared memory
// (8 nnz_LU = 336 KB / 1.8 MB), so it lives in a lane-major global scratch W[k][nnz_LU]
// -- a CTA's working set stays L2-resident for the n = 3600 system (148 x 336 KB) -- and
// the plan uses 32-bit fields (nnz_LU and the contribution counts exceed 16 bits at
// n = 18000).  The solve keeps y in shared memory (8 n bytes) and writes X in the batch
// layout [k / 32][R][n][32] (permuted rows) used by recover / residual / introspection.
#include <climits>
#include <cuda_runtime.h>

#include "psp_coopg.h"

namespace psp {

namespace {

#ifndef PSP_CG_THREADS
#define PSP_CG_THREADS 256
#endif
constexpr int kCgThreads = PSP_CG_THREADS;
#ifndef PSP_CG_MINBLOCKS
#define PSP_CG_MINBLOCKS (1024 / PSP_CG_THREADS)
#endif
constexpr int kCgMinBlocks = PSP_CG_MINBLOCKS;   // (64 registers per thread at 4 x 256)

__device__ __forceinline__ bool cg_pivot_bad(double piv, double tol) {
  return !(fabs(piv) > tol) || !isfinite(piv);
}

// One target's contribution chain x = fma(-a_q, b_q, x) for q = q0 .. q1-1 in order.  The
// chain is sequential in x (canonical order), but its operands are not: they are loaded
// kCgDepth at a time before the block's fmas, so a long chain (the dense separator rows:
// hundreds of contributions) costs one L2 latency per block instead of per contribution.
// Operand q: a = va(c[q].x), b = vb(c[q].y).
#ifndef PSP_CG_DEPTH
#define PSP_CG_DEPTH 8
#endif
constexpr int kCgDepth = PSP_CG_DEPTH;
template <class VA, class VB>
__device__ __forceinline__ double cg_chain(double x, const int2* __restrict__ c, int q0, int q1, VA va, VB vb) {
  int q = q0;
  if (q + kCgDepth <= q1) {
    // the next block's indices are fetched while the current block's operands load
    int2 w[kCgDepth];
#pragma unroll
    for (int t = 0; t < kCgDepth; ++t) w[t] = c[q + t];
    for (; q + kCgDepth <= q1; q += kCgDepth) {
      double a[kCgDepth], b[kCgDepth];
#pragma unroll
      for (int t = 0; t < kCgDepth; ++t) {
        a[t] = va(w[t].x);
        b[t] = vb(w[t].y);
      }
      if (q + 2 * kCgDepth <= q1) {
#pragma unroll
        for (int t = 0; t < kCgDepth; ++t) w[t] = c[q + kCgDepth + t];
      }
#pragma unroll
      for (int t = 0; t < kCgDepth; ++t) x = __fma_rn(-a[t], b[t], x);
    }
  }
  for (; q < q1; ++q) {
    const int2 w = c[q];
    x = __fma_rn(-va(w.x), vb(w.y), x);
  }
  return x;
}

__global__ void __launch_bounds__(kCgThreads, kCgMinBlocks) coopg_factor_kernel(const __grid_constant__ CoopGArgs a) {
  const CoopGDev& c = a.c;
  __shared__ int st;
  const int k = blockIdx.x, tid = threadIdx.x;
  double* __restrict__ v = a.W + (size_t)k * c.nnz_LU;
  if (tid == 0) st = INT_MAX;
  const double e = a.eps[k];
  const int jac = a.mj.jac(k);
  const double* __restrict__ A = a.A + (size_t)jac * a.mj.a_stride;
  for (int q = tid; q < c.nnz_LU; q += kCgThreads) {   // births (a + (eps d) on the diagonal)
    const int sidx = c.birth_src[q], d = c.birth_diag[q];
    const double av = sidx >= 0 ? A[sidx] : 0.0;
    v[q] = d >= 0 ? __dadd_rn(av, __dmul_rn(e, a.dperm[d])) : av;
  }
  const double tol = a.tol_dev ? a.tol_dev[jac] : a.tol_value;
  __syncthreads();
  for (int step = 0; step < c.steps; ++step) {
    for (int j = c.fp_ptr[step] + tid; j < c.fp_ptr[step + 1]; j += kCgThreads) {
      const int2 w = c.fp[j];
      if (cg_pivot_bad(v[w.x], tol)) atomicMin(&st, w.y + 1);
    }
    for (int j = c.fa_ptr[step] + tid; j < c.fa_ptr[step + 1]; j += kCgThreads) {
      const int2 w = c.fa[j];
      v[w.x] = __ddiv_rn(v[w.x], v[w.y]);
    }
    __syncthreads();
    for (int j = c.fb_ptr[step] + tid; j < c.fb_ptr[step + 1]; j += kCgThreads) {
      const int2 w = c.fbt[j];
      const int q1 = c.fbt[j + 1].y;
      auto vv = [v](int i) { return v[i]; };
      v[w.x] = cg_chain(v[w.x], c.fbc, w.y, q1, vv, vv);
    }
    __syncthreads();
  }
  if (tid == 0) a.status[k] = st == INT_MAX ? 0 : st;
}

__global__ void __launch_bounds__(kCgThreads, kCgMinBlocks) coopg_solve_kernel(const __grid_constant__ CoopGSolveArgs a) {
  const CoopGDev& c = a.c;
  extern __shared__ double y[];   // [n]
  // one CTA per (lane, right-hand side): the R solves of a lane run in parallel, sharing
  // (reading) the lane's factor image
  const int k = blockIdx.x / a.R, r = blockIdx.x - k * a.R, tid = threadIdx.x;
  const double* __restrict__ v = a.W + (size_t)k * c.nnz_LU;
  auto vg = [v](int i) { return v[i]; };
  auto ys = [](int i) { return y[i]; };
  const double* __restrict__ B = a.B + (size_t)a.mj.jac(k) * a.mj.b_stride;
  {
    for (int i = tid; i < c.n; i += kCgThreads) y[i] = B[(size_t)r * a.ldb + a.perm[i]];
    __syncthreads();
    for (int step = 0; step < c.steps; ++step) {   // forward: y_i = fma(-l_ip, y_p, y_i), p ascending
      for (int j = c.ya_ptr[step] + tid; j < c.ya_ptr[step + 1]; j += kCgThreads) {
        const int2 w = c.yat[j];
        const int q1 = c.yat[j + 1].y;
        y[w.x] = cg_chain(y[w.x], c.yac, w.y, q1, vg, ys);
      }
      __syncthreads();
    }
    for (int step = 0; step < c.steps; ++step) {   // backward, roots first: descending sum, division last
      for (int j = c.xb_ptr[step] + tid; j < c.xb_ptr[step + 1]; j += kCgThreads) {
        const int2 w = c.xbr[j];
        const int q1 = c.xbr[j + 1].y;
        const double acc = cg_chain(y[w.x], c.xbc, w.y, q1, vg, ys);
        y[w.x] = __ddiv_rn(acc, v[c.xbd[j]]);
      }
      __syncthreads();
    }
    double* xo = a.X + ((size_t)(k >> 5) * a.R + r) * c.n * 32 + (k & 31);
    for (int i = tid; i < c.n; i += kCgThreads) xo[(size_t)i * 32] = y[i];
    __syncthreads();
  }
}

}  // namespace

size_t coopg_solve_smem(int n) { return sizeof(double) * (size_t)n; }

cudaError_t configure_coopg(int n) {
  if (coopg_solve_smem(n) > 48 * 1024)
    return cudaFuncSetAttribute(coopg_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)coopg_solve_smem(n));
  return cudaSuccess;
}

cudaError_t launch_coopg_factor(const CoopGArgs& a, int K, cudaStream_t stream) {
  if (K <= 0) return cudaSuccess;
  coopg_factor_kernel<<<K, kCgThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_coopg_solve(const CoopGSolveArgs& a, int K, cudaStream_t stream) {
  if (K <= 0) return cudaSuccess;
  coopg_solve_kernel<<<K * a.R, kCgThreads, coopg_solve_smem(a.c.n), stream>>>(a);
  return cudaGetLastError();
}

}  // namespace psp
