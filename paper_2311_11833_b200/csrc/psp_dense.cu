// Dense path (SURVEY §8(f) 3 and the north star's "DMMA ... for the dense path on small
// n"): the paper's own formulation, a dense no-pivot getrf/trsm per perturbed copy
// ("getrf_batched! and trsm_batched! ... no-pivoting"), rebuilt for sm_100a
// with the trailing updates on the FP64 tensor path (mma.sync m8n8k4 f64 = DMMA.8x8x4).
// It also carries what the sparse path cannot: a general (dense) perturbation matrix D
// (footnote P:L72), since A + eps_k D has no shared sparse pattern.
//
// Layout: per lane k a padded N x N row-major matrix M_k = P (A + eps_k D) P^T in HBM,
// N = n rounded up to 32, padded by the identity (padding never changes the leading
// n x n factors or solutions: its rows of L and columns of U are zero).
//
// dense_lu_kernel: one CTA (8 warps) per lane, right-looking blocked elimination in
// panels of 32 columns:
//   1. perturb (Alg. 1 step 1, fused): the CTA writes M_k row by row;
//   2. per panel kb: the (N-kb) x 32 panel in shared memory; its 32 x 32 diagonal block
//      eliminated by one warp in registers (l = a / u_pp, then fma(-l, u_pj, a_ij),
//      ascending p; the status check of R10 on every pivot), then the rows below it
//      row by row (each entry's updates in ascending p, then its division);
//   3. U12 = L11^{-1} A12, one column per thread in registers (ascending p);
//   4. A22 -= L21 U12 on the tensor path: 32 x 32 tiles per warp, C in registers
//      (16 DMMA fragments), L21 (negated) from the shared-memory panel, U12 from L1/L2,
//      k ascending in steps of 4.
// Every entry therefore receives its updates panel by panel in ascending pivot order, and
// one DMMA.8x8x4 is EXACTLY four chained fmas in its k order (d = fma(a3, b3, fma(a2, b2,
// fma(a1, b1, fma(a0, b0, c))))): measured bit for bit on 256,000 random outputs on the
// B200 (tools/probe/fp64mma.cu, profiles/r2_fp64mma.txt; R19).  With the L
// operand negated exactly, a k-step is fma(-l_ip, u_pj, a_ij) for 4 ascending p: the dense
// path reproduces the canonical order (R11) and is bitwise equal to the oracle's
// lu_nopivot, on the tensor path.
//
// dense_solve_kernel: one CTA per lane, right-hand sides in chunks of 16 held in shared
// memory (permuted order), forward (unit L) then backward (U) by 32-row blocks: the
// off-diagonal block products on DMMA accumulating onto y itself (a warp per 8 x 8 output
// fragment, j ascending forward / descending backward through the fragment's k order),
// the diagonal 32 x 32 triangle by a warp per right-hand side with shuffles (forward
// ascending; backward descending with the division at the pivot) -- again the canonical
// order, bitwise the oracle's lu_solve.
// X is written in the batch layout [k / 32][R][n][32] (permuted rows), so the recover,
// residual and introspection calls of the sparse path apply unchanged.
#include <cuda_runtime.h>

#include "psp_dense.h"

namespace psp {

namespace {

constexpr int kDNB = 32;          // panel width
constexpr int kDThreads = 256;    // 8 warps
constexpr int kDWarps = kDThreads / 32;
constexpr int kDPS = 33;          // panel row stride in shared memory (doubles; conflict-free)
constexpr int kDRC = 16;          // right-hand sides per solve pass

__device__ __forceinline__ bool dense_pivot_bad(double piv, double tol) {
  return !(fabs(piv) > tol) || !isfinite(piv);
}

// D = A * B + C, A 8x4 (row), B 4x8 (col), C/D 8x8: lane t holds A[t/4][t%4],
// B[t%4][t/4], C[t/4][2(t%4)], C[t/4][2(t%4)+1].
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// U12 column j: u = L11^{-1} a (rows kb..kb+31 of column j, unit lower L11 from the
// panel in shared memory); entry i receives its updates in ascending p.
__device__ __noinline__ void trsm_column(double* __restrict__ col, int N, const double* ps) {
  double u[kDNB];
#pragma unroll
  for (int i = 0; i < kDNB; ++i) u[i] = col[(size_t)i * N];
#pragma unroll
  for (int p = 0; p < kDNB; ++p) {
    asm volatile("" ::: "memory");   // keep each pivot's L11 loads next to their use
#pragma unroll
    for (int i = p + 1; i < kDNB; ++i) u[i] = __fma_rn(-ps[i * kDPS + p], u[p], u[i]);
  }
#pragma unroll
  for (int i = 1; i < kDNB; ++i) col[(size_t)i * N] = u[i];
}

// A panel row below the diagonal block: pr[j] <- (pr[j] - sum_{q<j} l_q u_qj, q ascending) /
// u_jj with l_q the row's own new values and u from the factored diagonal block (u_qj at
// ps[q * kDPS + j]).
__device__ __noinline__ void panel_row(double* __restrict__ pr, const double* ps) {
  double a[kDNB];
#pragma unroll
  for (int j = 0; j < kDNB; ++j) a[j] = pr[j];
#pragma unroll
  for (int j = 0; j < kDNB; ++j) {
    asm volatile("" ::: "memory");   // keep column j's U loads next to their use
#pragma unroll
    for (int q = 0; q < j; ++q) a[j] = __fma_rn(-a[q], ps[q * kDPS + j], a[j]);
    a[j] = a[j] / ps[j * kDPS + j];
  }
#pragma unroll
  for (int j = 0; j < kDNB; ++j) pr[j] = a[j];
}

template <bool kDenseD>
__global__ void __launch_bounds__(kDThreads, 1) dense_lu_kernel(const __grid_constant__ DenseArgs a) {
  extern __shared__ double ps[];   // panel: (N - kb) rows x kDPS
  const int k = blockIdx.x;
  const int N = a.N, n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* __restrict__ Mk = a.M + (size_t)k * N * N;
  const double e = a.eps[k];
  const int jac = a.mj.jac(k);
  const double* __restrict__ Aj = a.A + (size_t)jac * a.mj.a_stride;
  const double tol = a.tol_dev ? a.tol_dev[jac] : a.tol_value;

  // 1. perturb: M_k = P (A + e D) P^T (diagonal D: a_ii + (e d_i), off-diagonal a_ij;
  //    dense D: a_ij + (e D_ij) for every entry, a_ij = 0 outside the pattern)
  for (int i = warp; i < N; i += kDWarps) {
    double* row = Mk + (size_t)i * N;
    for (int j = lane; j < N; j += 32) {
      double v = 0.0;
      if (i >= n) {
        v = (j == i) ? 1.0 : 0.0;
      } else if (kDenseD) {
        if (j < n) v = 0.0 + e * a.Dp[(size_t)i * n + j];
      } else if (j == i) {
        v = 0.0 + e * a.dperm[i];
      }
      row[j] = v;
    }
    __syncwarp();
    if (i < n) {
      for (int q = a.rp[i] + lane; q < a.rp[i + 1]; q += 32) {
        const int j = a.ci[q];
        const double av = Aj[a.src[q]];
        double v;
        if (kDenseD) v = av + e * a.Dp[(size_t)i * n + j];
        else v = (j == i) ? av + e * a.dperm[i] : av;
        row[j] = v;
      }
    }
  }
  __syncthreads();

  int st = 0;   // thread 0: first failing pivot + 1
  for (int kb = 0; kb < N; kb += kDNB) {
    const int M = N - kb;
    // 2. panel rows kb..N-1, columns kb..kb+31
    for (int r = warp; r < M; r += kDWarps) ps[r * kDPS + lane] = Mk[(size_t)(kb + r) * N + kb + lane];
    __syncthreads();
    // 2a. the 32 x 32 diagonal block by warp 0, lane r = panel row r in registers, right-
    //     looking: at step p lane p publishes its (final) U row, the lanes below divide
    //     (in parallel) and update their row -- entry (r, j) gets pivot p's update at step p
    if (warp == 0) {
      double row[kDNB];
#pragma unroll
      for (int j = 0; j < kDNB; ++j) row[j] = ps[lane * kDPS + j];
#pragma unroll
      for (int p = 0; p < kDNB; ++p) {
        if (lane == p) {
#pragma unroll
          for (int j = p; j < kDNB; ++j) ps[p * kDPS + j] = row[j];
        }
        __syncwarp();
        const double piv = ps[p * kDPS + p];
        if (lane == 0 && st == 0 && kb + p < n && dense_pivot_bad(piv, tol)) st = kb + p + 1;
        if (lane > p) {
          const double l = row[p] / piv;
          row[p] = l;
#pragma unroll
          for (int j = p + 1; j < kDNB; ++j) row[j] = __fma_rn(-l, ps[p * kDPS + j], row[j]);
        }
        __syncwarp();
      }
#pragma unroll
      for (int j = 0; j < kDNB; ++j)
        if (j < lane) ps[lane * kDPS + j] = row[j];
    }
    __syncthreads();
    // 2b. the panel's rows below it, one row per thread, row-oriented: entry (r, j) gets
    //     the updates of pivots q = 0 .. j-1 in ascending order, then l_rj = a_rj / u_jj --
    //     the same per-entry sequence as the right-looking steps, without 32 CTA barriers
    for (int r = kDNB + tid; r < M; r += kDThreads) panel_row(ps + r * kDPS, ps);
    __syncthreads();
    for (int r = warp; r < M; r += kDWarps) Mk[(size_t)(kb + r) * N + kb + lane] = ps[r * kDPS + lane];
    if (M == kDNB) break;
    // 3. U12 = L11^{-1} A12: rows kb..kb+31, one column per thread
    for (int j = kb + kDNB + tid; j < N; j += kDThreads) trsm_column(Mk + (size_t)kb * N + j, N, ps);
    __syncthreads();
    // 4. A22 -= L21 U12 on DMMA: tiles of 32 x 32, contiguous tile ranges per warp
    //    (column-major tile order, so a warp reloads its U12 fragments rarely)
    const int nt = (M - kDNB) / 32;
    const int T = nt * nt;
    const int per = (T + kDWarps - 1) / kDWarps;
    const int it0 = warp * per, it1 = min(T, it0 + per);
    const int g = lane >> 2, t4 = lane & 3;
    int cur_tj = -1;
    double bf[8][4];
    for (int it = it0; it < it1; ++it) {
      const int tj = it / nt, ti = it - tj * nt;
      const int c0 = kb + kDNB + 32 * tj;
      const int r0 = kDNB + 32 * ti;             // panel-relative row of the tile
      if (tj != cur_tj) {
        cur_tj = tj;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
#pragma unroll
          for (int b = 0; b < 4; ++b) bf[ks][b] = Mk[(size_t)(kb + 4 * ks + t4) * N + c0 + 8 * b + g];
      }
      double c[4][4][2];
#pragma unroll
      for (int aa = 0; aa < 4; ++aa)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double2 v =
              *reinterpret_cast<const double2*>(Mk + (size_t)(kb + r0 + 8 * aa + g) * N + c0 + 8 * b + 2 * t4);
          c[aa][b][0] = v.x;
          c[aa][b][1] = v.y;
        }
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        double af[4];
#pragma unroll
        for (int aa = 0; aa < 4; ++aa) af[aa] = -ps[(r0 + 8 * aa + g) * kDPS + 4 * ks + t4];
#pragma unroll
        for (int aa = 0; aa < 4; ++aa)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma(c[aa][b][0], c[aa][b][1], af[aa], bf[ks][b]);
      }
#pragma unroll
      for (int aa = 0; aa < 4; ++aa)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          *reinterpret_cast<double2*>(Mk + (size_t)(kb + r0 + 8 * aa + g) * N + c0 + 8 * b + 2 * t4) =
              make_double2(c[aa][b][0], c[aa][b][1]);
    }
    __syncthreads();
  }
  if (tid == 0) a.status[k] = st;
}

// Off-diagonal block product of the solves, in the canonical order: warp w owns the 8 x 8
// output fragment (rows row0 + 8 (w / 2), right-hand sides 8 (w % 2)) and accumulates onto
// Y itself, one DMMA per 4 columns j of the factor, each DMMA a chain of 4 fmas in its k
// order (measured, tools/probe/fp64mma.cu).  Forward (kDesc = false): j ascending over
// [jlo, jhi); backward (kDesc = true): j descending from jhi - 1 to jlo (the k index of a
// DMMA maps to j = j0 + 3 - k).  y_i = fma(-m_ij, y_j, y_i) for each j in that order.
template <bool kDesc>
__device__ __forceinline__ void block_update(const double* __restrict__ Mk, int N, int row0, int jlo, int jhi,
                                             double* Y, int warp, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  const int ra = row0 + 8 * (warp >> 1), cb = 8 * (warp & 1);
  double c0 = Y[(ra + g) * kDRC + cb + 2 * t4], c1 = Y[(ra + g) * kDRC + cb + 2 * t4 + 1];
  const double* mrow = Mk + (size_t)(ra + g) * N;
  const int nks = (jhi - jlo) / 4;
  for (int s = 0; s < nks; ++s) {
    const int j = kDesc ? jhi - 4 * s - 1 - t4 : jlo + 4 * s + t4;
    dmma(c0, c1, -mrow[j], Y[j * kDRC + cb + g]);
  }
  Y[(ra + g) * kDRC + cb + 2 * t4] = c0;
  Y[(ra + g) * kDRC + cb + 2 * t4 + 1] = c1;
}

// Diagonal 32 x 32 block of the factor into shared memory (rows / columns row0..row0+31).
__device__ __forceinline__ void load_diag_block(const double* __restrict__ Mk, int N, int row0, double* Tb,
                                                int tid) {
  for (int idx = tid; idx < 32 * 32; idx += kDThreads) {
    const int i = idx >> 5, j = idx & 31;
    Tb[i * kDPS + j] = Mk[(size_t)(row0 + i) * N + row0 + j];
  }
}

__global__ void __launch_bounds__(kDThreads, 2) dense_solve_kernel(const __grid_constant__ DenseSolveArgs a) {
  extern __shared__ double sm[];
  const int N = a.N, n = a.n, R = a.R;
  double* Y = sm;                              // [N][kDRC]
  double* Tb = Y + (size_t)N * kDRC;           // [32][kDPS] diagonal block
  const int k = blockIdx.x;
  // (the warp index through a shuffle: warp-uniform for the compiler -- no WARPSYNC guards
  // around the DMMA instructions; measured 0.628 -> 0.609 ms on cfg2, and +2% on the LU
  // kernel, which keeps the plain form)
  const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const double* __restrict__ Mk = a.M + (size_t)k * N * N;
  const double* __restrict__ Bk = a.B + (size_t)a.mj.jac(k) * a.mj.b_stride;
  for (int rc0 = 0; rc0 < R; rc0 += kDRC) {
    for (int idx = tid; idx < N * kDRC; idx += kDThreads) {
      const int i = idx / kDRC, r = idx - i * kDRC;
      Y[idx] = (i < n && rc0 + r < R) ? Bk[(size_t)(rc0 + r) * a.ldb + a.perm[i]] : 0.0;
    }
    __syncthreads();
    // forward: y = L^{-1} P b (unit lower), y_i receiving its updates in ascending j
    for (int row0 = 0; row0 < N; row0 += 32) {
      if (row0 > 0) block_update<false>(Mk, N, row0, 0, row0, Y, warp, lane);
      load_diag_block(Mk, N, row0, Tb, tid);
      __syncthreads();
      for (int r = warp; r < kDRC; r += kDWarps) {
        double y = Y[(row0 + lane) * kDRC + r];
        for (int p = 0; p < 31; ++p) {
          const double yp = __shfl_sync(0xffffffffu, y, p);
          if (lane > p) y = __fma_rn(-Tb[lane * kDPS + p], yp, y);
        }
        Y[(row0 + lane) * kDRC + r] = y;
      }
      __syncthreads();
    }
    // backward: x = U^{-1} y, y_i receiving its updates in descending j, the division last
    for (int row0 = N - 32; row0 >= 0; row0 -= 32) {
      if (row0 + 32 < N) block_update<true>(Mk, N, row0, row0 + 32, N, Y, warp, lane);
      load_diag_block(Mk, N, row0, Tb, tid);
      __syncthreads();
      for (int r = warp; r < kDRC; r += kDWarps) {
        double y = Y[(row0 + lane) * kDRC + r];
        for (int p = 31; p >= 0; --p) {
          if (lane == p) y = y / Tb[p * kDPS + p];
          const double xp = __shfl_sync(0xffffffffu, y, p);
          if (lane < p) y = __fma_rn(-Tb[lane * kDPS + p], xp, y);
        }
        Y[(row0 + lane) * kDRC + r] = y;
      }
      __syncthreads();
    }
    for (int idx = tid; idx < n * kDRC; idx += kDThreads) {
      const int r = idx / n, i = idx - r * n;
      if (rc0 + r < R)
        a.X[(((size_t)(k >> 5) * R + rc0 + r) * n + i) * 32 + (k & 31)] = Y[i * kDRC + r];
    }
    __syncthreads();
  }
}

}  // namespace

int dense_padded_order(int n) { return (n + kDNB - 1) / kDNB * kDNB; }

size_t dense_lu_smem(int N) { return sizeof(double) * (size_t)N * kDPS; }

size_t dense_solve_smem(int N) { return sizeof(double) * ((size_t)N * kDRC + 32 * kDPS); }

cudaError_t configure_dense(int N) {
  cudaError_t e = cudaFuncSetAttribute(dense_lu_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dense_lu_smem(N));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dense_lu_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)dense_lu_smem(N));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(dense_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)dense_solve_smem(N));
}

cudaError_t launch_dense_lu(const DenseArgs& a, int K, cudaStream_t stream) {
  if (K <= 0) return cudaSuccess;
  if (a.Dp)
    dense_lu_kernel<true><<<K, kDThreads, dense_lu_smem(a.N), stream>>>(a);
  else
    dense_lu_kernel<false><<<K, kDThreads, dense_lu_smem(a.N), stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_dense_solve(const DenseSolveArgs& a, int K, cudaStream_t stream) {
  if (K <= 0) return cudaSuccess;
  dense_solve_kernel<<<K, kDThreads, dense_solve_smem(a.N), stream>>>(a);
  return cudaGetLastError();
}

}  // namespace psp
