// Dense no-pivot LU / triangular-solve kernels (psp_dense.cu): the paper's dense
// getrf/trsm formulation on the FP64 tensor path, and the path for a
// general (dense) perturbation matrix D.  Internal; not part of the C ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "psp_internal.h"

namespace psp {

struct DenseArgs {
  int32_t n = 0, N = 0;                 // order, padded order (multiple of 32)
  const int32_t* rp = nullptr;          // permuted CSR of A: row_ptr [n+1]
  const int32_t* ci = nullptr;          //   permuted column index
  const int32_t* src = nullptr;         //   index into A_vals
  const double* A = nullptr;            // A_vals (the caller's, CSR order of the pattern)
  const double* eps = nullptr;          // [K] signed perturbations
  const double* dperm = nullptr;        // [n] diag(D), permuted (diagonal D)
  const double* Dp = nullptr;           // [n][n] P D P^T row-major (dense D) or nullptr
  const double* tol_dev = nullptr;      // device pivot tolerance or nullptr
  double tol_value = 0.0;
  double* M = nullptr;                  // [K][N][N] row-major factors
  int32_t* status = nullptr;            // [K]
  MultiJac mj;                          // (multi-Jacobian batches)
};

struct DenseSolveArgs {
  int32_t n = 0, N = 0, R = 0;
  int64_t ldb = 0;
  const int32_t* perm = nullptr;        // perm[new] = old
  const double* M = nullptr;            // [K][N][N] factors
  const double* B = nullptr;            // n x R column-major (ldb)
  double* X = nullptr;                  // [K/32][R][n][32], permuted rows
  MultiJac mj;
};

int dense_padded_order(int n);
size_t dense_lu_smem(int N);
size_t dense_solve_smem(int N);
cudaError_t configure_dense(int N);
cudaError_t launch_dense_lu(const DenseArgs& a, int K, cudaStream_t stream);
cudaError_t launch_dense_solve(const DenseSolveArgs& a, int K, cudaStream_t stream);

}  // namespace psp
