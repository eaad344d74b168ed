// Level-scheduled kernels for large systems with the factor image in global memory
// (psp_coopg.cu).  Internal; not part of the C ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "psp_internal.h"

namespace psp {

// The CoopPlan of psp_plan.h with 32-bit fields (device arrays).
struct CoopGDev {
  int32_t steps = 0, nnz_LU = 0, n = 0;
  const int32_t* birth_src = nullptr;   // [nnz_LU] CSR index of A or -1
  const int32_t* birth_diag = nullptr;  // [nnz_LU] row p for u_pp entries, else -1
  const int32_t *fa_ptr = nullptr, *fp_ptr = nullptr, *fb_ptr = nullptr;   // [steps + 1]
  const int2* fa = nullptr;    // (l position, its pivot's position)
  const int2* fp = nullptr;    // (pivot position, pivot index)
  const int2* fbt = nullptr;   // (target position, first contribution) + sentinel (., end)
  const int2* fbc = nullptr;   // (l position, u position), ascending pivot per target
  const int32_t *ya_ptr = nullptr, *xb_ptr = nullptr;                       // [steps + 1]
  const int2* yat = nullptr;   // (row, first contribution) + sentinel
  const int2* yac = nullptr;   // (l position, source row)
  const int2* xbr = nullptr;   // (row, first contribution) + sentinel
  const int32_t* xbd = nullptr;   // u_pp position of each backward row
  const int2* xbc = nullptr;   // (u position, column), descending column
};

struct CoopGArgs {
  CoopGDev c;
  const double* A = nullptr;       // A_vals (CSR order of the analysed pattern)
  const double* eps = nullptr;     // [K]
  const double* dperm = nullptr;   // [n] permuted diag(D)
  const double* tol_dev = nullptr;
  double tol_value = 0.0;
  double* W = nullptr;             // [K][nnz_LU] lane-major factor images (positions of V)
  int32_t* status = nullptr;
  MultiJac mj;                     // (multi-Jacobian batches)
};

struct CoopGSolveArgs {
  CoopGDev c;
  const int32_t* perm = nullptr;
  const double* W = nullptr;
  const double* B = nullptr;
  int64_t ldb = 0;
  int32_t R = 0;
  double* X = nullptr;             // [K/32][R][n][32]
  MultiJac mj;
};

size_t coopg_solve_smem(int n);
cudaError_t configure_coopg(int n);
cudaError_t launch_coopg_factor(const CoopGArgs& a, int K, cudaStream_t stream);
cudaError_t launch_coopg_solve(const CoopGSolveArgs& a, int K, cudaStream_t stream);

}  // namespace psp
