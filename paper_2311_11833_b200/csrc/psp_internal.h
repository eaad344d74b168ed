// Internal declarations shared by the host runtime (psp_host.cpp) and the CUDA
// kernels (psp_kernels.cu).  Not part of the C ABI (include/psp.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace psp {

// Lanes are grouped in slabs of kSlab consecutive lanes (one warp).  Every
// batch-major array is laid out [slab][item][kSlab]: a warp's 32 lanes of one item
// are 256 contiguous bytes (one coalesced access), and a slab's whole factor is one
// contiguous region.
constexpr int kSlab = 32;

// Device-side plan of the left-looking factorisation and the triangular solves,
// produced once by the symbolic analysis.  All indices are int32 "slots" into a
// lane's nnz_LU values (column-major over the filled pattern: for column j the U
// rows i<j ascending, then the diagonal, then the L rows i>j ascending).
struct DevicePlan {
  int32_t n = 0, nnz_A = 0, nnz_LU = 0;
  // perturb + scatter (Alg. 1 step 1): slot -> CSR index of A (or -1 for fill)
  const int32_t* a_src = nullptr;      // [nnz_LU]
  const int32_t* diag_slot = nullptr;  // [n]  slot of (j,j)
  const int32_t* col_end = nullptr;    // [n]  one past the last slot of column j
  // left-looking updates: column j owns groups [col_gptr[j], col_gptr[j+1]); group g
  // reads u = LU[g_u[g]] and applies LU[pr_d[q]] = fma(-LU[pr_l[q]], u, LU[pr_d[q]])
  // for q in [g_ptr[g], g_ptr[g+1]) — groups in ascending pivot order p.
  const int32_t* col_gptr = nullptr;   // [n+1]
  const int32_t* g_u = nullptr;        // [n_groups]
  const int32_t* g_ptr = nullptr;      // [n_groups+1]
  const int32_t* pr_l = nullptr;       // [n_pairs]
  const int32_t* pr_d = nullptr;       // [n_pairs]
  // row-oriented triangular solves
  const int32_t* rl_ptr = nullptr;     // [n+1]  row i of L: j ascending
  const int32_t* rl_slot = nullptr;
  const int32_t* rl_col = nullptr;
  const int32_t* ru_ptr = nullptr;     // [n+1]  row i of U (j > i): j descending
  const int32_t* ru_slot = nullptr;
  const int32_t* ru_col = nullptr;
  const int32_t* perm = nullptr;       // [n]  perm[new] = old
  // deterministic column sums for the default pivot tolerance
  const int32_t* acsc_ptr = nullptr;   // [n+1]
  const int32_t* acsc_q = nullptr;     // [nnz_A] CSR indices grouped by column
};

// Kernel launchers (psp_kernels.cu).  All asynchronous on `stream`.
cudaError_t launch_pivot_tol(const DevicePlan& p, const double* A_vals, double* tol_out,
                             cudaStream_t stream);
cudaError_t launch_factor(const DevicePlan& p, const double* A_vals, const double* eps,
                          const double* dperm, const double* tol_dev, double tol_value,
                          double* V, int32_t* status, int32_t K, int32_t K_pad,
                          cudaStream_t stream);
cudaError_t launch_solve(const DevicePlan& p, const double* V, const double* B, int64_t ldb,
                         int32_t R, double* X, int32_t K_pad, cudaStream_t stream);
cudaError_t launch_recover(const DevicePlan& p, int32_t W, int32_t R, const int32_t* w_ptr,
                           const int32_t* w_lane, const double* w_val, const double* X,
                           const int32_t* status, double* x_out, int32_t* infeasible_flag,
                           cudaStream_t stream);
cudaError_t launch_gather_solutions(const DevicePlan& p, int32_t K, int32_t R, const double* X,
                                    double* out, cudaStream_t stream);

}  // namespace psp
