// Internal declarations shared by the host runtime (psp_host.cpp) and the CUDA
// kernels (psp_kernels.cu).  Not part of the C ABI (include/psp.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace psp {

// Lanes are grouped in slabs of kSlab consecutive lanes (one warp, one thread per
// lane).  Every batch-major array is laid out [slab][item][kSlab]: a warp's 32 lanes
// of one item are 256 contiguous bytes (one coalesced access), and a slab's whole
// factor is one contiguous region.
constexpr int kSlab = 32;
// Source codes of the factor program: >= 0 pending slot; kZero = structural zero;
// otherwise A[-1 - code].
constexpr int32_t kZero = INT32_MIN;

// Device-side programs (see psp_plan.cpp for their meaning).
struct DevicePlan {
  int32_t n = 0, nnz_A = 0, nnz_LU = 0, c_max = 0;
  const int32_t* blk = nullptr;        // [n+1]
  const int32_t* perm = nullptr;       // [n]  perm[new] = old
  // factor
  int32_t f_slots = 0;                 // pending slots (+ c_max scratch slots follow)
  const int32_t* f_ptr = nullptr;      // [n+1]
  const int32_t* f_code = nullptr;
  const int32_t* f_upd_ptr = nullptr;  // [n+1] in int4 units
  const int4* f_upd = nullptr;         // 8 x uint16 pending slots per int4
  // solves
  int32_t y_slots = 0, x_slots = 0;
  const int32_t* y_ptr = nullptr;
  const int32_t* y_code = nullptr;
  const int32_t* x_ptr = nullptr;
  const int32_t* x_code = nullptr;
  // deterministic column sums for the default pivot tolerance
  const int32_t* acsc_ptr = nullptr;   // [n+1]
  const int32_t* acsc_q = nullptr;     // [nnz_A]
};

// Launch configuration chosen per plan (host).
struct LaunchInfo {
  int factor_smem_bytes = 0;   // per warp; 0 => pending buffer in global scratch
  int factor_warps_per_cta = 1;
  int solve_smem_bytes = 0;    // per warp
  int solve_warps_per_cta = 1;
};

// Kernel launchers (psp_kernels.cu).  All asynchronous on `stream`.
cudaError_t launch_pivot_tol(const DevicePlan& p, const double* A_vals, double* tol_out,
                             cudaStream_t stream);
cudaError_t launch_factor(const DevicePlan& p, const LaunchInfo& li, const double* A_vals,
                          const double* eps, const double* dperm, const double* tol_dev,
                          double tol_value, double* V, double* gscratch, int32_t* status,
                          int32_t K_pad, cudaStream_t stream);
cudaError_t launch_solve(const DevicePlan& p, const LaunchInfo& li, const double* V,
                         const double* B, int64_t ldb, int32_t R, double* X, double* gscratch,
                         int32_t K_pad, cudaStream_t stream);
cudaError_t launch_recover(const DevicePlan& p, int32_t W, int32_t R, const int32_t* w_ptr,
                           const int32_t* w_lane, const double* w_val, const double* X,
                           const int32_t* status, double* x_out, int32_t* infeasible_flag,
                           cudaStream_t stream);
cudaError_t launch_gather_solutions(const DevicePlan& p, int32_t K, int32_t R, const double* X,
                                    double* out, cudaStream_t stream);
cudaError_t configure_kernels(const DevicePlan& p, LaunchInfo& li);

}  // namespace psp
