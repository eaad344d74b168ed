// Internal declarations shared by the host runtime (psp_host.cpp) and the CUDA
// kernels (psp_kernels.cu).  Not part of the C ABI (include/psp.h is).
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

namespace psp {

// Lanes are grouped in slabs of kSlab consecutive lanes (one warp, one thread per
// lane).  Every batch-major array is laid out [slab][item][kSlab]: a warp's 32 lanes
// of one item are 256 contiguous bytes (one coalesced access), and a slab's whole
// factor is one contiguous region.
constexpr int kSlab = 32;
constexpr int kRowBytes = kSlab * 8;   // one item of one slab
// Source codes of the factor program: >= 0 pending slot; kZero = structural zero;
// otherwise A[-1 - code].
constexpr int32_t kZero = INT32_MIN;
constexpr int kStages = 3;             // depth of every shared-memory streaming ring
constexpr int kDataRows = 16;          // factor rows per stage of the solve's data ring

// Device-side programs (see psp_plan.cpp for their meaning).
struct DevicePlan {
  int32_t n = 0, nnz_A = 0, nnz_LU = 0, nnz_L = 0, c_max = 0;
  const int32_t* perm = nullptr;       // [n]  perm[new] = old
  // factor program (record stream in chunks)
  int32_t f_slots = 0, f_chunk_words = 0, f_nchunks = 0;
  const int32_t* f_stream = nullptr;
  // forward (ascending) and backward (descending) substitution programs
  int32_t y_slots = 0, y_chunk_words = 0, y_nchunks = 0;
  int32_t x_slots = 0, x_chunk_words = 0, x_nchunks = 0;
  const int32_t* y_stream = nullptr;
  const int32_t* x_stream = nullptr;
  // deterministic column sums for the default pivot tolerance
  const int32_t* acsc_ptr = nullptr;   // [n+1]
  const int32_t* acsc_q = nullptr;     // [nnz_A]
};

// Launch configuration chosen per plan (host, psp_kernels.cu: configure_kernels).
struct LaunchInfo {
  // factor
  bool f_pend_smem = false;    // pending slots in shared memory (else global scratch)
  bool f_a_smem = false;       // A values and d staged in shared memory
  int f_warps = 1;             // warps (slabs) per CTA
  int f_smem = 0;              // dynamic shared memory per CTA
  int f_off_a = 0, f_off_d = 0, f_off_warp = 0, f_warp_bytes = 0;
  // solve
  bool s_live_smem = false;
  int s_warps = 1;
  int s_smem = 0;
  int s_off_b = 0, s_off_warp = 0, s_warp_bytes = 0, s_ring_bytes = 0;
};

// Kernel launchers (psp_kernels.cu).  All asynchronous on `stream`.
void choose_launch(const DevicePlan& p, LaunchInfo& li);   // pure host logic
cudaError_t configure_kernels(const DevicePlan& p, LaunchInfo& li);
cudaError_t launch_pivot_tol(const DevicePlan& p, const double* A_vals, double* tol_out,
                             cudaStream_t stream);
cudaError_t launch_factor(const DevicePlan& p, const LaunchInfo& li, const double* A_vals,
                          const double* eps, const double* dperm, const double* tol_dev,
                          double tol_value, double* V, double* gscratch, int32_t* status,
                          int32_t K_pad, const int32_t* only, cudaStream_t stream);
cudaError_t launch_solve(const DevicePlan& p, const LaunchInfo& li, const double* V,
                         const double* B, int64_t ldb, int32_t R, double* X, double* gscratch,
                         int32_t K_pad, const int32_t* only, cudaStream_t stream);
cudaError_t launch_recover(const DevicePlan& p, int32_t W, int32_t R, const int32_t* w_ptr,
                           const int32_t* w_lane, const double* w_val, const double* X,
                           const int32_t* status, double* x_out, int32_t* infeasible_flag,
                           cudaStream_t stream);
cudaError_t launch_gather_solutions(const DevicePlan& p, int32_t K, int32_t R, const double* X,
                                    double* out, cudaStream_t stream);

}  // namespace psp
