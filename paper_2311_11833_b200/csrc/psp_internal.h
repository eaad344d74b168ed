// Internal declarations shared by the host runtime (psp_host.cpp) and the CUDA
// kernels (psp_kernels.cu).  Not part of the C ABI (include/psp.h is).
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

namespace psp {

// Lanes (perturbed systems) are padded to a multiple of kBlock = 32.  The factor
// kernel works on slabs of L = 32 / G lanes: one warp = G thread groups of L
// threads, all groups working on the SAME L lanes (each group takes a different
// subset of the independent updates of a pivot).  Batch-major arrays
// are laid out [slab][item][L]; the solve kernel's warp covers kBlock = 32 lanes =
// G consecutive factor slabs; X is [lane / 32][R][n][32].
constexpr int kBlock = 32;
// Source codes of the factor program: >= 0 pending slot; otherwise A[-1 - code] of A
// extended by one structural zero, A[nnz_A] = 0.
constexpr int kStages = 4;            // depth of the CTA-shared program ring (solve)
constexpr int kFMaxStages = 8;        // factor ring: 4 or 8 stages (LaunchInfo::f_stages)
constexpr int kYRows = 16;            // y rows per stage of the solve's y ring
constexpr int kDataStages = 2;        // depth of the solve's per-warp factor-row ring
constexpr int kSolveMaxC = 16;        // records with c <= kSolveMaxC take the unrolled path
constexpr int kMaxWarpsCta = 16;      // warps per CTA (all consumers: self-refilling ring)
constexpr int kFusedMax = 12;         // pivots with c <= kFusedMax: u in registers, no scratch
constexpr int kPairMax = 8;          // supernode pairs for c <= kPairMax
constexpr int kSpillCap = 127;        // capacity-planned programs: pending slots per lane (+ the
                                      // dummy = 128 slots = 256 TMEM columns, 2 CTAs per SM)

// Record types of the programs (bits 28..31 of a record's first word).
enum : uint32_t { kRecBirth = 1u, kRecPivot = 2u, kRecUpdate = 3u, kRecEnd = 4u, kRecYEnd = 5u,
                  kRecSpill = 6u, kRecReload = 7u };

// Device-side programs (see psp_plan.cpp for their meaning).
struct DevicePlan {
  int32_t n = 0, nnz_A = 0, nnz_LU = 0, nnz_L = 0, c_max = 0;
  const int32_t* perm = nullptr;       // [n]  perm[new] = old
  const int32_t* iperm = nullptr;      // [n]  iperm[old] = new
  const int32_t* adiag = nullptr;      // [n]  CSR index of A(perm[i], perm[i]) or -1
  // factor program (records packed in chunks of f_chunk_words)
  int32_t f_slots = 0, f_chunk_words = 0, f_nchunks = 0, c_scr = 0;  // c_scr: scratch rows
  const int32_t* f_stream = nullptr;   // the handle's patched copy (immediates filled in)
  int32_t f_npatch = 0;
  const int32_t* f_patch_pos = nullptr;
  const int32_t* f_patch_src = nullptr;
  int32_t f_aug = 0;                   // 1: program of [A | b] (y_p written to X)
  int32_t f_gspill = 0;                // capacity-planned program: spill entries per lane
  // solve program: forward (ascending) records, YEND, backward (descending) records, END
  int32_t y_slots = 0, x_slots = 0, s_chunk_words = 0, s_nchunks = 0;
  const int32_t* s_stream = nullptr;
  int32_t s_rows = 16, s_nfwd = 0, s_nfc = 0;   // ring stage rows; forward / all row chunks
  const int2* s_fchunks = nullptr;              // [s_nfc] row ranges [r0, r1)
  int32_t s_bwd_chunk = 0;                      // first chunk of the backward records
  // deterministic column sums for the default pivot tolerance
  const int32_t* acsc_ptr = nullptr;   // [n+1]
  const int32_t* acsc_q = nullptr;     // [nnz_A]
};

// Multi-Jacobian batches (many Jacobians of one pattern in one launch):
// lane k uses Jacobian jac(k) = k / lanes_per (0 = a single Jacobian): its values at
// A + jac * a_stride, its right-hand sides at B + jac * b_stride, its tolerance tol[jac].
struct MultiJac {
  int32_t lanes_per = 0;
  int64_t a_stride = 0, b_stride = 0;
  __host__ __device__ int jac(int k) const { return lanes_per > 0 ? k / lanes_per : 0; }
};

// Device copy of the level-scheduled plan of the cooperative small-batch kernels
// (psp_plan.h CoopPlan): one CTA per system, its factor image in shared memory.
struct CoopDev {
  int32_t steps = 0;
  const int32_t *birth_src = nullptr, *birth_diag = nullptr;
  // packed plans (uint32 words, 16-bit fields), copied into shared memory by each CTA:
  // factor: [fa_ptr, fp_ptr, fb_ptr][steps+1] | fa (l | d<<16) | fp (d | p<<16) |
  //         fbt (t | start<<16, + sentinel) | fbc (l | u<<16)
  // solve:  [ya_ptr, xb_ptr][steps+1] | yat (i | start<<16, + sentinel) | yac (l | p<<16) |
  //         xbr (r | start<<16, + sentinel) | xbd (u_pp position) | xbc (u | k<<16)
  const uint32_t *fplan = nullptr, *splan = nullptr;
  int32_t f_words = 0, fo_fa = 0, fo_fp = 0, fo_fbt = 0, fo_fbc = 0;
  int32_t s_words = 0, so_yat = 0, so_yac = 0, so_xbr = 0, so_xbd = 0, so_xbc = 0;
};
// Cooperative kernels: factor (births, per step: pivot checks + L columns, then the
// updates) and solve (forward, backward, R right-hand sides), V and X in the layouts of
// the batch kernels (LS lanes per factor slab).
cudaError_t launch_coop_factor(const DevicePlan& p, const CoopDev& c, const double* A,
                               const double* eps, const double* dperm, const double* tol_dev,
                               double tol_value, double* V, int32_t* status, int32_t K, int32_t LS,
                               cudaStream_t stream, MultiJac mj = MultiJac{});
cudaError_t launch_coop_solve(const DevicePlan& p, const CoopDev& c, const double* V, const double* B,
                              int64_t ldb, int32_t R, double* X, int32_t K, int32_t LS,
                              cudaStream_t stream, MultiJac mj = MultiJac{});
size_t coop_smem_bytes(const DevicePlan& p, const CoopDev& c, bool solve);
cudaError_t configure_coop(const DevicePlan& p, const CoopDev& c);

// Launch configuration chosen per plan (host, psp_kernels.cu: choose_launch).
struct LaunchInfo {
  // factor
  int f_groups = 1;            // G: thread groups per warp
  int f_lanes = 1;             // J: lanes per thread; a slab has LS = 32 / G * J lanes
  int f_slab_warps = 1;        // P: warps sharing one slab (rows split, named barriers)
  bool f_pend_smem = false;    // pending slots in shared memory (else global scratch)
  bool f_scr_smem = true;      // l/u scratch rows of large pivots in shared memory
  int f_warps = 1;             // consumer warps per CTA (f_warps / P slabs)
  int f_smem = 0;              // dynamic shared memory per CTA
  int f_off_warp = 0, f_warp_bytes = 0, f_off_scr = 0;
  int f_ctas_per_sm = 0;
  int f_stages = 4;            // program ring stages of the factor (4 or 8)
  bool f_tmem = false;         // (1, 1, 1) with warps 0..3 holding their slots in TMEM
  bool f_pair_lanes = false;   // compact TMEM kernel, 2 lanes (32-lane slabs) per thread
  bool f_hybrid = false;       // ... with every warp's slots split TMEM / shared memory (PendHyb)
  bool f_mix = false;          // factor_kernel_mix: TMEM warps x 2 lanes, shared-memory warps x 1 lane
  int f_off_tscr = 0;          // TMEM warps' scratch rows (shared memory)
  // solve
  bool s_live_smem = false;
  bool s_b_smem = true;        // b staged in shared memory (else read from global)
  int s_warps = 1;
  int s_smem = 0;
  int s_off_b = 0, s_off_warp = 0, s_warp_bytes = 0, s_off_data = 0;
  int s_ctas_per_sm = 0;
  bool s_tmem = false;         // live slots in tensor memory (solve_kernel_tmem)
  int s_yrows = 16;            // rows per stage of the solve's y ring
  int n_sm = 148;              // SMs of the device (a batch smaller than one round is
                               // spread over all of them with fewer warps per CTA)
  int s_tmem_cols = 0;         // TMEM columns allocated per CTA
};

// Kernel launchers (psp_kernels.cu).  All asynchronous on `stream`.
// force_groups: 0 = automatic, else G in {1, 2, 4, 8}; force_warps: 0 = automatic.
// Returns false when no configuration fits the shared memory (the program's records or
// the solve's working set are too large).
// force_tmem / force_solve_tmem: 0 = automatic, 1 = require the factor's / solve's TMEM
// variant, 2 = disable it.
bool choose_launch(const DevicePlan& p, LaunchInfo& li, int force_groups, int force_warps,
                   int force_lanes, int force_slab_warps, int force_tmem, int force_solve_tmem);
// mode: 0 / 2 default layout, 1 hybrid slot store, 3 mixed lanes per thread
bool choose_launch_spill(const DevicePlan& p, LaunchInfo& li, int force_warps, int mode = 0);
cudaError_t configure_kernels(const DevicePlan& p, LaunchInfo& li, int force_groups,
                              int force_warps, int force_lanes, int force_slab_warps,
                              int force_tmem, int force_solve_tmem);
// Fill the factor stream's immediates (A values, d, b for the augmented program) in
// `stream_out` (device copy).
cudaError_t launch_patch_program(const DevicePlan& p, int32_t* stream_out, const double* A_vals,
                                 const double* dperm, const double* b, cudaStream_t stream);
cudaError_t launch_patch_tol(const DevicePlan& p, int32_t* stream_out, const double* A_vals,
                             const double* dperm, const double* b, double* tol_out, cudaStream_t stream);
cudaError_t launch_pivot_tol(const DevicePlan& p, const double* A_vals, double* tol_out,
                             cudaStream_t stream, int32_t n_jac = 1);
cudaError_t launch_factor(const DevicePlan& p, const LaunchInfo& li, const int32_t* prog,
                          const double* eps, const double* tol_dev, double tol_value, double* V,
                          double* gscratch, double* gscr, int32_t* status, int32_t K_pad,
                          double* Y, double* gspill, cudaStream_t stream);
// g_k = max|U| / max|A_k| per lane, from the factor in V (growth monitoring)
cudaError_t launch_residual(int32_t n, const int32_t* row_ptr, const int32_t* col_idx,
                            const double* A, int32_t W, int32_t R, const double* B, const double* x,
                            double* res, cudaStream_t stream);
cudaError_t launch_growth(const DevicePlan& p, const LaunchInfo& li, const double* V, const double* A,
                          const uint8_t* isdiag, const double* eps, const double* dperm, int32_t K,
                          double* offmax_scratch, double* growth, cudaStream_t stream);
cudaError_t launch_solve(const DevicePlan& p, const LaunchInfo& li, const double* V,
                         const double* B, int64_t ldb, int32_t R, double* X, double* gscratch,
                         int32_t K_pad, bool forward, cudaStream_t stream);
cudaError_t launch_recover(const DevicePlan& p, int32_t W, int32_t R, const int32_t* w_ptr,
                           const int32_t* w_lane, const double* w_val, const double* X,
                           const int32_t* status, double* x_out, int32_t* infeasible_flag,
                           cudaStream_t stream);
cudaError_t launch_recover_uni(const DevicePlan& p, int32_t W, int32_t R, int32_t L,
                               const double* w_val, const double* X, const int32_t* status,
                               double* x_out, int32_t* flag, cudaStream_t stream);
cudaError_t launch_recover_seg(const DevicePlan& p, int32_t W, int32_t R, const int32_t* w_ptr,
                               const int32_t* w_lane, const double* w_val, const double* X,
                               const int32_t* status, double* x_out, int32_t* flag,
                               cudaStream_t stream);
// Iterative-refinement baseline: r = b - A x per lane ([K][n], original ordering), and
// x += (the correction in X, batch layout, R = 1).
cudaError_t launch_refine_step(const DevicePlan& p, int32_t K, const int32_t* row_ptr, const int32_t* col_idx,
                               const double* A, const double* b, const double* x, double* r, cudaStream_t stream);
cudaError_t launch_refine_update(const DevicePlan& p, int32_t K, const double* X, double* x, cudaStream_t stream);
// Structural transversal: dst[j][q'] = src[j * nnz + amap[q']] (n_jac value arrays), and
// dst[(j R + r) n + i] = src[j * jac_stride + r * ldb + q[i]] (compact B_hat, ldb' = n).
cudaError_t launch_gather_a(const int32_t* amap, int32_t nnz, int32_t n_jac, const double* src, double* dst,
                            cudaStream_t stream);
cudaError_t launch_gather_b(const int32_t* q, int32_t n, int32_t R, int32_t n_jac, const double* src, int64_t ldb,
                            int64_t jac_stride, double* dst, cudaStream_t stream);
cudaError_t launch_gather_solutions(const DevicePlan& p, int32_t K, int32_t R, const double* X,
                                    double* out, cudaStream_t stream);

}  // namespace psp
