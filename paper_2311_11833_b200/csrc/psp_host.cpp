// Host runtime of libpsp: C ABI (include/psp.h), symbolic analysis, device plans.
//
// Symbolic analysis ("a pivot/permutation
// sequence ... computed once, and perpetually reused"): the elimination order, the
// filled pattern of L+U for the symmetric pattern of A+A^T+I, the batch-major slot
// layout and the kernel plans are computed once per sparsity pattern on the host.
// The numeric work of every step of Alg. 1 runs in the CUDA kernels of
// psp_kernels.cu; nothing here touches a lane's values.
#include <dlfcn.h>
#include <nccl.h>   // types only: libnccl is loaded at run time (psp_nccl below)

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "../../include/psp.h"
#include "psp_internal.h"
#include "psp_coopg.h"
#include "psp_dataflow.h"
#include "psp_dense.h"
#include "psp_plan.h"

using psp::DevicePlan;
using psp::kBlock;
using psp::kSpillCap;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// NCCL, loaded on first use (dlopen "libnccl.so.2"; the process's already-loaded copy —
// e.g. torch's — when there is one): the library itself has no link-time NCCL dependency,
// so host-only and single-GPU use never need it.
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl_api() {
  static NcclApi api;
  if (!api.tried) {
    api.tried = true;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (lib) {
      api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(lib, "ncclGetUniqueId"));
      api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(lib, "ncclCommInitRank"));
      api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(lib, "ncclCommDestroy"));
      api.reduce = reinterpret_cast<decltype(api.reduce)>(dlsym(lib, "ncclReduce"));
      api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(lib, "ncclAllReduce"));
      api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(lib, "ncclGetErrorString"));
      api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.reduce && api.allReduce &&
               api.errorString;
    }
  }
  return api;
}

}  // namespace

struct psp_ctx {
  int device = 0;
  int n_sm = 148;                  // SMs of the device (wave counts of the solve launch)
  cudaStream_t stream = nullptr;
  std::string detail;

  // --- symbolic ---
  bool analysed = false;
  int32_t n = 0, nnz_A = 0, nnz_LU = 0, nnz_L = 0, n_levels = 0, n_struct_zero_diag = 0;
  int64_t factor_fma = 0, solve_fma = 0;
  int32_t max_live = 0, y_slots = 0, x_slots = 0, c_max = 0, f_births = 0;
  std::vector<int32_t> perm;
  std::vector<DevBuf> plan_bufs;
  DevicePlan plan;
  psp::LaunchInfo launch;
  // the solve with its live slots in TMEM (more warps per SM, more instructions per
  // row): used when it needs fewer waves than `launch`'s (PSP_OPT_SOLVE_TMEM = 0)
  psp::LaunchInfo launch_stm;
  bool stm_ok = false;
  // cooperative small-batch kernels (one CTA per system, level-scheduled)
  psp::CoopDev coop;
  bool coop_ok = false;
  int64_t opt_coop = 0;            // PSP_OPT_COOP: 0 automatic (K <= 8 * SMs), 1 on, 2 off
  // fused factor + solve by dataflow (psp_dataflow.cu): the small-batch, one-RHS latency path
  bool df_ok = false;
  int64_t opt_df = 0;              // PSP_OPT_DATAFLOW: 0 automatic (with the coop kernels), 1 on, 2 off
  const uint32_t* df_plan = nullptr;
  int32_t df_words = 0;
  size_t df_smem = 0;
  // level-scheduled kernels for large systems (CTA per system, factor image lane-major in
  // V_d: psp_coopg.cu), used when the cooperative kernels' shared-memory image does not fit
  psp::CoopGDev coopg;
  bool coopg_ok = false;
  int64_t opt_coopg = 0;           // PSP_OPT_COOP_GLOBAL: 0 automatic, 1 on, 2 off
  bool coopg_factored = false;     // the last factorisation ran them (V_d is lane-major)
  psp::MultiJac mj;                // multi-Jacobian layout of the last factorisation
  // structural transversal (PSP_OPT_TRANSVERSAL): the analysed matrix is the
  // row-permuted A_hat = A[q, :]; entry points gather A's values and b's rows into it
  int64_t opt_transversal = 0;
  bool transversal = false;
  std::vector<int32_t> tq;             // q[j] = row of A placed at row j
  const int32_t* tq_d = nullptr;       // plan buffers: q, and A_hat CSR index -> A CSR index
  const int32_t* tamap_d = nullptr;
  DevBuf tA_d, tB_d, tb2_d;            // gathered A_hat values, B_hat, refine's b_hat
  // program of the augmented matrix [A | b] (psp_factor_solve_batch); its own slots,
  // stream and factor launch configuration, the rest shared with `plan`
  DevicePlan plan_aug;
  psp::LaunchInfo launch_aug;
  bool aug_ok = false;
  bool aug_fast = false;   // the augmented program keeps the plain one's slot store (TMEM /
                           // shared / global): psp_factor_solve_batch fuses, else it runs
                           // the two calls (measured: a store downgrade costs more)
  // capacity-planned factor programs (plain and augmented): <= kSpillCap pending slots per
  // lane, idle entries spilled to a global area; the TMEM kernel at 2 CTAs per SM
  DevicePlan plan_spill, plan_spill_aug;
  psp::LaunchInfo launch_spill, launch_spill_aug;
  bool spill_ok = false, spill_aug_ok = false;
  int32_t dead_l = 0, dead_rows[2] = {0, 0};   // structural-zero multipliers; rows skipped [plain, aug]
  int32_t spill_stats[2][3] = {{0, 0, 0}, {0, 0, 0}};   // [plain, aug] x (spills, reloads, entries)
  int64_t opt_spill = 0;           // PSP_OPT_FACTOR_SPILL: 0 automatic, 1 require, 2 off
  int64_t opt_hybrid = 0;          // PSP_OPT_FACTOR_HYBRID: 0 automatic, 1 on, 2 off
  DevBuf gspill_d;
  int64_t opt_groups = 0, opt_warps = 0, opt_lanes = 0, opt_slab_warps = 0;  // PSP_OPT_FACTOR_*
  int64_t opt_skip_dead = 1;                                                  // PSP_OPT_SKIP_ZERO_ROWS
  int64_t opt_pairs = 1;                                                      // PSP_OPT_FACTOR_PAIRS
  int64_t opt_tmem = 0;                                                       // PSP_OPT_FACTOR_TMEM
  int64_t opt_solve_tmem = 0;                                                 // PSP_OPT_SOLVE_TMEM
  DevBuf fscratch_d, sscratch_d;   // global pending buffers when shared memory is too small
  DevBuf fscr_d;                   // global l/u scratch rows (large pivots) when needed
  // PSP_OPT_PHASE_EVENTS: event pairs around every factor / solve kernel launch since
  // the last psp_get_phase_times (pools grow on demand, reused after a read)
  bool phase_events = false;
  // PSP_OPT_GROWTH: per-lane growth g_k = max|U| / max|A_k| after every factorisation
  bool growth = false;
  DevBuf growth_d, offmax_d;
  const uint8_t* isdiag_d = nullptr;   // plan buffer: CSR entry is a diagonal entry
  const int32_t* rowptr_d = nullptr;   // plan buffers: the analysed CSR pattern (psp_residual)
  const int32_t* colidx_d = nullptr;
  DevBuf res_d;                        // psp_residual output
  DevBuf ref_r_d;                      // psp_refine: per-lane residuals [K][n]
  std::vector<cudaEvent_t> fev, sev;
  size_t nf = 0, ns = 0;

  // --- multi-GPU: this rank owns global lanes [k_begin, k_begin + K) of
  // K_global; the partial sums of psp_recover are reduced over `comm` ---
  ncclComm_t comm = nullptr;
  int32_t nranks = 1, rank = 0;
  int32_t K_global = 0, k_begin = 0;

  // --- perturbations ---
  int32_t K = 0, K_pad = 0;
  DevBuf eps_d, dperm_d, V_d, status_d, tol_d;
  bool factored = false;
  bool growth_valid = false;
  std::vector<double> d_host;   // D's diagonal, original ordering (psp_estimate_rho)
  std::vector<double> eps_host; // eps of the K lanes (psp_rescale_failed_rows)
  std::vector<int32_t> wptr_host, wlane_host;   // the stored weight rows (same)
  DevBuf rho_r_d, rho_x_d;      // psp_estimate_rho: right-hand side D v, recovered rows

  // --- solve ---
  int32_t R = 0;
  DevBuf X_d;
  bool solved = false;

  // --- weights ---
  int32_t W = 0;
  DevBuf wptr_d, wlane_d, wval_d, flag_d;
  // fast combination layout (every row a contiguous run of <= 16 lanes in one 32-lane block)
  bool w_seg = false;
  int32_t w_uni = 0;            // L when weight row w is lanes [w*L, w*L+L) for every w
  bool recovered = false;

  // --- dense path (PSP_OPT_PATH = PSP_PATH_DENSE, psp_dense.cu): the paper's dense
  // no-pivot getrf/trsm formulation on DMMA; also the only path for a dense D ---
  int64_t opt_path = 0;
  int32_t dense_N = 0;                 // n padded to a multiple of 32
  const int32_t* drp_d = nullptr;      // plan buffers: permuted CSR of A (row_ptr, col, src)
  const int32_t* dci_d = nullptr;
  const int32_t* dsrc_d = nullptr;
  bool dense_configured = false;
  DevBuf Md_d;                         // [K][N][N] dense factors
  DevBuf Dp_d;                         // P D P^T (n x n) when a dense D is set
  bool dense_D = false;
  std::vector<double> D_host;          // the dense D, original ordering (psp_estimate_rho)
  bool dense_factored = false;         // the last factorisation ran the dense path

  // kernels of the last numeric calls (psp_get_last_kernels)
  int32_t last_factor = 0, last_factor_aug = 0, last_solve = 0, last_solve_fwd = 0;

  // --- host-API staging ---
  DevBuf stageA_d, stageB_d, stageX_d;
  DevBuf stageA2_d, stageB2_d;              // (second input staging pair of the async pipeline)
  cudaStream_t in_stream = nullptr;         // the async pipeline's host -> device copies
  cudaEvent_t in_ready[2] = {nullptr, nullptr};
  bool x_ready_set[2] = {false, false};
  // psp_solve_host_async: x-hat staging double buffer, D2H on a copy stream
  DevBuf stageX2_d;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t x_ready[2] = {nullptr, nullptr}, x_copied[2] = {nullptr, nullptr};
  bool x_copied_set[2] = {false, false};
  int pipe = 0;
};

static psp_status fail(psp_ctx* h, psp_status s, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->detail = buf;
  }
  return s;
}

#define CUDA_TRY(h, expr)                                                                   \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(h, PSP_ERR_CUDA, "%s failed: %s (%d)", #expr, cudaGetErrorString(e_),     \
                  (int)e_);                                                                 \
  } while (0)

static psp_status ensure(psp_ctx* h, DevBuf& b, size_t bytes) {
  if (b.bytes >= bytes && b.p) return PSP_OK;
  b.release();
  if (bytes == 0) bytes = 8;
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    b.p = nullptr;
    return fail(h, PSP_ERR_ALLOC, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
  }
  b.bytes = bytes;
  return PSP_OK;
}

template <class T>
static psp_status upload(psp_ctx* h, const std::vector<T>& v, const T** out) {
  DevBuf b;
  psp_status s = ensure(h, b, sizeof(T) * std::max<size_t>(v.size(), 1));
  if (s) return s;
  if (!v.empty()) {
    cudaError_t e = cudaMemcpy(b.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      b.release();
      return fail(h, PSP_ERR_CUDA, "plan upload: %s", cudaGetErrorString(e));
    }
  }
  h->plan_bufs.push_back(b);
  *out = static_cast<const T*>(b.p);
  return PSP_OK;
}

static void release_plan(psp_ctx* h) {
  for (auto& b : h->plan_bufs) b.release();
  h->plan_bufs.clear();
  h->plan = DevicePlan{};
  h->isdiag_d = nullptr;
  h->rowptr_d = h->colidx_d = nullptr;
  h->drp_d = h->dci_d = h->dsrc_d = nullptr;
  h->tq_d = h->tamap_d = nullptr;
  h->transversal = false;
  h->tq.clear();
  h->dense_N = 0;
  h->dense_configured = false;
  h->Dp_d.release();
  h->dense_D = false;
  h->D_host.clear();
}

static void reset_numeric(psp_ctx* h) {
  h->eps_d.release();
  h->dperm_d.release();
  h->V_d.release();
  h->status_d.release();
  h->X_d.release();
  h->fscratch_d.release();
  h->fscr_d.release();
  h->gspill_d.release();
  h->sscratch_d.release();
  h->wptr_d.release();
  h->wlane_d.release();
  h->wval_d.release();
  h->w_seg = false;
  h->w_uni = 0;
  h->growth_d.release();
  h->offmax_d.release();
  h->Md_d.release();
  h->dense_factored = false;
  h->K = h->K_pad = h->R = h->W = 0;
  h->factored = h->solved = h->recovered = h->growth_valid = false;
}

extern "C" {

const char* psp_status_string(psp_status s) {
  switch (s) {
    case PSP_OK: return "PSP_OK";
    case PSP_ERR_ARG: return "PSP_ERR_ARG";
    case PSP_ERR_DIM: return "PSP_ERR_DIM";
    case PSP_ERR_STATE: return "PSP_ERR_STATE";
    case PSP_ERR_ZERO_PIVOT: return "PSP_ERR_ZERO_PIVOT";
    case PSP_ERR_BATCH_INFEASIBLE: return "PSP_ERR_BATCH_INFEASIBLE";
    case PSP_ERR_CUDA: return "PSP_ERR_CUDA";
    case PSP_ERR_ALLOC: return "PSP_ERR_ALLOC";
    case PSP_ERR_UNSUPPORTED: return "PSP_ERR_UNSUPPORTED";
    case PSP_ERR_NCCL: return "PSP_ERR_NCCL";
    case PSP_ERR_STRUCT_SINGULAR: return "PSP_ERR_STRUCT_SINGULAR";
    default: return "PSP_ERR_UNKNOWN";
  }
}

const char* psp_last_error_detail(psp_handle h) { return h ? h->detail.c_str() : "null handle"; }

psp_status psp_create(psp_handle* out, int32_t device, void* cuda_stream) {
  if (!out) return PSP_ERR_ARG;
  *out = nullptr;
  if (device < 0) {  // host-only handle: symbolic analysis and its info only
    psp_ctx* h = new (std::nothrow) psp_ctx();
    if (!h) return PSP_ERR_ALLOC;
    h->device = -1;
    *out = h;
    return PSP_OK;
  }
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || device < 0 || device >= count) {
    cudaGetLastError();
    return PSP_ERR_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) return PSP_ERR_CUDA;
  psp_ctx* h = new (std::nothrow) psp_ctx();
  if (!h) return PSP_ERR_ALLOC;
  h->device = device;
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  int nsm = 0;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && nsm > 0)
    h->n_sm = nsm;
  *out = h;
  return PSP_OK;
}

psp_status psp_destroy(psp_handle h) {
  if (!h) return PSP_ERR_ARG;
  if (h->device < 0) {
    delete h;
    return PSP_OK;
  }
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  release_plan(h);
  reset_numeric(h);
  h->tol_d.release();
  h->flag_d.release();
  h->stageA_d.release();
  h->stageB_d.release();
  h->stageA2_d.release();
  h->stageB2_d.release();
  if (h->in_stream) {
    cudaStreamSynchronize(h->in_stream);
    cudaStreamDestroy(h->in_stream);
    h->in_stream = nullptr;
  }
  for (int q = 0; q < 2; ++q) {
    if (h->in_ready[q]) cudaEventDestroy(h->in_ready[q]);
    h->in_ready[q] = nullptr;
    h->x_ready_set[q] = false;
  }
  h->stageX_d.release();
  h->stageX2_d.release();
  if (h->copy_stream) {
    cudaStreamSynchronize(h->copy_stream);
    cudaStreamDestroy(h->copy_stream);
  }
  for (int q = 0; q < 2; ++q) {
    if (h->x_ready[q]) cudaEventDestroy(h->x_ready[q]);
    if (h->x_copied[q]) cudaEventDestroy(h->x_copied[q]);
  }
  for (auto* v : {&h->fev, &h->sev})
    for (cudaEvent_t e : *v) cudaEventDestroy(e);
  if (h->comm) nccl_api().commDestroy(h->comm);
  delete h;
  return PSP_OK;
}

psp_status psp_set_option(psp_handle h, int32_t option, int64_t value) {
  if (!h) return PSP_ERR_ARG;
  switch (option) {
    case PSP_OPT_FACTOR_GROUPS:
      if (value != 0 && value != 1 && value != 2 && value != 4)
        return fail(h, PSP_ERR_ARG, "PSP_OPT_FACTOR_GROUPS must be 0, 1, 2 or 4");
      h->opt_groups = value;
      return PSP_OK;
    case PSP_OPT_FACTOR_LANES:
      if (value != 0 && value != 1 && value != 2)
        return fail(h, PSP_ERR_ARG, "PSP_OPT_FACTOR_LANES must be 0, 1 or 2");
      h->opt_lanes = value;
      return PSP_OK;
    case PSP_OPT_FACTOR_TMEM:
      if (value < 0 || value > 2) return fail(h, PSP_ERR_ARG, "PSP_OPT_FACTOR_TMEM must be 0, 1 or 2");
      h->opt_tmem = value;
      return PSP_OK;
    case PSP_OPT_COOP:
      if (value < 0 || value > 2) return fail(h, PSP_ERR_ARG, "PSP_OPT_COOP must be 0, 1 or 2");
      h->opt_coop = value;
      return PSP_OK;
    case PSP_OPT_COOP_GLOBAL:
      if (value < 0 || value > 2) return fail(h, PSP_ERR_ARG, "PSP_OPT_COOP_GLOBAL must be 0, 1 or 2");
      h->opt_coopg = value;
      return PSP_OK;
    case PSP_OPT_FACTOR_SPILL:
      if (value < 0 || value > 2) return fail(h, PSP_ERR_ARG, "PSP_OPT_FACTOR_SPILL must be 0, 1 or 2");
      h->opt_spill = value;
      return PSP_OK;
    case PSP_OPT_GROWTH:
      if (value != 0 && value != 1) return fail(h, PSP_ERR_ARG, "PSP_OPT_GROWTH must be 0 or 1");
      h->growth = value != 0;
      return PSP_OK;
    case PSP_OPT_PHASE_EVENTS:
      if (value != 0 && value != 1) return fail(h, PSP_ERR_ARG, "PSP_OPT_PHASE_EVENTS must be 0 or 1");
      if (value && h->device < 0) return fail(h, PSP_ERR_STATE, "host-only handle");
      h->phase_events = value != 0;
      h->nf = h->ns = 0;
      return PSP_OK;
    case PSP_OPT_SOLVE_TMEM:
      if (value < 0 || value > 2) return fail(h, PSP_ERR_ARG, "PSP_OPT_SOLVE_TMEM must be 0, 1 or 2");
      h->opt_solve_tmem = value;
      return PSP_OK;
    case PSP_OPT_FACTOR_PAIRS:
      if (value != 0 && value != 1) return fail(h, PSP_ERR_ARG, "PSP_OPT_FACTOR_PAIRS must be 0 or 1");
      h->opt_pairs = value;
      return PSP_OK;
    case PSP_OPT_SKIP_ZERO_ROWS:
      if (value != 0 && value != 1) return fail(h, PSP_ERR_ARG, "PSP_OPT_SKIP_ZERO_ROWS must be 0 or 1");
      h->opt_skip_dead = value;
      return PSP_OK;
    case PSP_OPT_FACTOR_SLAB_WARPS:
      if (value != 0 && value != 1 && value != 2)
        return fail(h, PSP_ERR_ARG, "PSP_OPT_FACTOR_SLAB_WARPS must be 0, 1 or 2");
      h->opt_slab_warps = value;
      return PSP_OK;
    case PSP_OPT_FACTOR_HYBRID:
      if (value < 0 || value > 3) return fail(h, PSP_ERR_ARG, "PSP_OPT_FACTOR_HYBRID must be 0, 1, 2 or 3");
      h->opt_hybrid = value;
      return PSP_OK;
    case PSP_OPT_DATAFLOW:
      if (value < 0 || value > 2) return fail(h, PSP_ERR_ARG, "PSP_OPT_DATAFLOW must be 0, 1 or 2");
      h->opt_df = value;
      return PSP_OK;
    case PSP_OPT_TRANSVERSAL:
      if (value != 0 && value != 1) return fail(h, PSP_ERR_ARG, "PSP_OPT_TRANSVERSAL must be 0 or 1");
      h->opt_transversal = value;
      return PSP_OK;
    case PSP_OPT_PATH:
      if (value != PSP_PATH_SPARSE && value != PSP_PATH_DENSE)
        return fail(h, PSP_ERR_ARG, "PSP_OPT_PATH must be PSP_PATH_SPARSE or PSP_PATH_DENSE");
      h->opt_path = value;
      return PSP_OK;
    case PSP_OPT_FACTOR_WARPS:
      if (value < 0 || value > psp::kMaxWarpsCta)
        return fail(h, PSP_ERR_ARG, "PSP_OPT_FACTOR_WARPS must be in [0, %d]", psp::kMaxWarpsCta);
      h->opt_warps = value;
      return PSP_OK;
    default:
      return fail(h, PSP_ERR_ARG, "unknown option %d", option);
  }
}

psp_status psp_set_stream(psp_handle h, void* cuda_stream) {
  if (!h) return PSP_ERR_ARG;
  // the programs, factor and staging buffers are reused by the next call: finish the work
  // queued on the old stream before a call on the new one can overwrite them
  if (h->device >= 0) {
    cudaSetDevice(h->device);
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  }
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  return PSP_OK;
}

psp_status psp_synchronize(psp_handle h) {
  if (!h) return PSP_ERR_ARG;
  if (h->device < 0) return PSP_OK;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  if (h->copy_stream) CUDA_TRY(h, cudaStreamSynchronize(h->copy_stream));
  return PSP_OK;
}

psp_status psp_solve_host_async(psp_handle h, const double* A_vals_h, int32_t R, const double* B_h,
                                double pivot_tol, double* x_h) {
  if (!h || !A_vals_h || !B_h || !x_h || R < 1) return PSP_ERR_ARG;
  if (h->K == 0 || h->W == 0) return fail(h, PSP_ERR_STATE, "set_perturbations and set_weights first");
  cudaSetDevice(h->device);
  psp_status s;
  if (!h->copy_stream) {
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->in_stream, cudaStreamNonBlocking));
    for (int q = 0; q < 2; ++q) {
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->x_ready[q], cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->in_ready[q], cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->x_copied[q], cudaEventDisableTiming));
    }
  }
  const int q = h->pipe;
  DevBuf& xs = q ? h->stageX2_d : h->stageX_d;
  const size_t xbytes = sizeof(double) * (size_t)h->W * R * h->n;
  DevBuf& sa = q ? h->stageA2_d : h->stageA_d;
  DevBuf& sb = q ? h->stageB2_d : h->stageB_d;
  if (xs.bytes < xbytes || sa.bytes < sizeof(double) * h->nnz_A ||
      sb.bytes < sizeof(double) * (size_t)h->n * R) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->copy_stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->in_stream));
    if ((s = ensure(h, sa, sizeof(double) * h->nnz_A))) return s;
    if ((s = ensure(h, sb, sizeof(double) * (size_t)h->n * R))) return s;
    if ((s = ensure(h, xs, xbytes))) return s;
  }
  // the buffer's previous copy to the host must be done before recover overwrites it
  if (h->x_copied_set[q]) CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->x_copied[q], 0));
  // the inputs travel on their own stream into this step's staging pair, so that their
  // copies overlap the previous call's kernels; the pair was last read by the call two
  // steps back (everything up to its x_ready event)
  if (h->x_ready_set[q]) CUDA_TRY(h, cudaStreamWaitEvent(h->in_stream, h->x_ready[q], 0));
  CUDA_TRY(h, cudaMemcpyAsync(sa.p, A_vals_h, sizeof(double) * h->nnz_A, cudaMemcpyHostToDevice,
                              h->in_stream));
  CUDA_TRY(h, cudaMemcpyAsync(sb.p, B_h, sizeof(double) * (size_t)h->n * R, cudaMemcpyHostToDevice,
                              h->in_stream));
  CUDA_TRY(h, cudaEventRecord(h->in_ready[q], h->in_stream));
  CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->in_ready[q], 0));
  if (R == 1) {
    if ((s = psp_factor_solve_batch(h, (const double*)sa.p, (const double*)sb.p, pivot_tol, nullptr)))
      return s;
  } else {
    if ((s = psp_factor_batch(h, (const double*)sa.p, pivot_tol, nullptr))) return s;
    if ((s = psp_solve_batch(h, R, (const double*)sb.p, h->n))) return s;
  }
  if ((s = psp_recover(h, (double*)xs.p))) return s;
  CUDA_TRY(h, cudaEventRecord(h->x_ready[q], h->stream));
  h->x_ready_set[q] = true;
  CUDA_TRY(h, cudaStreamWaitEvent(h->copy_stream, h->x_ready[q], 0));
  CUDA_TRY(h, cudaMemcpyAsync(x_h, xs.p, xbytes, cudaMemcpyDeviceToHost, h->copy_stream));
  CUDA_TRY(h, cudaEventRecord(h->x_copied[q], h->copy_stream));
  h->x_copied_set[q] = true;
  h->pipe ^= 1;
  return PSP_OK;
}

psp_status psp_symbolic_analyse(psp_handle h, int32_t n, const int32_t* row_ptr_h,
                                const int32_t* col_idx_h, int32_t ordering,
                                const int32_t* user_perm_h, int32_t first_node) {
  if (!h) return PSP_ERR_ARG;
  if (n < 1 || !row_ptr_h || (row_ptr_h[n] > 0 && !col_idx_h))
    return fail(h, PSP_ERR_ARG, "bad pattern arguments");
  if (row_ptr_h[0] != 0) return fail(h, PSP_ERR_ARG, "row_ptr[0] must be 0");
  for (int32_t i = 0; i < n; ++i) {
    if (row_ptr_h[i + 1] < row_ptr_h[i]) return fail(h, PSP_ERR_ARG, "row_ptr not monotone");
    for (int32_t q = row_ptr_h[i]; q < row_ptr_h[i + 1]; ++q) {
      int32_t c = col_idx_h[q];
      if (c < 0 || c >= n) return fail(h, PSP_ERR_ARG, "column index out of range");
      if (q > row_ptr_h[i] && c <= col_idx_h[q - 1])
        return fail(h, PSP_ERR_ARG, "column indices must be strictly increasing per row");
    }
  }
  if (ordering < PSP_ORDER_NATURAL || ordering > PSP_ORDER_MINDEG_FIRST)
    return fail(h, PSP_ERR_ARG, "unknown ordering %d", ordering);
  if (ordering == PSP_ORDER_MINDEG_FIRST && (first_node < 0 || first_node >= n))
    return fail(h, PSP_ERR_ARG, "first_node out of range");
  if (ordering == PSP_ORDER_USER) {
    if (!user_perm_h) return fail(h, PSP_ERR_ARG, "USER ordering needs user_perm_h");
    std::vector<char> seen(n, 0);
    for (int32_t i = 0; i < n; ++i) {
      int32_t v = user_perm_h[i];
      if (v < 0 || v >= n || seen[v]) return fail(h, PSP_ERR_ARG, "user_perm is not a permutation");
      seen[v] = 1;
    }
  }
  const bool host_only = h->device < 0;
  if (!host_only) {
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
  }
  release_plan(h);
  reset_numeric(h);
  h->analysed = false;

  // structural transversal: analyse A_hat = A[q, :] (zero-free diagonal) instead of A
  std::vector<int32_t> t_rp, t_ci, t_amap, t_q;
  if (h->opt_transversal) {
    t_q = psp::transversal_hk(n, row_ptr_h, col_idx_h);
    int32_t matched = 0;
    for (int32_t j = 0; j < n; ++j) matched += t_q[j] >= 0;
    if (matched < n)
      return fail(h, PSP_ERR_STRUCT_SINGULAR, "structurally singular: a maximum matching covers %d of %d columns",
                  matched, n);
    t_rp.assign(n + 1, 0);
    for (int32_t j = 0; j < n; ++j) {
      const int32_t r = t_q[j];
      for (int32_t q = row_ptr_h[r]; q < row_ptr_h[r + 1]; ++q) {
        t_ci.push_back(col_idx_h[q]);
        t_amap.push_back(q);
      }
      t_rp[j + 1] = (int32_t)t_ci.size();
    }
    row_ptr_h = t_rp.data();
    col_idx_h = t_ci.data();
  }

  const int32_t nnzA = row_ptr_h[n];
  // symmetric adjacency of A + A^T (no self loops), original numbering
  std::vector<std::vector<int32_t>> adj(n);
  int32_t nzd = 0;
  for (int32_t i = 0; i < n; ++i) {
    bool has_diag = false;
    for (int32_t q = row_ptr_h[i]; q < row_ptr_h[i + 1]; ++q) {
      int32_t j = col_idx_h[q];
      if (j == i) {
        has_diag = true;
        continue;
      }
      adj[i].push_back(j);
      adj[j].push_back(i);
    }
    if (!has_diag) ++nzd;
  }
  for (auto& a : adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }

  std::vector<int32_t> perm(n);
  if (ordering == PSP_ORDER_NATURAL) {
    for (int32_t i = 0; i < n; ++i) perm[i] = i;
  } else if (ordering == PSP_ORDER_USER) {
    perm.assign(user_perm_h, user_perm_h + n);
  } else {
    const int32_t first = ordering == PSP_ORDER_MINDEG_FIRST ? first_node : -1;
    std::vector<int32_t> perm0 = psp::min_degree_order(n, adj, first);
    std::vector<int32_t> inv0(n);
    for (int32_t i = 0; i < n; ++i) inv0[perm0[i]] = i;
    std::vector<std::vector<int32_t>> adj0(n);
    for (int32_t i = 0; i < n; ++i) {
      for (int32_t j : adj[perm0[i]]) adj0[i].push_back(inv0[j]);
      std::sort(adj0[i].begin(), adj0[i].end());
    }
    psp::EtreeResult S0 = psp::symbolic_etree(n, adj0);
    std::vector<int32_t> post = psp::postorder_big_first(n, S0);
    for (int32_t i = 0; i < n; ++i) perm[i] = perm0[post[i]];
    if (first >= 0) {  // the forced-first vertex is an etree leaf: moving it to the front
      perm.erase(std::find(perm.begin(), perm.end(), first));  // keeps a topological order
      perm.insert(perm.begin(), first);
    }
  }
  std::vector<int32_t> inv(n);
  for (int32_t i = 0; i < n; ++i) inv[perm[i]] = i;

  std::vector<std::vector<int32_t>> adjp(n);
  for (int32_t i = 0; i < n; ++i) {
    for (int32_t j : adj[perm[i]]) adjp[i].push_back(inv[j]);
    std::sort(adjp[i].begin(), adjp[i].end());
  }
  psp::EtreeResult S = psp::symbolic_etree(n, adjp);
  int64_t nnzLU64 = n;
  for (int32_t j = 0; j < n; ++j) nnzLU64 += 2 * (int64_t)S.lcol[j].size();
  if (nnzLU64 > INT32_MAX / 2) return fail(h, PSP_ERR_ARG, "pattern too large");

  psp::HostPlan HP, HPa;
  HP.fuse_pairs = HPa.fuse_pairs = h->opt_pairs != 0;
  HP.skip_dead = HPa.skip_dead = h->opt_skip_dead != 0;
  HPa.aug = true;
  psp::build_programs(n, S.lcol, perm, row_ptr_h, col_idx_h, HP);
  psp::build_programs(n, S.lcol, perm, row_ptr_h, col_idx_h, HPa);
  if (!HP.plan_ok || !HPa.plan_ok)
    return fail(h, PSP_ERR_UNSUPPORTED, "internal: factor program failed its slot self-check");
  // capacity-planned programs (spills) for the 2-CTA TMEM factor kernel
  psp::HostPlan HPc, HPac;
  HPc.fuse_pairs = HPac.fuse_pairs = h->opt_pairs != 0;
  HPc.skip_dead = HPac.skip_dead = h->opt_skip_dead != 0;
  HPac.aug = true;
  HPc.cap = HPac.cap = kSpillCap;
  HPc.all_slots = HPac.all_slots = true;
  const bool try_spill = h->opt_spill != 2 && (HP.f_slots > kSpillCap + 1 || h->opt_spill == 1);
  if (try_spill) {
    psp::build_programs(n, S.lcol, perm, row_ptr_h, col_idx_h, HPc);
    psp::build_programs(n, S.lcol, perm, row_ptr_h, col_idx_h, HPac);
    if (!HPc.plan_ok || !HPac.plan_ok)
      return fail(h, PSP_ERR_UNSUPPORTED, "internal: capacity-planned program failed its slot self-check");
  }
  psp::CoopPlan CP;
  psp::build_coop(n, S.lcol, perm, row_ptr_h, col_idx_h, HP, CP);

  // CSC grouping of A's entries (original numbering) for the deterministic 1-norm
  std::vector<int32_t> acsc_ptr(n + 1, 0), acsc_q(nnzA);
  for (int32_t q = 0; q < nnzA; ++q) acsc_ptr[col_idx_h[q] + 1]++;
  for (int32_t c = 0; c < n; ++c) acsc_ptr[c + 1] += acsc_ptr[c];
  {
    std::vector<int32_t> fillp(acsc_ptr.begin(), acsc_ptr.end() - 1);
    for (int32_t r = 0; r < n; ++r)
      for (int32_t q = row_ptr_h[r]; q < row_ptr_h[r + 1]; ++q) acsc_q[fillp[col_idx_h[q]]++] = q;
  }

  DevicePlan P;
  P.n = n;
  P.nnz_A = nnzA;
  P.nnz_LU = HP.nnz_LU;
  P.nnz_L = HP.nnz_L;
  P.c_max = HP.c_max;
  P.f_slots = HP.f_slots;
  P.f_chunk_words = HP.f_chunk_words;
  P.f_nchunks = (int32_t)(HP.f_stream.size() / HP.f_chunk_words);
  P.c_scr = HP.c_max > psp::kFusedMax ? (HP.c_max + 3) & ~3 : 0;   // (rows padded to 4)
  P.f_npatch = (int32_t)HP.f_patch_pos.size();
  P.y_slots = HP.y_slots;
  P.x_slots = HP.x_slots;
  P.s_chunk_words = HP.s_chunk_words;
  P.s_nchunks = (int32_t)(HP.s_stream.size() / HP.s_chunk_words);
  P.s_rows = HP.s_rows;
  P.s_nfwd = HP.s_nfwd;
  P.s_nfc = (int32_t)HP.s_fchunks.size() / 2;
  P.s_bwd_chunk = HP.s_bwd_chunk;
  psp_status s;
#define UP(vec, field) \
  if (!host_only && (s = upload(h, vec, &P.field))) return s;
  UP(perm, perm);
  std::vector<int32_t> iperm(n);
  for (int32_t i = 0; i < n; ++i) iperm[perm[i]] = i;
  UP(iperm, iperm);
  UP(HP.adiag, adiag);
  UP(HP.f_stream, f_stream);   // patched in place with A and d before every factorisation
  UP(HP.f_patch_pos, f_patch_pos);
  UP(HP.f_patch_src, f_patch_src);
  UP(HP.s_stream, s_stream);
  if (!host_only) {
    const int32_t* fc = nullptr;
    if ((s = upload(h, HP.s_fchunks, &fc))) return s;
    P.s_fchunks = reinterpret_cast<const int2*>(fc);
  }
  UP(acsc_ptr, acsc_ptr);
  UP(acsc_q, acsc_q);
  {
    std::vector<uint8_t> isdiag(std::max(nnzA, 1), 0);
    for (int32_t r = 0; r < n; ++r)
      for (int32_t q = row_ptr_h[r]; q < row_ptr_h[r + 1]; ++q) isdiag[q] = col_idx_h[q] == r;
    if (!host_only && (s = upload(h, isdiag, &h->isdiag_d))) return s;
    std::vector<int32_t> rp(row_ptr_h, row_ptr_h + n + 1), ci(col_idx_h, col_idx_h + nnzA);
    if (ci.empty()) ci.push_back(0);
    if (!host_only && (s = upload(h, rp, &h->rowptr_d))) return s;
    if (!host_only && (s = upload(h, ci, &h->colidx_d))) return s;
  }
#undef UP
  if (!psp::choose_launch(P, h->launch, (int)h->opt_groups, (int)h->opt_warps,
                          (int)h->opt_lanes, (int)h->opt_slab_warps, (int)h->opt_tmem,
                          (int)h->opt_solve_tmem))
    return fail(h, PSP_ERR_UNSUPPORTED, "no kernel configuration fits shared memory "
                "(program chunk %d words, c_max %d, solve live slots %d)", P.f_chunk_words,
                P.c_max, P.y_slots + P.x_slots);
  if (!host_only)
    CUDA_TRY(h, psp::configure_kernels(P, h->launch, (int)h->opt_groups, (int)h->opt_warps,
                                        (int)h->opt_lanes, (int)h->opt_slab_warps, (int)h->opt_tmem,
                          (int)h->opt_solve_tmem));
  h->coop_ok = false;
  h->coop = psp::CoopDev{};
  if (!host_only) {
    // packed plans (16-bit fields): positions, rows and contribution counts must fit
    const size_t nc = std::max({CP.fb_l.size(), CP.ya_l.size(), CP.xb_u.size()});
    bool fits = P.nnz_LU < 65536 && n < 65536 && nc < 65536;
    std::vector<uint32_t> fw, sw;
    psp::CoopDev& c = h->coop;
    if (fits) {
      const int32_t S1 = CP.steps + 1;
      auto add_ptr = [](std::vector<uint32_t>& w, const std::vector<int32_t>& ptr) {
        for (int32_t x : ptr) w.push_back((uint32_t)x);
      };
      auto pack = [](std::vector<uint32_t>& w, const std::vector<int32_t>& lo, const std::vector<int32_t>& hi) {
        for (size_t q = 0; q < lo.size(); ++q) w.push_back((uint32_t)lo[q] | ((uint32_t)hi[q] << 16));
      };
      auto pad4 = [](std::vector<uint32_t>& w) { while (w.size() % 4) w.push_back(0); };
      add_ptr(fw, CP.fa_ptr); add_ptr(fw, CP.fp_ptr); add_ptr(fw, CP.fb_ptr);
      pad4(fw); c.fo_fa = (int32_t)fw.size(); pack(fw, CP.fa_l, CP.fa_d);
      pad4(fw); c.fo_fp = (int32_t)fw.size(); pack(fw, CP.fp_d, CP.fp_p);
      pad4(fw); c.fo_fbt = (int32_t)fw.size();
      {
        std::vector<int32_t> start(CP.fb_cptr.begin(), CP.fb_cptr.end() - 1);
        pack(fw, CP.fb_t, start);
        fw.push_back((uint32_t)CP.fb_cptr.back() << 16);   // sentinel: end of the last target
      }
      pad4(fw); c.fo_fbc = (int32_t)fw.size(); pack(fw, CP.fb_l, CP.fb_u);
      pad4(fw); c.f_words = (int32_t)fw.size();
      add_ptr(sw, CP.ya_ptr); add_ptr(sw, CP.xb_ptr);
      pad4(sw); c.so_yat = (int32_t)sw.size();
      {
        std::vector<int32_t> start(CP.ya_cptr.begin(), CP.ya_cptr.end() - 1);
        pack(sw, CP.ya_t, start);
        sw.push_back((uint32_t)CP.ya_cptr.back() << 16);
      }
      pad4(sw); c.so_yac = (int32_t)sw.size(); pack(sw, CP.ya_l, CP.ya_p);
      pad4(sw); c.so_xbr = (int32_t)sw.size();
      {
        std::vector<int32_t> start(CP.xb_cptr.begin(), CP.xb_cptr.end() - 1);
        pack(sw, CP.xb_r, start);
        sw.push_back((uint32_t)CP.xb_cptr.back() << 16);
      }
      pad4(sw); c.so_xbd = (int32_t)sw.size();
      for (int32_t d : CP.xb_d) sw.push_back((uint32_t)d);
      pad4(sw); c.so_xbc = (int32_t)sw.size(); pack(sw, CP.xb_u, CP.xb_k);
      pad4(sw); c.s_words = (int32_t)sw.size();
      (void)S1;
      c.steps = CP.steps;
      // (the kernels' static shared memory, a few words, counts against the same 227 KB)
      fits = psp::coop_smem_bytes(P, c, false) <= (size_t)(227 * 1024 - 256) &&
             psp::coop_smem_bytes(P, c, true) <= (size_t)(227 * 1024 - 256);
    }
    if (fits) {
      if ((s = upload(h, CP.birth_src, &c.birth_src))) return s;
      if ((s = upload(h, CP.birth_diag, &c.birth_diag))) return s;
      if ((s = upload(h, fw, &c.fplan))) return s;
      if ((s = upload(h, sw, &c.splan))) return s;
      if (psp::configure_coop(P, c) == cudaSuccess) {
        h->coop_ok = true;
      } else {   // (an unusable configuration only disables the cooperative path)
        cudaGetLastError();
        c = psp::CoopDev{};
      }
    } else {
      c = psp::CoopDev{};
    }
  }
  h->df_ok = false;
  h->df_plan = nullptr;
  if (!host_only && h->coop_ok && h->opt_df != 2) {
    psp::DataflowPlan DF;
    psp::build_dataflow(n, S.lcol, HP, psp::kDfWorkers, DF);
    const size_t smem = DF.ok ? psp::dataflow_smem(HP.nnz_LU, n, (int)DF.words.size()) : 0;
    if (DF.ok && smem <= (size_t)(227 * 1024 - 64)) {
      if ((s = upload(h, DF.words, &h->df_plan))) return s;
      h->df_words = (int32_t)DF.words.size();
      h->df_smem = smem;
      if (psp::configure_dataflow(smem) == cudaSuccess) {
        h->df_ok = true;
      } else {
        cudaGetLastError();
      }
    }
  }
  h->coopg_ok = false;
  h->coopg = psp::CoopGDev{};
  if (!host_only && h->opt_coopg != 2 && (!h->coop_ok || h->opt_coopg == 1)) {
    psp::CoopGDev& g = h->coopg;
    auto pairs = [](const std::vector<int32_t>& x, const std::vector<int32_t>& y) {
      std::vector<int2> v(x.size());
      for (size_t q = 0; q < x.size(); ++q) v[q] = make_int2(x[q], y[q]);
      return v;
    };
    auto heads = [](const std::vector<int32_t>& t, const std::vector<int32_t>& cptr) {
      std::vector<int2> v(t.size() + 1);
      for (size_t q = 0; q < t.size(); ++q) v[q] = make_int2(t[q], cptr[q]);
      v[t.size()] = make_int2(0, cptr.back());   // sentinel: end of the last one
      return v;
    };
    g.steps = CP.steps;
    g.nnz_LU = HP.nnz_LU;
    g.n = n;
    if ((s = upload(h, CP.birth_src, &g.birth_src))) return s;
    if ((s = upload(h, CP.birth_diag, &g.birth_diag))) return s;
    if ((s = upload(h, CP.fa_ptr, &g.fa_ptr))) return s;
    if ((s = upload(h, CP.fp_ptr, &g.fp_ptr))) return s;
    if ((s = upload(h, CP.fb_ptr, &g.fb_ptr))) return s;
    if ((s = upload(h, pairs(CP.fa_l, CP.fa_d), &g.fa))) return s;
    if ((s = upload(h, pairs(CP.fp_d, CP.fp_p), &g.fp))) return s;
    if ((s = upload(h, heads(CP.fb_t, CP.fb_cptr), &g.fbt))) return s;
    if ((s = upload(h, pairs(CP.fb_l, CP.fb_u), &g.fbc))) return s;
    if ((s = upload(h, CP.ya_ptr, &g.ya_ptr))) return s;
    if ((s = upload(h, CP.xb_ptr, &g.xb_ptr))) return s;
    if ((s = upload(h, heads(CP.ya_t, CP.ya_cptr), &g.yat))) return s;
    if ((s = upload(h, pairs(CP.ya_l, CP.ya_p), &g.yac))) return s;
    if ((s = upload(h, heads(CP.xb_r, CP.xb_cptr), &g.xbr))) return s;
    if ((s = upload(h, CP.xb_d, &g.xbd))) return s;
    if ((s = upload(h, pairs(CP.xb_u, CP.xb_k), &g.xbc))) return s;
    if (psp::coopg_solve_smem(n) <= (size_t)(227 * 1024) && psp::configure_coopg(n) == cudaSuccess) {
      h->coopg_ok = true;
    } else {
      cudaGetLastError();
      g = psp::CoopGDev{};
    }
  }
  h->stm_ok = false;
  if (h->opt_solve_tmem == 0) {
    psp::LaunchInfo ls = h->launch;
    if (psp::choose_launch(P, ls, (int)h->opt_groups, (int)h->opt_warps, (int)h->opt_lanes,
                           (int)h->opt_slab_warps, (int)h->opt_tmem, 1)) {
      h->launch_stm = ls;
      h->stm_ok = true;
    }
  }
  // the augmented program: same layout and solve; its own factor stream, slots, launch
  DevicePlan Pa = P;
  Pa.f_aug = 1;
  Pa.f_slots = HPa.f_slots;
  Pa.f_chunk_words = HPa.f_chunk_words;
  Pa.f_nchunks = (int32_t)(HPa.f_stream.size() / HPa.f_chunk_words);
  Pa.c_scr = HP.c_max + 1 > psp::kFusedMax ? (HP.c_max + 4) & ~3 : 0;
  Pa.f_npatch = (int32_t)HPa.f_patch_pos.size();
  psp::LaunchInfo la = h->launch;
  // (the augmented factor kernels exist for G = J = P = 1 only, and the factor they write
  // must have the plain launch's lane layout — V[slab][item][LS], LS = 32 / G * J — that
  // the solve, psp_get_factor and the growth pass read: only when the plain launch is
  // (1, 1, 1) too)
  h->aug_ok = h->launch.f_groups == 1 && h->launch.f_lanes == 1 && h->launch.f_slab_warps == 1 &&
              psp::choose_launch(Pa, la, 1, (int)h->opt_warps, 1, 1, (int)h->opt_tmem, 2);
  if (h->aug_ok && !host_only) {   // (its stream is patched in place, like plan's)
    if ((s = upload(h, HPa.f_stream, &Pa.f_stream))) return s;
    if ((s = upload(h, HPa.f_patch_pos, &Pa.f_patch_pos))) return s;
    if ((s = upload(h, HPa.f_patch_src, &Pa.f_patch_src))) return s;
  }
  h->plan_aug = Pa;
  h->launch_aug = la;
  // capacity-planned variants (same V layout as the (1, 1, 1) launches: 32-lane slabs)
  h->spill_ok = h->spill_aug_ok = false;
  std::memset(h->spill_stats, 0, sizeof h->spill_stats);
  h->dead_l = HP.f_dead_l;
  h->dead_rows[0] = h->dead_rows[1] = 0;
  if (try_spill && h->launch.f_groups == 1 && h->launch.f_lanes == 1 && h->launch.f_slab_warps == 1) {
    for (int q = 0; q < 2; ++q) {
      const psp::HostPlan& H = q ? HPac : HPc;
      DevicePlan Pc = q ? Pa : P;
      Pc.f_slots = H.f_slots;
      Pc.f_chunk_words = H.f_chunk_words;
      Pc.f_nchunks = (int32_t)(H.f_stream.size() / H.f_chunk_words);
      Pc.c_scr = (H.c_scr_need + 3) & ~3;   // (scratch rows padded to 4: the compact
                                             // update reads its columns in batches of 4)
      Pc.f_npatch = (int32_t)H.f_patch_pos.size();
      Pc.f_gspill = H.f_gspill;
      psp::LaunchInfo lc = h->launch;
      if (!psp::choose_launch_spill(Pc, lc, (int)h->opt_warps, (int)h->opt_hybrid)) continue;
      if (!host_only) {
        if ((s = upload(h, H.f_stream, &Pc.f_stream))) return s;
        if ((s = upload(h, H.f_patch_pos, &Pc.f_patch_pos))) return s;
        if ((s = upload(h, H.f_patch_src, &Pc.f_patch_src))) return s;
      }
      (q ? h->plan_spill_aug : h->plan_spill) = Pc;
      (q ? h->launch_spill_aug : h->launch_spill) = lc;
      (q ? h->spill_aug_ok : h->spill_ok) = true;
      h->spill_stats[q][0] = H.f_spills;
      h->spill_stats[q][1] = H.f_reloads;
      h->spill_stats[q][2] = H.f_gspill;
      h->dead_rows[q] = H.f_dead_rows;
    }
  }
  if (h->opt_spill == 1 && !h->spill_ok)
    return fail(h, PSP_ERR_UNSUPPORTED, "PSP_OPT_FACTOR_SPILL = 1 but no capacity-planned launch fits");
  {
    auto store = [](const psp::LaunchInfo& li) { return li.f_tmem ? 2 : (li.f_pend_smem ? 1 : 0); };
    h->aug_fast = h->aug_ok && store(la) == store(h->launch);
  }
  if (!host_only) {   // the dense path's permuted CSR: row i of P A P^T, ascending columns
    std::vector<int32_t> ip(n), drp(n + 1, 0), dci, dsrc;
    for (int32_t i = 0; i < n; ++i) ip[perm[i]] = i;
    dci.reserve(nnzA);
    dsrc.reserve(nnzA);
    std::vector<std::pair<int32_t, int32_t>> row;
    for (int32_t i = 0; i < n; ++i) {
      const int32_t o = perm[i];
      row.clear();
      for (int32_t q = row_ptr_h[o]; q < row_ptr_h[o + 1]; ++q) row.emplace_back(ip[col_idx_h[q]], q);
      std::sort(row.begin(), row.end());
      for (auto& e : row) {
        dci.push_back(e.first);
        dsrc.push_back(e.second);
      }
      drp[i + 1] = (int32_t)dci.size();
    }
    if ((s = upload(h, drp, &h->drp_d))) return s;
    if ((s = upload(h, dci, &h->dci_d))) return s;
    if ((s = upload(h, dsrc, &h->dsrc_d))) return s;
    h->dense_N = psp::dense_padded_order(n);
  }
  if (h->opt_transversal) {
    if (!host_only) {
      if ((s = upload(h, t_q, &h->tq_d))) return s;
      if ((s = upload(h, t_amap, &h->tamap_d))) return s;
    }
    h->tq = t_q;
    h->transversal = true;
  }
  h->plan = P;
  h->perm = perm;
  h->n = n;
  h->nnz_A = nnzA;
  h->nnz_LU = HP.nnz_LU;
  h->nnz_L = HP.nnz_L;
  h->n_levels = S.height;
  h->n_struct_zero_diag = nzd;
  h->factor_fma = HP.factor_fma;
  h->solve_fma = HP.solve_fma;
  h->max_live = HP.f_slots;
  h->y_slots = HP.y_slots;
  h->x_slots = HP.x_slots;
  h->c_max = HP.c_max;
  h->f_births = HP.f_births;
  h->analysed = true;
  return PSP_OK;
}

psp_status psp_get_symbolic_info(psp_handle h, psp_symbolic_info* info, int32_t* perm_h) {
  if (!h || !info) return PSP_ERR_ARG;
  if (!h->analysed) return fail(h, PSP_ERR_STATE, "not analysed");
  info->n = h->n;
  info->nnz_A = h->nnz_A;
  info->nnz_LU = h->nnz_LU;
  info->nnz_L = h->nnz_L;
  info->n_struct_zero_diag = h->n_struct_zero_diag;
  info->n_levels = h->n_levels;
  info->factor_fma = h->factor_fma;
  info->factor_div = h->nnz_L;
  info->solve_fma = h->solve_fma;
  info->max_live = h->max_live;
  info->factor_groups = h->launch.f_groups;
  info->factor_lanes_per_thread = h->launch.f_lanes;
  info->factor_slab_warps = h->launch.f_slab_warps;
  info->factor_warps_per_cta = h->launch.f_warps;
  info->factor_pend_smem = h->launch.f_tmem ? 2 : (h->launch.f_pend_smem ? 1 : 0);
  info->solve_live_smem = h->launch.s_tmem ? 2 : (h->launch.s_live_smem ? 1 : 0);
  info->solve_live = h->y_slots + h->x_slots;
  info->aug_ok = h->aug_fast ? 2 : (h->aug_ok ? 1 : 0);
  info->aug_max_live = h->plan_aug.f_slots;
  info->aug_warps_per_cta = h->aug_ok ? h->launch_aug.f_warps : 0;
  info->aug_pend_smem = !h->aug_ok ? 0 : (h->launch_aug.f_tmem ? 2 : (h->launch_aug.f_pend_smem ? 1 : 0));
  info->births = h->f_births;
  info->spill_ok = (h->spill_ok ? 1 : 0) | (h->spill_aug_ok ? 2 : 0);
  info->spill_cap = kSpillCap;
  info->spill_ops = h->spill_stats[0][0] + h->spill_stats[0][1];
  info->spill_entries = h->spill_stats[0][2];
  info->aug_spill_ops = h->spill_stats[1][0] + h->spill_stats[1][1];
  info->spill_warps_per_cta = h->spill_ok ? h->launch_spill.f_warps : 0;
  info->struct_zero_l = h->dead_l;
  info->skipped_rows = h->dead_rows[0];
  info->aug_skipped_rows = h->dead_rows[1];
  if (perm_h) std::copy(h->perm.begin(), h->perm.end(), perm_h);
  return PSP_OK;
}

psp_status psp_set_perturbations(psp_handle h, int32_t K, const double* eps_h, const double* d_h) {
  if (!h) return PSP_ERR_ARG;
  if (h->device < 0) return fail(h, PSP_ERR_UNSUPPORTED, "host-only handle (device < 0)");
  if (!h->analysed) return fail(h, PSP_ERR_STATE, "psp_symbolic_analyse first");
  if (K < 1 || !eps_h || !d_h) return fail(h, PSP_ERR_ARG, "K >= 1, eps_h and d_h required");
  cudaSetDevice(h->device);
  // (a multiple of 64: the capacity-planned factor gives a thread two 32-lane slabs)
  const int32_t Kp = (K + 2 * kBlock - 1) / (2 * kBlock) * (2 * kBlock);
  std::vector<double> eps(Kp);
  for (int32_t k = 0; k < Kp; ++k) eps[k] = eps_h[k < K ? k : K - 1];  // pad: repeat last lane
  std::vector<double> dperm(h->n);
  for (int32_t i = 0; i < h->n; ++i) dperm[i] = d_h[h->perm[i]];
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  psp_status s;
  if ((s = ensure(h, h->eps_d, sizeof(double) * Kp))) return s;
  if ((s = ensure(h, h->dperm_d, sizeof(double) * h->n))) return s;
  if ((s = ensure(h, h->status_d, sizeof(int32_t) * Kp))) return s;
  if ((s = ensure(h, h->V_d, sizeof(double) * (size_t)Kp * h->nnz_LU))) return s;
  if ((s = ensure(h, h->tol_d, sizeof(double)))) return s;
  if ((s = ensure(h, h->flag_d, sizeof(int32_t)))) return s;
  CUDA_TRY(h, cudaMemcpy(h->eps_d.p, eps.data(), sizeof(double) * Kp, cudaMemcpyHostToDevice));
  CUDA_TRY(h, cudaMemcpy(h->dperm_d.p, dperm.data(), sizeof(double) * h->n, cudaMemcpyHostToDevice));
  CUDA_TRY(h, cudaMemset(h->flag_d.p, 0, sizeof(int32_t)));
  if (K != h->K) {   // weights were validated against the old lane count: drop them
    h->W = 0;
    h->w_seg = false;
    h->w_uni = 0;
    h->wptr_host.clear();
    h->wlane_host.clear();
  }
  h->K = K;
  h->K_pad = Kp;
  h->K_global = K;   // (psp_set_perturbations_shard overrides)
  h->k_begin = 0;
  h->d_host.assign(d_h, d_h + h->n);
  h->eps_host.assign(eps_h, eps_h + K);
  h->factored = h->solved = h->recovered = false;
  return PSP_OK;
}

// The solve's launch configuration for this batch: the TMEM one when it needs fewer
// waves (rounds of resident warps over the SMs), else the shared-memory one.
static const psp::LaunchInfo& solve_launch(psp_ctx* h, int32_t R = 1) {
  if (!h->stm_ok) return h->launch;
  const int64_t blocks = h->K_pad / psp::kBlock * (R > 1 ? R : 1);   // (R-parallel items)
  auto rounds = [&](const psp::LaunchInfo& li) {
    const int64_t per = (int64_t)li.s_warps * std::max(1, li.s_ctas_per_sm) * h->n_sm;
    return (blocks + per - 1) / per;
  };
  return rounds(h->launch_stm) < rounds(h->launch) ? h->launch_stm : h->launch;
}

// The cooperative small-batch kernels for this batch? (few systems: one CTA each beats
// one thread each; PSP_OPT_COOP overrides)
static bool use_coop(psp_ctx* h, int32_t R = 1) {
  if (!h->coop_ok || h->opt_coop == 2) return false;
  // (solves: a CTA runs its right-hand sides in turn; from ~12 of them the batch
  // solve's warp-per-(block, RHS) parallelism wins: measured on cfg2, R = 16)
  return h->opt_coop == 1 || (h->K <= 8 * h->n_sm && R <= 8);
}

// The global-memory level-scheduled kernels for this batch? (large systems whose factor
// image does not fit shared memory, few systems: a CTA per system beats a thread per
// lane; PSP_OPT_COOP_GLOBAL overrides)
static bool use_coopg(psp_ctx* h) {
  if (!h->coopg_ok || h->opt_coopg == 2 || use_coop(h)) return false;
  return h->opt_coopg == 1 || h->K <= 8 * h->n_sm;
}

// Structural transversal: the caller's A values / right-hand sides -> the analysed A_hat =
// A[q, :] (gathered on the handle's stream into library buffers; no-ops without it).
static psp_status tv_A(psp_ctx* h, const double*& A, int32_t n_jac) {
  if (!h->transversal || !A) return PSP_OK;
  psp_status s;
  const size_t need = sizeof(double) * (size_t)n_jac * h->nnz_A;
  if (h->tA_d.bytes < need) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if ((s = ensure(h, h->tA_d, need))) return s;
  }
  CUDA_TRY(h, psp::launch_gather_a(h->tamap_d, h->nnz_A, n_jac, A, (double*)h->tA_d.p, h->stream));
  A = (const double*)h->tA_d.p;
  return PSP_OK;
}
static psp_status tv_B(psp_ctx* h, const double*& B, int32_t R, int64_t& ldb, int32_t n_jac = 1,
                       int64_t* jac_stride = nullptr, DevBuf* buf = nullptr) {
  if (!h->transversal || !B) return PSP_OK;
  DevBuf& b = buf ? *buf : h->tB_d;
  psp_status s;
  const size_t need = sizeof(double) * (size_t)n_jac * R * h->n;
  if (b.bytes < need) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if ((s = ensure(h, b, need))) return s;
  }
  CUDA_TRY(h, psp::launch_gather_b(h->tq_d, h->n, R, n_jac, B, ldb, jac_stride ? *jac_stride : 0, (double*)b.p,
                                   h->stream));
  B = (const double*)b.p;
  ldb = h->n;
  if (jac_stride) *jac_stride = (int64_t)R * h->n;
  return PSP_OK;
}

// Record the next event of a phase pool on the handle's stream (growing the pool).
static psp_status phase_mark(psp_ctx* h, std::vector<cudaEvent_t>& pool, size_t& used) {
  if (used == pool.size()) {
    cudaEvent_t e;
    CUDA_TRY(h, cudaEventCreate(&e));
    pool.push_back(e);
  }
  CUDA_TRY(h, cudaEventRecord(pool[used++], h->stream));
  return PSP_OK;
}

// Factorisation of the K perturbed copies with `plan` (aug = false) or of the augmented
// [A | b] with `plan_aug` (aug = true: y = L^{-1} b goes to X).
// The capacity-planned (spilling, 2 CTAs per SM) factor for this batch?  When it is
// available and the batch needs more than one round of the plain launch (its extra
// resident warps pay only then; PSP_OPT_FACTOR_SPILL overrides).
static bool use_spill(psp_ctx* h, bool aug) {
  if (h->opt_spill == 2 || !(aug ? h->spill_aug_ok : h->spill_ok)) return false;
  if (h->opt_spill == 1) return true;
  const psp::LaunchInfo& L = aug ? h->launch_aug : h->launch;
  const int64_t round = (int64_t)h->n_sm * L.f_warps * std::max(1, L.f_ctas_per_sm);
  return (int64_t)(h->K_pad / kBlock) > round;
}

static psp_status solve_impl(psp_handle h, int32_t R, const double* B, int64_t ldb);

// Fused factor + forward + backward for one right-hand side by dataflow (psp_dataflow.cu):
// the small-batch latency path; bitwise the coop factor + solve.
static psp_status dataflow_factor_solve(psp_handle h, const double* A_vals, const double* b, double pivot_tol,
                                        int32_t* lane_status) {
  if (!A_vals) return fail(h, PSP_ERR_ARG, "A_vals required");
  if (!(pivot_tol == pivot_tol)) return fail(h, PSP_ERR_ARG, "pivot_tol is NaN");
  cudaSetDevice(h->device);
  psp_status s;
  const size_t need = sizeof(double) * (size_t)h->K_pad * h->n;
  if (h->X_d.bytes < need) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if ((s = ensure(h, h->X_d, need))) return s;
  }
  psp::DataflowArgs a;
  a.n = h->n;
  a.nnz_LU = h->nnz_LU;
  a.LS = kBlock / h->launch.f_groups * h->launch.f_lanes;
  a.plan = h->df_plan;
  a.plan_words = h->df_words;
  a.birth_src = h->coop.birth_src;
  a.birth_diag = h->coop.birth_diag;
  a.perm = h->plan.perm;
  a.A = A_vals;
  a.eps = (const double*)h->eps_d.p;
  a.dperm = (const double*)h->dperm_d.p;
  a.b = b;
  if (pivot_tol <= 0) {
    CUDA_TRY(h, psp::launch_pivot_tol(h->plan, A_vals, (double*)h->tol_d.p, h->stream));
    a.tol_dev = (const double*)h->tol_d.p;
  }
  a.tol_value = pivot_tol;
  a.V = (double*)h->V_d.p;
  a.X = (double*)h->X_d.p;
  a.status = (int32_t*)h->status_d.p;
  if (h->phase_events) {
    if ((s = phase_mark(h, h->fev, h->nf))) return s;
  }
  CUDA_TRY(h, psp::launch_dataflow(a, h->K, h->df_smem, h->stream));
  if (h->phase_events) {
    if ((s = phase_mark(h, h->fev, h->nf))) return s;
  }
  h->last_factor = h->last_solve = PSP_KERNEL_DATAFLOW;
  h->last_factor_aug = 1;
  h->last_solve_fwd = 0;
  h->growth_valid = false;
  if (lane_status)
    CUDA_TRY(h, cudaMemcpyAsync(lane_status, h->status_d.p, sizeof(int32_t) * h->K,
                                cudaMemcpyDeviceToDevice, h->stream));
  h->factored = true;
  h->dense_factored = h->coopg_factored = false;
  h->mj = psp::MultiJac{};
  h->R = 1;
  h->solved = true;
  h->recovered = false;
  return PSP_OK;
}

// Dense path (psp_dense.cu): K padded N x N factors, one CTA per lane.
static psp_status dense_factor(psp_handle h, const double* A_vals, double pivot_tol,
                               int32_t* lane_status, psp::MultiJac mj = psp::MultiJac{}) {
  if (h->growth) return fail(h, PSP_ERR_UNSUPPORTED, "PSP_OPT_GROWTH is a sparse-path pass");
  const int32_t N = h->dense_N;
  cudaSetDevice(h->device);
  psp_status s;
  const size_t need = sizeof(double) * (size_t)h->K * N * N;
  if (h->Md_d.bytes < need) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if ((s = ensure(h, h->Md_d, need))) return s;
  }
  if (!h->dense_configured) {
    if (psp::dense_lu_smem(N) > (size_t)(227 * 1024))
      return fail(h, PSP_ERR_UNSUPPORTED, "dense path: n = %d exceeds the panel's shared memory", h->n);
    CUDA_TRY(h, psp::configure_dense(N));
    h->dense_configured = true;
  }
  const double* tol_dev = nullptr;
  if (pivot_tol <= 0) {
    CUDA_TRY(h, psp::launch_pivot_tol(h->plan, A_vals, (double*)h->tol_d.p, h->stream,
                                      mj.lanes_per > 0 ? h->K / mj.lanes_per : 1));
    tol_dev = (const double*)h->tol_d.p;
  }
  psp::DenseArgs a;
  a.mj = mj;
  a.n = h->n;
  a.N = N;
  a.rp = h->drp_d;
  a.ci = h->dci_d;
  a.src = h->dsrc_d;
  a.A = A_vals;
  a.eps = (const double*)h->eps_d.p;
  a.dperm = (const double*)h->dperm_d.p;
  a.Dp = h->dense_D ? (const double*)h->Dp_d.p : nullptr;
  a.tol_dev = tol_dev;
  a.tol_value = pivot_tol;
  a.M = (double*)h->Md_d.p;
  a.status = (int32_t*)h->status_d.p;
  if (h->phase_events) {
    if ((s = phase_mark(h, h->fev, h->nf))) return s;
  }
  h->last_factor = PSP_KERNEL_DENSE;
  h->last_factor_aug = 0;
  CUDA_TRY(h, psp::launch_dense_lu(a, h->K, h->stream));
  if (h->phase_events) {
    if ((s = phase_mark(h, h->fev, h->nf))) return s;
  }
  h->growth_valid = false;
  if (lane_status)
    CUDA_TRY(h, cudaMemcpyAsync(lane_status, h->status_d.p, sizeof(int32_t) * h->K,
                                cudaMemcpyDeviceToDevice, h->stream));
  h->factored = true;
  h->dense_factored = true;
  h->coopg_factored = false;
  h->mj = mj;
  h->solved = h->recovered = false;
  return PSP_OK;
}

static psp_status dense_solve(psp_handle h, int32_t R, const double* B, int64_t ldb,
                              psp::MultiJac mj = psp::MultiJac{}) {
  psp_status s;
  if (h->phase_events) {
    if ((s = phase_mark(h, h->sev, h->ns))) return s;
  }
  psp::DenseSolveArgs a;
  a.n = h->n;
  a.N = h->dense_N;
  a.R = R;
  a.ldb = ldb;
  a.perm = h->plan.perm;
  a.M = (const double*)h->Md_d.p;
  a.B = B;
  a.X = (double*)h->X_d.p;
  a.mj = mj;
  h->last_solve = PSP_KERNEL_DENSE;
  h->last_solve_fwd = 1;
  CUDA_TRY(h, psp::launch_dense_solve(a, h->K, h->stream));
  if (h->phase_events) {
    if ((s = phase_mark(h, h->sev, h->ns))) return s;
  }
  h->R = R;
  h->solved = true;
  return PSP_OK;
}

// Global-memory level-scheduled factor (psp_coopg.cu): V_d holds lane-major images.
static psp_status coopg_factor(psp_handle h, const double* A_vals, double pivot_tol,
                               int32_t* lane_status, psp::MultiJac mj = psp::MultiJac{}) {
  if (h->growth) return fail(h, PSP_ERR_UNSUPPORTED, "PSP_OPT_GROWTH reads the batch factor layout");
  cudaSetDevice(h->device);
  psp_status s;
  psp::CoopGArgs a;
  a.c = h->coopg;
  a.A = A_vals;
  a.eps = (const double*)h->eps_d.p;
  a.dperm = (const double*)h->dperm_d.p;
  if (pivot_tol <= 0) {
    CUDA_TRY(h, psp::launch_pivot_tol(h->plan, A_vals, (double*)h->tol_d.p, h->stream,
                                      mj.lanes_per > 0 ? h->K / mj.lanes_per : 1));
    a.tol_dev = (const double*)h->tol_d.p;
  }
  a.tol_value = pivot_tol;
  a.mj = mj;
  a.W = (double*)h->V_d.p;   // (K_pad x nnz_LU doubles: the same bytes as the batch layout)
  a.status = (int32_t*)h->status_d.p;
  if (h->phase_events) {
    if ((s = phase_mark(h, h->fev, h->nf))) return s;
  }
  h->last_factor = PSP_KERNEL_COOP_GLOBAL;
  h->last_factor_aug = 0;
  CUDA_TRY(h, psp::launch_coopg_factor(a, h->K, h->stream));
  if (h->phase_events) {
    if ((s = phase_mark(h, h->fev, h->nf))) return s;
  }
  h->growth_valid = false;
  if (lane_status)
    CUDA_TRY(h, cudaMemcpyAsync(lane_status, h->status_d.p, sizeof(int32_t) * h->K,
                                cudaMemcpyDeviceToDevice, h->stream));
  h->factored = true;
  h->dense_factored = false;
  h->coopg_factored = true;
  h->mj = mj;
  h->solved = h->recovered = false;
  return PSP_OK;
}

static psp_status coopg_solve(psp_handle h, int32_t R, const double* B, int64_t ldb,
                              psp::MultiJac mj = psp::MultiJac{}) {
  psp_status s;
  if (h->phase_events) {
    if ((s = phase_mark(h, h->sev, h->ns))) return s;
  }
  psp::CoopGSolveArgs a;
  a.c = h->coopg;
  a.perm = h->plan.perm;
  a.W = (const double*)h->V_d.p;
  a.B = B;
  a.ldb = ldb;
  a.R = R;
  a.X = (double*)h->X_d.p;
  a.mj = mj;
  h->last_solve = PSP_KERNEL_COOP_GLOBAL;
  h->last_solve_fwd = 1;
  CUDA_TRY(h, psp::launch_coopg_solve(a, h->K, h->stream));
  if (h->phase_events) {
    if ((s = phase_mark(h, h->sev, h->ns))) return s;
  }
  h->R = R;
  h->solved = true;
  return PSP_OK;
}

static psp_status factor_impl(psp_handle h, const double* A_vals, double pivot_tol,
                              int32_t* lane_status, bool aug, const double* b,
                              psp::MultiJac mj = psp::MultiJac{}) {
  if (!h) return PSP_ERR_ARG;
  if (!h->analysed || h->K == 0) return fail(h, PSP_ERR_STATE, "set_perturbations first");
  if (!A_vals) return fail(h, PSP_ERR_ARG, "A_vals required");
  if (!(pivot_tol == pivot_tol)) return fail(h, PSP_ERR_ARG, "pivot_tol is NaN");
  if (h->opt_path == PSP_PATH_DENSE) return dense_factor(h, A_vals, pivot_tol, lane_status, mj);
  if (h->dense_D)
    return fail(h, PSP_ERR_UNSUPPORTED, "a dense D needs the dense path (PSP_OPT_PATH = PSP_PATH_DENSE)");
  if (use_coopg(h)) return coopg_factor(h, A_vals, pivot_tol, lane_status, mj);
  if (mj.lanes_per > 0 && !use_coop(h))
    return fail(h, PSP_ERR_UNSUPPORTED,
                "multi-Jacobian batches run the cooperative / global level-scheduled / dense kernels "
                "(K <= 8 x SMs, or PSP_OPT_COOP = 1); factor larger batches per Jacobian");
  const bool spill = !use_coop(h) && use_spill(h, aug);
  const DevicePlan& P = spill ? (aug ? h->plan_spill_aug : h->plan_spill) : (aug ? h->plan_aug : h->plan);
  const psp::LaunchInfo& LI = spill ? (aug ? h->launch_spill_aug : h->launch_spill)
                                    : (aug ? h->launch_aug : h->launch);
  cudaSetDevice(h->device);
  psp_status s;
  const double* tol_dev = nullptr;
  // (one Jacobian: the default tolerance rides in the program-patch launch below)
  const bool tol_fused = pivot_tol <= 0 && mj.lanes_per <= 0 && P.f_npatch > 0;
  if (pivot_tol <= 0) {
    if (!tol_fused)
      CUDA_TRY(h, psp::launch_pivot_tol(P, A_vals, (double*)h->tol_d.p, h->stream,
                                        mj.lanes_per > 0 ? h->K / mj.lanes_per : 1));
    tol_dev = (const double*)h->tol_d.p;
  }
  if (!LI.f_pend_smem) {
    size_t need = sizeof(double) * (size_t)h->K_pad * P.f_slots;
    if (h->fscratch_d.bytes < need) {
      CUDA_TRY(h, cudaStreamSynchronize(h->stream));
      if ((s = ensure(h, h->fscratch_d, need))) return s;
    }
  }
  if (aug) {
    size_t need = sizeof(double) * (size_t)h->K_pad * h->n;
    if (h->X_d.bytes < need) {
      CUDA_TRY(h, cudaStreamSynchronize(h->stream));
      if ((s = ensure(h, h->X_d, need))) return s;
    }
  }
  if (tol_fused)
    CUDA_TRY(h, psp::launch_patch_tol(P, const_cast<int32_t*>(P.f_stream), A_vals,
                                      (const double*)h->dperm_d.p, b, (double*)h->tol_d.p, h->stream));
  else
    CUDA_TRY(h, psp::launch_patch_program(P, const_cast<int32_t*>(P.f_stream), A_vals,
                                          (const double*)h->dperm_d.p, b, h->stream));
  if (!LI.f_scr_smem) {
    size_t need = sizeof(double) * (size_t)h->K_pad * 2 * P.c_scr;
    if (h->fscr_d.bytes < need) {
      CUDA_TRY(h, cudaStreamSynchronize(h->stream));
      if ((s = ensure(h, h->fscr_d, need))) return s;
    }
  }
  if (spill) {
    size_t need = sizeof(double) * (size_t)h->K_pad * std::max(1, P.f_gspill);
    if (h->gspill_d.bytes < need) {
      CUDA_TRY(h, cudaStreamSynchronize(h->stream));
      if ((s = ensure(h, h->gspill_d, need))) return s;
    }
  }
  if (h->phase_events) {
    if ((s = phase_mark(h, h->fev, h->nf))) return s;
  }
  if (h->growth && h->growth_d.bytes < sizeof(double) * (size_t)h->K_pad) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if ((s = ensure(h, h->growth_d, sizeof(double) * (size_t)h->K_pad))) return s;
    if ((s = ensure(h, h->offmax_d, sizeof(double)))) return s;
  }
  if (use_coop(h)) {   // (the augmented program is not needed: the solve does its forward)
    h->last_factor = PSP_KERNEL_COOP;
    h->last_factor_aug = 0;
    CUDA_TRY(h, psp::launch_coop_factor(h->plan, h->coop, A_vals, (const double*)h->eps_d.p,
                                        (const double*)h->dperm_d.p, tol_dev, pivot_tol,
                                        (double*)h->V_d.p, (int32_t*)h->status_d.p, h->K,
                                        kBlock / h->launch.f_groups * h->launch.f_lanes, h->stream, mj));
  } else {
    h->last_factor = spill ? PSP_KERNEL_BATCH_SPILL : (LI.f_tmem ? PSP_KERNEL_BATCH_TMEM : PSP_KERNEL_BATCH);
    h->last_factor_aug = aug ? 1 : 0;
    CUDA_TRY(h, psp::launch_factor(P, LI, P.f_stream, (const double*)h->eps_d.p, tol_dev, pivot_tol,
                                   (double*)h->V_d.p, (double*)h->fscratch_d.p, (double*)h->fscr_d.p,
                                   (int32_t*)h->status_d.p, h->K_pad,
                                   aug ? (double*)h->X_d.p : nullptr, (double*)h->gspill_d.p,
                                   h->stream));
  }
  if (h->phase_events) {
    if ((s = phase_mark(h, h->fev, h->nf))) return s;
  }
  if (h->growth)
    CUDA_TRY(h, psp::launch_growth(P, LI, (const double*)h->V_d.p, A_vals, h->isdiag_d,
                                   (const double*)h->eps_d.p, (const double*)h->dperm_d.p, h->K,
                                   (double*)h->offmax_d.p, (double*)h->growth_d.p, h->stream));
  h->growth_valid = h->growth;
  if (lane_status)
    CUDA_TRY(h, cudaMemcpyAsync(lane_status, h->status_d.p, sizeof(int32_t) * h->K,
                                cudaMemcpyDeviceToDevice, h->stream));
  h->factored = true;
  h->dense_factored = false;
  h->coopg_factored = false;
  h->mj = mj;
  h->solved = h->recovered = false;
  return PSP_OK;
}

psp_status psp_factor_batch(psp_handle h, const double* A_vals, double pivot_tol,
                            int32_t* lane_status) {
  if (!h) return PSP_ERR_ARG;
  psp_status s;
  if (h->analysed && h->K > 0 && (s = tv_A(h, A_vals, 1))) return s;
  return factor_impl(h, A_vals, pivot_tol, lane_status, false, nullptr);
}

static psp_status solve_scratch(psp_handle h, int32_t R) {
  psp_status s;
  if (!solve_launch(h, R).s_live_smem) {   // (R-parallel solves: one live set per RHS)
    size_t need2 = sizeof(double) * (size_t)h->K_pad * (h->plan.y_slots + h->plan.x_slots + 1) *
                   (size_t)(R > 1 ? R : 1);
    if (h->sscratch_d.bytes < need2) {
      CUDA_TRY(h, cudaStreamSynchronize(h->stream));
      if ((s = ensure(h, h->sscratch_d, need2))) return s;
    }
  }
  return PSP_OK;
}

psp_status psp_factor_solve_batch(psp_handle h, const double* A_vals, const double* b,
                                  double pivot_tol, int32_t* lane_status) {
  if (!h) return PSP_ERR_ARG;
  if (!b) return fail(h, PSP_ERR_ARG, "b required");
  psp_status s;
  if (h->analysed && h->K > 0) {
    int64_t ldb = h->n;
    if ((s = tv_A(h, A_vals, 1))) return s;
    if ((s = tv_B(h, b, 1, ldb))) return s;
  }
  // (automatic only for small systems: measured on the B200, cfg0 (nnz_LU = 2.3e2) 28.7 us vs
  // 40.0 us per step for the cooperative factor + solve, but cfg1 (5.5e3) 330 vs 135 us --
  // the walkers' per-contribution flag checks cost more than the barriers they replace)
  if (h->analysed && h->K > 0 && h->opt_path != PSP_PATH_DENSE && !h->dense_D && use_coop(h) && h->df_ok &&
      (h->opt_df == 1 || (h->opt_df == 0 && h->nnz_LU <= 1024)) && !h->growth)
    return dataflow_factor_solve(h, A_vals, b, pivot_tol, lane_status);
  if (h->analysed && (h->opt_path == PSP_PATH_DENSE || use_coopg(h))) {
    if ((s = factor_impl(h, A_vals, pivot_tol, lane_status, false, nullptr))) return s;
    return solve_impl(h, 1, b, h->n);
  }
  const bool fuse = h->analysed && !use_coop(h) && (use_spill(h, true) || h->aug_fast);
  if (h->analysed && !fuse) {   // the two calls (bitwise the same)
    if ((s = factor_impl(h, A_vals, pivot_tol, lane_status, false, nullptr))) return s;
    return solve_impl(h, 1, b, h->n);
  }
  s = factor_impl(h, A_vals, pivot_tol, lane_status, true, b);
  if (s) return s;
  if ((s = solve_scratch(h, 1))) return s;
  if (h->phase_events) {
    if ((s = phase_mark(h, h->sev, h->ns))) return s;
  }
  h->last_solve = solve_launch(h).s_tmem ? PSP_KERNEL_BATCH_TMEM : PSP_KERNEL_BATCH;
  h->last_solve_fwd = 0;
  CUDA_TRY(h, psp::launch_solve(h->plan, solve_launch(h), (const double*)h->V_d.p, b, h->n, 1,
                                (double*)h->X_d.p, (double*)h->sscratch_d.p, h->K_pad, false,
                                h->stream));
  if (h->phase_events) {
    if ((s = phase_mark(h, h->sev, h->ns))) return s;
  }
  h->R = 1;
  h->solved = true;
  return PSP_OK;
}

psp_status psp_solve_batch(psp_handle h, int32_t R, const double* B, int64_t ldb) {
  if (!h) return PSP_ERR_ARG;
  if (!h->factored) return fail(h, PSP_ERR_STATE, "factor_batch first");
  if (R < 1 || !B || ldb < h->n) return fail(h, PSP_ERR_ARG, "R >= 1, B, ldb >= n required");
  cudaSetDevice(h->device);
  psp_status s;
  if ((s = tv_B(h, B, R, ldb))) return s;
  return solve_impl(h, R, B, ldb);
}

static psp_status solve_impl(psp_handle h, int32_t R, const double* B, int64_t ldb) {
  cudaSetDevice(h->device);
  psp_status s;
  size_t need = sizeof(double) * (size_t)h->K_pad * R * h->n;
  if (h->X_d.bytes < need) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if ((s = ensure(h, h->X_d, need))) return s;
  }
  if (h->dense_factored) return dense_solve(h, R, B, ldb);
  if (h->coopg_factored) return coopg_solve(h, R, B, ldb);
  if ((s = solve_scratch(h, R))) return s;
  if (h->phase_events) {
    if ((s = phase_mark(h, h->sev, h->ns))) return s;
  }
  if (use_coop(h, R)) {
    h->last_solve = PSP_KERNEL_COOP;
    h->last_solve_fwd = 1;
    CUDA_TRY(h, psp::launch_coop_solve(h->plan, h->coop, (const double*)h->V_d.p, B, ldb, R,
                                       (double*)h->X_d.p, h->K,
                                       kBlock / h->launch.f_groups * h->launch.f_lanes, h->stream));
    if (h->phase_events) {
      if ((s = phase_mark(h, h->sev, h->ns))) return s;
    }
    h->R = R;
    h->solved = true;
    return PSP_OK;
  }
  h->last_solve = solve_launch(h, R).s_tmem ? PSP_KERNEL_BATCH_TMEM : PSP_KERNEL_BATCH;
  h->last_solve_fwd = 1;
  CUDA_TRY(h, psp::launch_solve(h->plan, solve_launch(h, R), (const double*)h->V_d.p, B, ldb, R,
                                (double*)h->X_d.p, (double*)h->sscratch_d.p, h->K_pad, true,
                                h->stream));
  if (h->phase_events) {
    if ((s = phase_mark(h, h->sev, h->ns))) return s;
  }
  h->R = R;
  h->solved = true;
  return PSP_OK;
}

psp_status psp_factor_batch_multi(psp_handle h, int32_t n_jac, const double* A_vals, double pivot_tol,
                                  int32_t* lane_status) {
  if (!h) return PSP_ERR_ARG;
  if (!h->analysed || h->K == 0) return fail(h, PSP_ERR_STATE, "set_perturbations first");
  if (n_jac < 1 || h->K % n_jac) return fail(h, PSP_ERR_ARG, "n_jac >= 1 must divide K = %d", h->K);
  if (n_jac == 1) return psp_factor_batch(h, A_vals, pivot_tol, lane_status);
  psp_status s;
  if ((s = tv_A(h, A_vals, n_jac))) return s;
  if (h->tol_d.bytes < sizeof(double) * (size_t)n_jac) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if ((s = ensure(h, h->tol_d, sizeof(double) * (size_t)n_jac))) return s;
  }
  psp::MultiJac mj;
  mj.lanes_per = h->K / n_jac;
  mj.a_stride = h->nnz_A;
  return factor_impl(h, A_vals, pivot_tol, lane_status, false, nullptr, mj);
}

psp_status psp_solve_batch_multi(psp_handle h, int32_t R, const double* B, int64_t ldb, int64_t jac_stride) {
  if (!h) return PSP_ERR_ARG;
  if (!h->factored || h->mj.lanes_per == 0)
    return fail(h, PSP_ERR_STATE, "psp_factor_batch_multi (n_jac > 1) first");
  if (R < 1 || !B || ldb < h->n || jac_stride < (int64_t)(R - 1) * ldb + h->n)
    return fail(h, PSP_ERR_ARG, "R >= 1, B, ldb >= n, jac_stride >= (R - 1) ldb + n required");
  cudaSetDevice(h->device);
  psp_status s;
  size_t need = sizeof(double) * (size_t)h->K_pad * R * h->n;
  if (h->X_d.bytes < need) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if ((s = ensure(h, h->X_d, need))) return s;
  }
  if ((s = tv_B(h, B, R, ldb, h->K / h->mj.lanes_per, &jac_stride))) return s;
  psp::MultiJac mj = h->mj;
  mj.b_stride = jac_stride;
  if (h->dense_factored) return dense_solve(h, R, B, ldb, mj);
  if (h->coopg_factored) return coopg_solve(h, R, B, ldb, mj);
  if (h->last_factor != PSP_KERNEL_COOP)
    return fail(h, PSP_ERR_UNSUPPORTED, "multi-Jacobian solves follow a multi-Jacobian factorisation");
  if (h->phase_events) {
    if ((s = phase_mark(h, h->sev, h->ns))) return s;
  }
  h->last_solve = PSP_KERNEL_COOP;
  h->last_solve_fwd = 1;
  CUDA_TRY(h, psp::launch_coop_solve(h->plan, h->coop, (const double*)h->V_d.p, B, ldb, R, (double*)h->X_d.p,
                                     h->K, kBlock / h->launch.f_groups * h->launch.f_lanes, h->stream, mj));
  if (h->phase_events) {
    if ((s = phase_mark(h, h->sev, h->ns))) return s;
  }
  h->R = R;
  h->solved = true;
  return PSP_OK;
}

psp_status psp_refine(psp_handle h, const double* A_vals, const double* b, int32_t iters, double* x_out) {
  if (!h) return PSP_ERR_ARG;
  if (!h->factored) return fail(h, PSP_ERR_STATE, "factor_batch first");
  if (!A_vals || !b || !x_out || iters < 0) return fail(h, PSP_ERR_ARG, "A_vals, b, x_out, iters >= 0 required");
  if (h->mj.lanes_per > 0) return fail(h, PSP_ERR_UNSUPPORTED, "psp_refine follows a single-Jacobian factorisation");
  const bool coop = !h->dense_factored && !h->coopg_factored && h->last_factor == PSP_KERNEL_COOP;
  if (!h->dense_factored && !h->coopg_factored && !coop)
    return fail(h, PSP_ERR_UNSUPPORTED,
                "psp_refine needs per-lane right-hand sides: the cooperative, global level-scheduled or "
                "dense kernels (K <= 8 x SMs, PSP_OPT_COOP / PSP_OPT_COOP_GLOBAL, or PSP_OPT_PATH)");
  cudaSetDevice(h->device);
  psp_status s;
  int64_t ldb1 = h->n;
  if ((s = tv_A(h, A_vals, 1))) return s;
  if ((s = tv_B(h, b, 1, ldb1, 1, nullptr, &h->tb2_d))) return s;
  // x^0 = F_k^{-1} b
  if ((s = solve_impl(h, 1, b, h->n))) return s;
  CUDA_TRY(h, psp::launch_gather_solutions(h->plan, h->K, 1, (const double*)h->X_d.p, x_out, h->stream));
  if (iters == 0) return PSP_OK;
  const size_t need = sizeof(double) * (size_t)h->K * h->n;
  if (h->ref_r_d.bytes < need) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if ((s = ensure(h, h->ref_r_d, need))) return s;
  }
  psp::MultiJac mj;          // each lane its own right-hand side r_k
  mj.lanes_per = 1;
  mj.b_stride = h->n;
  double* r = (double*)h->ref_r_d.p;
  for (int32_t it = 0; it < iters; ++it) {
    CUDA_TRY(h, psp::launch_refine_step(h->plan, h->K, h->rowptr_d, h->colidx_d, A_vals, b, x_out, r, h->stream));
    if (h->dense_factored) {
      if ((s = dense_solve(h, 1, r, h->n, mj))) return s;
    } else if (h->coopg_factored) {
      if ((s = coopg_solve(h, 1, r, h->n, mj))) return s;
    } else {
      h->last_solve = PSP_KERNEL_COOP;
      h->last_solve_fwd = 1;
      CUDA_TRY(h, psp::launch_coop_solve(h->plan, h->coop, (const double*)h->V_d.p, r, h->n, 1,
                                         (double*)h->X_d.p, h->K,
                                         kBlock / h->launch.f_groups * h->launch.f_lanes, h->stream, mj));
    }
    CUDA_TRY(h, psp::launch_refine_update(h->plan, h->K, (const double*)h->X_d.p, x_out, h->stream));
  }
  h->solved = false;   // (X holds the last correction, not solutions)
  h->recovered = false;
  return PSP_OK;
}

psp_status psp_estimate_rho(psp_handle h, int32_t w, int32_t max_iter, double rtol,
                            const double* v0_h, double* rho_h, int32_t* iters_h,
                            int32_t* converged_h) {
  if (!h || !v0_h || !rho_h || max_iter < 1 || !(rtol > 0)) return PSP_ERR_ARG;
  if (!h->factored || h->W == 0) return fail(h, PSP_ERR_STATE, "factor_batch and set_weights first");
  if (w < 0 || w >= h->W) return fail(h, PSP_ERR_ARG, "w out of range");
  if (h->transversal) return fail(h, PSP_ERR_UNSUPPORTED, "psp_estimate_rho with PSP_OPT_TRANSVERSAL");
  const int32_t n = h->n;
  cudaSetDevice(h->device);
  psp_status s;
  if ((s = ensure(h, h->rho_r_d, sizeof(double) * n))) return s;
  if ((s = ensure(h, h->rho_x_d, sizeof(double) * (size_t)h->W * n))) return s;
  // v = v0 / ||v0||_2
  std::vector<double> v(v0_h, v0_h + n), r(n), u(n);
  auto nrm = [&](const std::vector<double>& x) {
    long double a = 0;
    for (double t : x) a += (long double)t * t;
    return (double)std::sqrt(a);
  };
  double nv = nrm(v);
  if (!(nv > 0) || !std::isfinite(nv)) return fail(h, PSP_ERR_ARG, "v0 must be nonzero and finite");
  for (double& t : v) t /= nv;
  double rho = 0.0;
  int32_t it = 0, conv = 0;
  for (it = 1; it <= max_iter; ++it) {
    if (h->dense_D) {   // r = D v (dense D, original ordering; long double row sums)
      for (int32_t i = 0; i < n; ++i) {
        long double acc = 0;
        for (int32_t j = 0; j < n; ++j) acc += (long double)h->D_host[(size_t)i * n + j] * v[j];
        r[i] = (double)acc;
      }
    } else {
      for (int32_t i = 0; i < n; ++i) r[i] = h->d_host[i] * v[i];   // r = D v
    }
    CUDA_TRY(h, cudaMemcpyAsync(h->rho_r_d.p, r.data(), sizeof(double) * n, cudaMemcpyHostToDevice,
                                h->stream));
    if ((s = solve_impl(h, 1, (const double*)h->rho_r_d.p, n))) return s;
    if ((s = psp_recover(h, (double*)h->rho_x_d.p))) return s;
    CUDA_TRY(h, cudaMemcpyAsync(u.data(), (const double*)h->rho_x_d.p + (size_t)w * n,
                                sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    const double nu = nrm(u);   // ||x-hat(D v)|| with ||v|| = 1
    if (!std::isfinite(nu))
      return fail(h, PSP_ERR_BATCH_INFEASIBLE, "non-finite iterate (a weight on a failed lane)");
    const double prev = rho;
    rho = nu;
    if (nu == 0.0) break;
    for (int32_t i = 0; i < n; ++i) v[i] = u[i] / nu;
    if (it > 1 && std::fabs(rho - prev) < rtol * rho) {
      conv = 1;
      break;
    }
  }
  *rho_h = rho;
  if (iters_h) *iters_h = std::min(it, max_iter);
  if (converged_h) *converged_h = conv;
  return PSP_OK;
}

psp_status psp_get_lane_growth(psp_handle h, double* growth_h) {
  if (!h || !growth_h) return PSP_ERR_ARG;
  if (!h->growth_valid) return fail(h, PSP_ERR_STATE, "factor with PSP_OPT_GROWTH = 1 first");
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaMemcpy(growth_h, h->growth_d.p, sizeof(double) * h->K, cudaMemcpyDeviceToHost));
  return PSP_OK;
}

psp_status psp_get_phase_times(psp_handle h, float* ms_h) {
  if (!h || !ms_h) return PSP_ERR_ARG;
  if (!h->phase_events) return fail(h, PSP_ERR_STATE, "PSP_OPT_PHASE_EVENTS is off");
  cudaSetDevice(h->device);
  for (int q = 0; q < 2; ++q) {
    const std::vector<cudaEvent_t>& v = q ? h->sev : h->fev;
    const size_t m = q ? h->ns : h->nf;
    double sum = 0.0;
    for (size_t k = 0; k + 1 < m; k += 2) {
      float t = 0.f;
      CUDA_TRY(h, cudaEventSynchronize(v[k + 1]));
      CUDA_TRY(h, cudaEventElapsedTime(&t, v[k], v[k + 1]));
      sum += t;
    }
    ms_h[q] = m >= 2 ? (float)(sum / (double)(m / 2)) : 0.f;
  }
  h->nf = h->ns = 0;
  return PSP_OK;
}

psp_status psp_get_last_kernels(psp_handle h, int32_t* kernels_h) {
  if (!h || !kernels_h) return PSP_ERR_ARG;
  kernels_h[0] = h->last_factor;
  kernels_h[1] = h->last_factor_aug;
  kernels_h[2] = h->last_solve;
  kernels_h[3] = h->last_solve_fwd;
  return PSP_OK;
}

psp_status psp_get_solutions(psp_handle h, double* X) {
  if (!h || !X) return PSP_ERR_ARG;
  if (!h->solved) return fail(h, PSP_ERR_STATE, "solve_batch first");
  CUDA_TRY(h, psp::launch_gather_solutions(h->plan, h->K, h->R, (const double*)h->X_d.p, X,
                                           h->stream));
  return PSP_OK;
}

psp_status psp_get_factor(psp_handle h, int32_t k, double* vals_h) {
  if (!h || !vals_h) return PSP_ERR_ARG;
  if (!h->factored) return fail(h, PSP_ERR_STATE, "factor_batch first");
  if (k < 0 || k >= h->K) return fail(h, PSP_ERR_ARG, "lane %d out of range", k);
  if (h->dense_factored)
    return fail(h, PSP_ERR_UNSUPPORTED, "dense factorisation: use psp_get_dense_factor");
  if (h->coopg_factored) {   // lane-major images
    cudaSetDevice(h->device);
    CUDA_TRY(h, cudaMemcpyAsync(vals_h, (const double*)h->V_d.p + (size_t)k * h->nnz_LU,
                                sizeof(double) * h->nnz_LU, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return PSP_OK;
  }
  const int L = kBlock / h->launch.f_groups * h->launch.f_lanes;
  const double* src = (const double*)h->V_d.p + (size_t)(k / L) * h->nnz_LU * L + (k % L);
  CUDA_TRY(h, cudaMemcpy2DAsync(vals_h, sizeof(double), src, sizeof(double) * L, sizeof(double),
                                (size_t)h->nnz_LU, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return PSP_OK;
}

psp_status psp_get_transversal(psp_handle h, int32_t* q_h) {
  if (!h || !q_h) return PSP_ERR_ARG;
  if (!h->analysed || !h->transversal) return fail(h, PSP_ERR_STATE, "analyse with PSP_OPT_TRANSVERSAL = 1 first");
  std::copy(h->tq.begin(), h->tq.end(), q_h);
  return PSP_OK;
}

psp_status psp_get_dense_factor(psp_handle h, int32_t k, double* lu_h) {
  if (!h || !lu_h) return PSP_ERR_ARG;
  if (!h->factored || !h->dense_factored) return fail(h, PSP_ERR_STATE, "dense factor_batch first");
  if (k < 0 || k >= h->K) return fail(h, PSP_ERR_ARG, "lane %d out of range", k);
  const int32_t N = h->dense_N;
  cudaSetDevice(h->device);
  const double* src = (const double*)h->Md_d.p + (size_t)k * N * N;
  CUDA_TRY(h, cudaMemcpy2DAsync(lu_h, sizeof(double) * h->n, src, sizeof(double) * N,
                                sizeof(double) * h->n, (size_t)h->n, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return PSP_OK;
}

psp_status psp_set_perturbation_matrix(psp_handle h, const double* D_h) {
  if (!h) return PSP_ERR_ARG;
  if (h->device < 0) return fail(h, PSP_ERR_UNSUPPORTED, "host-only handle (device < 0)");
  if (!h->analysed) return fail(h, PSP_ERR_STATE, "psp_symbolic_analyse first");
  if (D_h && h->transversal) return fail(h, PSP_ERR_UNSUPPORTED, "a dense D with PSP_OPT_TRANSVERSAL");
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  if (!D_h) {
    h->Dp_d.release();
    h->D_host.clear();
    h->dense_D = false;
    h->factored = h->solved = h->recovered = false;
    return PSP_OK;
  }
  const int32_t n = h->n;
  std::vector<double> Dp((size_t)n * n);
  for (int32_t i = 0; i < n; ++i) {
    const double* row = D_h + (size_t)h->perm[i] * n;
    for (int32_t j = 0; j < n; ++j) {
      const double v = row[h->perm[j]];
      if (!std::isfinite(v)) return fail(h, PSP_ERR_ARG, "D has a non-finite entry");
      Dp[(size_t)i * n + j] = v;
    }
  }
  psp_status s;
  if ((s = ensure(h, h->Dp_d, sizeof(double) * Dp.size()))) return s;
  CUDA_TRY(h, cudaMemcpy(h->Dp_d.p, Dp.data(), sizeof(double) * Dp.size(), cudaMemcpyHostToDevice));
  h->D_host.assign(D_h, D_h + (size_t)n * n);
  h->dense_D = true;
  h->factored = h->solved = h->recovered = false;
  return PSP_OK;
}

psp_status psp_set_weights(psp_handle h, int32_t W, const int32_t* w_ptr_h,
                           const int32_t* w_lane_h, const double* w_val_h) {
  if (!h) return PSP_ERR_ARG;
  if (h->K == 0) return fail(h, PSP_ERR_STATE, "set_perturbations first");
  if (W < 1 || !w_ptr_h || w_ptr_h[0] != 0) return fail(h, PSP_ERR_ARG, "bad weight CSR");
  std::vector<int32_t> ptr(1, 0), lane;
  std::vector<double> val;
  for (int32_t w = 0; w < W; ++w) {
    if (w_ptr_h[w + 1] < w_ptr_h[w]) return fail(h, PSP_ERR_ARG, "w_ptr not monotone");
    int32_t prev = -1;
    for (int32_t q = w_ptr_h[w]; q < w_ptr_h[w + 1]; ++q) {
      int32_t k = w_lane_h[q];
      if (k < 0 || k >= h->K || k <= prev)
        return fail(h, PSP_ERR_ARG, "weight lanes must be strictly ascending in [0, K)");
      prev = k;
      if (!std::isfinite(w_val_h[q])) return fail(h, PSP_ERR_ARG, "non-finite weight");
      if (w_val_h[q] != 0.0) {
        lane.push_back(k);
        val.push_back(w_val_h[q]);
      }
    }
    ptr.push_back((int32_t)lane.size());
  }
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  psp_status s;
  if ((s = ensure(h, h->wptr_d, sizeof(int32_t) * ptr.size()))) return s;
  if ((s = ensure(h, h->wlane_d, sizeof(int32_t) * std::max<size_t>(lane.size(), 1)))) return s;
  if ((s = ensure(h, h->wval_d, sizeof(double) * std::max<size_t>(val.size(), 1)))) return s;
  CUDA_TRY(h, cudaMemcpy(h->wptr_d.p, ptr.data(), sizeof(int32_t) * ptr.size(), cudaMemcpyHostToDevice));
  if (!lane.empty()) {
    CUDA_TRY(h, cudaMemcpy(h->wlane_d.p, lane.data(), sizeof(int32_t) * lane.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(h, cudaMemcpy(h->wval_d.p, val.data(), sizeof(double) * val.size(), cudaMemcpyHostToDevice));
  }
  // fast-path detection (psp_kernels.cu recover_seg_kernel): every row a contiguous run
  // of <= 16 lanes inside one 32-lane block
  {
    bool ok = true;
    for (int32_t w = 0; w < W && ok; ++w) {
      const int32_t q0 = ptr[w], q1 = ptr[w + 1];
      if (q0 == q1) continue;
      const int32_t k0 = lane[q0], k1 = lane[q1 - 1];
      ok = k1 - k0 == q1 - q0 - 1 && k0 / kBlock == k1 / kBlock && q1 - q0 <= 16;
    }
    h->w_seg = ok;
    // uniform ladders (recover_uni_kernel): row w = lanes [w*L, w*L + L)
    int32_t L = W > 0 ? ptr[1] - ptr[0] : 0;
    bool uni = L == 2 || L == 4 || L == 8 || L == 16;
    for (int32_t w = 0; w < W && uni; ++w) {
      uni = ptr[w] == w * L && ptr[w + 1] == (w + 1) * L;
      for (int32_t j = 0; j < L && uni; ++j) uni = lane[ptr[w] + j] == w * L + j;
    }
    h->w_uni = uni ? L : 0;
  }
  h->wptr_host = ptr;
  h->wlane_host = lane;
  h->W = W;
  return PSP_OK;
}

psp_status psp_rescale_failed_rows(psp_handle h, double scale, int32_t* n_rows_h) {
  if (!h) return PSP_ERR_ARG;
  if (!(scale != 0.0) || !std::isfinite(scale)) return fail(h, PSP_ERR_ARG, "scale must be finite and non-zero");
  if (!h->factored || h->W == 0) return fail(h, PSP_ERR_STATE, "factor_batch and set_weights first");
  cudaSetDevice(h->device);
  const int32_t K = h->K, Kp = h->K_pad;
  std::vector<int32_t> st(K);
  CUDA_TRY(h, cudaMemcpyAsync(st.data(), h->status_d.p, sizeof(int32_t) * K, cudaMemcpyDeviceToHost,
                              h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  std::vector<uint8_t> mark(K, 0);
  int32_t rows = 0;
  for (int32_t w = 0; w < h->W; ++w) {
    bool bad = false;
    for (int32_t q = h->wptr_host[w]; q < h->wptr_host[w + 1] && !bad; ++q)
      bad = h->wlane_host[q] < K && st[h->wlane_host[q]] != 0;
    if (!bad) continue;
    ++rows;
    for (int32_t q = h->wptr_host[w]; q < h->wptr_host[w + 1]; ++q)
      if (h->wlane_host[q] < K) mark[h->wlane_host[q]] = 1;
  }
  if (n_rows_h) *n_rows_h = rows;
  if (rows == 0) return PSP_OK;
  for (int32_t k = 0; k < K; ++k)
    if (mark[k]) h->eps_host[k] *= scale;
  std::vector<double> eps(Kp);
  for (int32_t k = 0; k < Kp; ++k) eps[k] = h->eps_host[k < K ? k : K - 1];
  CUDA_TRY(h, cudaMemcpy(h->eps_d.p, eps.data(), sizeof(double) * Kp, cudaMemcpyHostToDevice));
  h->factored = h->solved = h->recovered = false;
  return PSP_OK;
}

psp_status psp_get_perturbations(psp_handle h, double* eps_h) {
  if (!h || !eps_h) return PSP_ERR_ARG;
  if (h->K == 0) return fail(h, PSP_ERR_STATE, "set_perturbations first");
  std::copy(h->eps_host.begin(), h->eps_host.end(), eps_h);
  return PSP_OK;
}

psp_status psp_recover(psp_handle h, double* x) {
  if (!h || !x) return PSP_ERR_ARG;
  if (!h->solved || h->W == 0) return fail(h, PSP_ERR_STATE, "solve_batch and set_weights first");
  // the batch-infeasible flag describes THIS combination (a re-perturbed, refactored batch
  // must not inherit an earlier call's flag)
  CUDA_TRY(h, cudaMemsetAsync(h->flag_d.p, 0, sizeof(int32_t), h->stream));
  if (h->w_uni) {
    CUDA_TRY(h, psp::launch_recover_uni(h->plan, h->W, h->R, h->w_uni, (const double*)h->wval_d.p,
                                        (const double*)h->X_d.p, (const int32_t*)h->status_d.p, x,
                                        (int32_t*)h->flag_d.p, h->stream));
  } else if (h->w_seg) {
    CUDA_TRY(h, psp::launch_recover_seg(h->plan, h->W, h->R, (const int32_t*)h->wptr_d.p,
                                        (const int32_t*)h->wlane_d.p, (const double*)h->wval_d.p,
                                        (const double*)h->X_d.p, (const int32_t*)h->status_d.p, x,
                                        (int32_t*)h->flag_d.p, h->stream));
  } else {
    CUDA_TRY(h, psp::launch_recover(h->plan, h->W, h->R, (const int32_t*)h->wptr_d.p,
                                    (const int32_t*)h->wlane_d.p, (const double*)h->wval_d.p,
                                    (const double*)h->X_d.p, (const int32_t*)h->status_d.p, x,
                                    (int32_t*)h->flag_d.p, h->stream));
  }
  h->recovered = true;
  return PSP_OK;
}

psp_status psp_residual(psp_handle h, const double* A_vals, int32_t W, int32_t R, const double* B,
                        const double* x, double* res_h) {
  if (!h || !A_vals || !B || !x || !res_h || W < 1 || R < 1) return PSP_ERR_ARG;
  if (!h->rowptr_d) return fail(h, PSP_ERR_STATE, "symbolic_analyse first");
  cudaSetDevice(h->device);
  psp_status s;
  int64_t ldb = h->n;
  if ((s = tv_A(h, A_vals, 1))) return s;   // (||A_hat x - b_hat|| = ||A x - b||)
  if ((s = tv_B(h, B, R, ldb))) return s;
  if ((s = ensure(h, h->res_d, sizeof(double) * (size_t)W * R))) return s;
  CUDA_TRY(h, psp::launch_residual(h->n, h->rowptr_d, h->colidx_d, A_vals, W, R, B, x,
                                   (double*)h->res_d.p, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(res_h, h->res_d.p, sizeof(double) * (size_t)W * R,
                              cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return PSP_OK;
}

psp_status psp_get_lane_status(psp_handle h, int32_t* status_h) {
  if (!h) return PSP_ERR_ARG;
  if (!h->factored) return fail(h, PSP_ERR_STATE, "factor_batch first");
  std::vector<int32_t> st(h->K);
  int32_t flag = 0;
  CUDA_TRY(h, cudaMemcpyAsync(st.data(), h->status_d.p, sizeof(int32_t) * h->K,
                              cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(&flag, h->flag_d.p, sizeof(int32_t), cudaMemcpyDeviceToHost,
                              h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  if (status_h) std::copy(st.begin(), st.end(), status_h);
  if (h->recovered && flag) return PSP_ERR_BATCH_INFEASIBLE;
  for (int32_t v : st)
    if (v) return PSP_ERR_ZERO_PIVOT;
  return PSP_OK;
}

psp_status psp_solve_host(psp_handle h, const double* A_vals_h, int32_t R, const double* B_h,
                          double pivot_tol, double* x_h) {
  if (!h || !A_vals_h || !B_h || !x_h || R < 1) return PSP_ERR_ARG;
  if (h->K == 0 || h->W == 0) return fail(h, PSP_ERR_STATE, "set_perturbations and set_weights first");
  cudaSetDevice(h->device);
  psp_status s;
  if (h->copy_stream) CUDA_TRY(h, cudaStreamSynchronize(h->copy_stream));   // (async calls' copies)
  if ((s = ensure(h, h->stageA_d, sizeof(double) * h->nnz_A))) return s;
  if ((s = ensure(h, h->stageB_d, sizeof(double) * (size_t)h->n * R))) return s;
  if ((s = ensure(h, h->stageX_d, sizeof(double) * (size_t)h->W * R * h->n))) return s;
  CUDA_TRY(h, cudaMemcpyAsync(h->stageA_d.p, A_vals_h, sizeof(double) * h->nnz_A,
                              cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(h->stageB_d.p, B_h, sizeof(double) * (size_t)h->n * R,
                              cudaMemcpyHostToDevice, h->stream));
  if (R == 1) {   // one right-hand side: psp_factor_solve_batch (fused when it pays)
    if ((s = psp_factor_solve_batch(h, (const double*)h->stageA_d.p, (const double*)h->stageB_d.p,
                                    pivot_tol, nullptr)))
      return s;
  } else {
    if ((s = psp_factor_batch(h, (const double*)h->stageA_d.p, pivot_tol, nullptr))) return s;
    if ((s = psp_solve_batch(h, R, (const double*)h->stageB_d.p, h->n))) return s;
  }
  if ((s = psp_recover(h, (double*)h->stageX_d.p))) return s;
  CUDA_TRY(h, cudaMemcpyAsync(x_h, h->stageX_d.p, sizeof(double) * (size_t)h->W * R * h->n,
                              cudaMemcpyDeviceToHost, h->stream));
  return psp_get_lane_status(h, nullptr);
}

// ---- multi-GPU: sharded lanes and the NCCL reduce of the partial sums (row a6) --------

psp_status psp_get_unique_id(void* id_h) {
  if (!id_h) return PSP_ERR_ARG;
  NcclApi& api = nccl_api();
  if (!api.ok) return PSP_ERR_UNSUPPORTED;
  ncclUniqueId id;
  if (api.getUniqueId(&id) != ncclSuccess) return PSP_ERR_NCCL;
  std::memcpy(id_h, &id, sizeof id);
  return PSP_OK;
}

psp_status psp_comm_init(psp_handle h, int32_t nranks, int32_t rank, const void* id_h) {
  if (!h || !id_h || nranks < 1 || rank < 0 || rank >= nranks) return PSP_ERR_ARG;
  if (h->device < 0) return fail(h, PSP_ERR_UNSUPPORTED, "host-only handle");
  NcclApi& api = nccl_api();
  if (!api.ok) return fail(h, PSP_ERR_UNSUPPORTED, "libnccl.so.2 not found");
  cudaSetDevice(h->device);
  if (h->comm) {
    api.commDestroy(h->comm);
    h->comm = nullptr;
  }
  ncclUniqueId id;
  std::memcpy(&id, id_h, sizeof id);
  ncclComm_t c = nullptr;
  const ncclResult_t r = api.commInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return fail(h, PSP_ERR_NCCL, "ncclCommInitRank: %s", api.errorString(r));
  h->comm = c;
  h->nranks = nranks;
  h->rank = rank;
  return PSP_OK;
}

psp_status psp_set_perturbations_shard(psp_handle h, int32_t K_global, const double* eps_h, const double* d_h,
                                       int32_t k_begin, int32_t k_count) {
  if (!h) return PSP_ERR_ARG;
  if (K_global < 1 || !eps_h || k_begin < 0 || k_count < 1 || k_begin + k_count > K_global)
    return fail(h, PSP_ERR_ARG, "shard [k_begin, k_begin + k_count) must lie in [0, K_global)");
  psp_status s = psp_set_perturbations(h, k_count, eps_h + k_begin, d_h);
  if (s) return s;
  h->K_global = K_global;
  h->k_begin = k_begin;
  return PSP_OK;
}

psp_status psp_shard_weights(int32_t W, const double* weights_h, int32_t K_global, int32_t k_begin,
                             int32_t k_count, int32_t* w_ptr_h, int32_t* w_lane_h, double* w_val_h,
                             int32_t* nnz_h) {
  if (W < 1 || !weights_h || K_global < 1 || k_begin < 0 || k_count < 1 || k_begin + k_count > K_global ||
      !w_ptr_h || !nnz_h)
    return PSP_ERR_ARG;
  int32_t q = 0;
  w_ptr_h[0] = 0;
  for (int32_t w = 0; w < W; ++w) {
    const double* row = weights_h + (size_t)w * K_global;
    for (int32_t k = 0; k < k_count; ++k) {
      const double v = row[k_begin + k];
      if (!std::isfinite(v)) return PSP_ERR_ARG;
      if (v != 0.0) {
        if (w_lane_h) w_lane_h[q] = k;
        if (w_val_h) w_val_h[q] = v;
        ++q;
      }
    }
    w_ptr_h[w + 1] = q;
  }
  *nnz_h = q;
  return PSP_OK;
}

psp_status psp_set_weights_dense(psp_handle h, int32_t W, const double* weights_h) {
  if (!h || !weights_h || W < 1) return PSP_ERR_ARG;
  if (h->K == 0) return fail(h, PSP_ERR_STATE, "set_perturbations first");
  std::vector<int32_t> ptr(W + 1), lane((size_t)W * h->K);
  std::vector<double> val((size_t)W * h->K);
  int32_t nnz = 0;
  psp_status s = psp_shard_weights(W, weights_h, h->K_global, h->k_begin, h->K, ptr.data(), lane.data(),
                                   val.data(), &nnz);
  if (s) return fail(h, s, "non-finite weight");
  return psp_set_weights(h, W, ptr.data(), lane.data(), val.data());
}

psp_status psp_recover_reduce(psp_handle h, double* x, int32_t root) {
  if (!h || !x) return PSP_ERR_ARG;
  if (root < -1 || root >= h->nranks) return fail(h, PSP_ERR_ARG, "root out of range");
  psp_status s = psp_recover(h, x);
  if (s) return s;
  if (!h->comm) return PSP_OK;   // (single process without a communicator: the local sums)
  NcclApi& api = nccl_api();
  const size_t count = (size_t)h->W * h->R * h->n;
  const ncclResult_t r = root < 0 ? api.allReduce(x, x, count, ncclFloat64, ncclSum, h->comm, h->stream)
                                  : api.reduce(x, x, count, ncclFloat64, ncclSum, root, h->comm, h->stream);
  if (r != ncclSuccess) return fail(h, PSP_ERR_NCCL, "%s: %s", root < 0 ? "ncclAllReduce" : "ncclReduce",
                                    api.errorString(r));
  return PSP_OK;
}

psp_status psp_ladder_weights(int32_t m, const double* s_h, double* eps_out_h, double* w_out_h) {
  if (m < 1 || m > 256 || !s_h || !eps_out_h || !w_out_h) return PSP_ERR_ARG;
  for (int32_t j = 0; j < m; ++j) {
    if (!(s_h[j] != 0.0) || !std::isfinite(s_h[j])) return PSP_ERR_ARG;
    for (int32_t l = 0; l < j; ++l)
      if (std::fabs(s_h[l]) == std::fabs(s_h[j])) return PSP_ERR_ARG;
  }
  for (int32_t j = 0; j < m; ++j) {
    long double tj = (long double)s_h[j] * (long double)s_h[j];
    long double beta = 1.0L;
    for (int32_t l = 0; l < m; ++l) {
      if (l == j) continue;
      long double tl = (long double)s_h[l] * (long double)s_h[l];
      beta *= tl / (tl - tj);
    }
    double half = (double)(beta / 2.0L);
    eps_out_h[2 * j] = std::fabs(s_h[j]);
    eps_out_h[2 * j + 1] = -std::fabs(s_h[j]);
    w_out_h[2 * j] = half;
    w_out_h[2 * j + 1] = half;
  }
  return PSP_OK;
}

}  // extern "C"
