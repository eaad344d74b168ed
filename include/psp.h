/*
 * psp.h — C ABI of the B200-native batched perturbation-induced static-pivoting
 * solver (arXiv 2311.11833, "Towards Perturbation-Induced Static Pivoting on
 * GPU-Based Linear Solvers"; PAPER.md = /root/reference/PAPER.md, line refs P:Lnnn).
 *
 * The library solves one sparse system A x = b by solving K diagonally perturbed
 * copies  A_k = A + eps_k * D  (D = diag(d)) WITHOUT pivoting — all copies share
 * one symbolic pattern and one static elimination order — and recombining the K
 * solutions with the paper's weights (Alg. 1):
 *
 *   psp_symbolic_analyse   once per sparsity pattern (host; ordering, fill, plans)
 *   psp_set_perturbations  signed eps_k per lane and d          (Alg. 1 step 1)
 *   psp_factor_batch       batched pivot-free numeric LU         (Alg. 1 step 2)
 *   psp_solve_batch        batched forward/back substitution     (Alg. 1 step 2)
 *   psp_factor_solve_batch the two fused for one right-hand side (Alg. 1 step 2)
 *   psp_set_weights +
 *   psp_recover            x_hat[w] = sum_k w[w][k] x_k          (Alg. 1 steps 3-4,
 *                                                                 Eq. (13)/(14))
 *
 * Conventions (all functions):
 *  - Every function returns psp_status (PSP_OK == 0).  Arguments are validated
 *    before any device work; on error nothing is launched and the handle state
 *    is unchanged (except psp_destroy).  psp_last_error_detail() gives a message.
 *  - Pointers suffixed _h are HOST memory.  Every other pointer is DEVICE memory
 *    of the handle's device.  Calls are stream-ordered on the handle's stream
 *    (like cuBLAS): device inputs must stay valid until the stream reaches the
 *    operation; the library never retains a caller pointer past the call (it
 *    copies patterns, eps, d and weights into its own memory).
 *  - Floating point is IEEE binary64.  Each lane's arithmetic is performed in the
 *    canonical order of DESIGN.md R11/R12 (one fma per "a - l*u" update, updates
 *    to each entry in ascending pivot order, forward substitution ascending,
 *    backward descending, true division), so per-lane results are bitwise
 *    reproducible and independent of K, the lane's position and the GPU count.
 *  - Handles are not thread-safe; distinct handles are independent.
 */
#ifndef PSP_H_
#define PSP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct psp_ctx* psp_handle;
typedef int32_t psp_status;

enum {
  PSP_OK = 0,
  PSP_ERR_ARG = 1,               /* NULL / out-of-range argument, malformed pattern */
  PSP_ERR_DIM = 2,               /* sizes inconsistent with the analysed pattern    */
  PSP_ERR_STATE = 3,             /* call order violated (e.g. factor before set_perturbations) */
  PSP_ERR_ZERO_PIVOT = 4,        /* >= 1 lane hit |u_pp| <= tol or a non-finite pivot
                                    (SPEC S:L46 ZeroPivot; P:L304 failure mode).  The
                                    batch is still complete; see per-lane status.     */
  PSP_ERR_BATCH_INFEASIBLE = 5,  /* a non-zero weight touches a failed lane */
  PSP_ERR_CUDA = 6,              /* CUDA runtime error; detail string has the code   */
  PSP_ERR_ALLOC = 7,             /* device or host allocation failed                 */
  PSP_ERR_UNSUPPORTED = 8,       /* feature not available in this build / handle     */
  PSP_ERR_NCCL = 9,              /* NCCL error; detail string has NCCL's message     */
  PSP_ERR_STRUCT_SINGULAR = 10   /* PSP_OPT_TRANSVERSAL: no perfect matching (the pattern
                                    is structurally singular)                        */
};

/* Elimination orders for psp_symbolic_analyse (R13). */
enum {
  PSP_ORDER_NATURAL = 0,         /* the given order                                  */
  PSP_ORDER_MINDEG = 1,          /* exact minimum degree on pattern(A+A^T), ties to
                                    the lowest original index                        */
  PSP_ORDER_USER = 2,            /* user_perm_h[new] = old                          */
  PSP_ORDER_MINDEG_FIRST = 3     /* eliminate `first_node` first, then MINDEG: the
                                    'leading-zero' regime of P:L304                  */
};

typedef struct {
  int32_t n;                     /* matrix dimension                                 */
  int32_t nnz_A;                 /* stored entries of A                              */
  int32_t nnz_LU;                /* slots of the filled L+U pattern (incl. diagonal) */
  int32_t nnz_L;                 /* strictly-lower slots                             */
  int32_t n_struct_zero_diag;    /* diagonal positions absent from A's pattern       */
  int32_t n_levels;              /* elimination-tree height (levels of the schedule) */
  int64_t factor_fma;            /* fused multiply-adds per lane in the factorisation */
  int64_t factor_div;            /* divisions per lane (strictly-lower slots)        */
  int64_t solve_fma;             /* fmas per lane per right-hand side (fwd + bwd)    */
  int32_t max_live;              /* pending slots per lane: peak number of partially-
                                    updated entries of the right-looking factorisation */
  int32_t solve_live;            /* live slots per lane of the triangular solves     */
  int32_t births;                /* pending-slot initialisations per lane            */
  int32_t factor_groups;         /* G: thread groups sharing one slab in the factor
                                    kernel                            */
  int32_t factor_lanes_per_thread; /* J: adjacent lanes per thread; a slab holds
                                    32/G*J lanes                                     */
  int32_t factor_slab_warps;     /* P: warps sharing one slab (rows split)          */
  int32_t factor_warps_per_cta;  /* consumer warps per factor CTA                    */
  int32_t factor_pend_smem;      /* 1: pending slots in shared memory, 0: global,
                                    2: 4 warps per CTA in tensor memory, the rest in
                                    shared memory (PSP_OPT_FACTOR_TMEM)               */
  int32_t solve_live_smem;       /* 1: solve's live slots in shared memory, 0: global,
                                    2: tensor memory (PSP_OPT_SOLVE_TMEM)             */
  /* the augmented program of psp_factor_solve_batch ([A | b]): aug_ok = 2 fused, 1
   * available but slower (a weaker slot store: the call runs factor + solve), 0 none */
  int32_t aug_ok, aug_max_live, aug_warps_per_cta, aug_pend_smem;
  /* capacity-planned programs (PSP_OPT_FACTOR_SPILL): spill_ok bit 0 plain, bit 1 augmented
   * available; spill_cap = slots per lane; spill_ops = spill + reload operations per lane
   * (plain program; aug_spill_ops for [A | b]); spill_entries = spill-area entries per lane;
   * spill_warps_per_cta = warps of the 2-CTA-per-SM launch */
  int32_t spill_ok, spill_cap, spill_ops, spill_entries, aug_spill_ops, spill_warps_per_cta;
  /* PSP_OPT_SKIP_ZERO_ROWS: struct_zero_l = multipliers l_{i p} of the (symmetrised) fill that
   * are structural zeros of A's own pattern (0 with the option off); skipped_rows /
   * aug_skipped_rows = rows the capacity-planned programs (plain / [A | b]) skip */
  int32_t struct_zero_l, skipped_rows, aug_skipped_rows;
} psp_symbolic_info;

/* ---- lifetime ---------------------------------------------------------------- */

/* Create a handle bound to CUDA device `device` and stream `cuda_stream`
 * (a cudaStream_t; NULL = the legacy default stream).  *out receives the handle.
 * device < 0 creates a HOST-ONLY handle: psp_symbolic_analyse and
 * psp_get_symbolic_info work (no device plans are uploaded); every numeric call
 * returns PSP_ERR_UNSUPPORTED or PSP_ERR_STATE.  Errors: ARG, CUDA (bad device). */
psp_status psp_create(psp_handle* out, int32_t device, void* cuda_stream);

/* Release all device and host memory of the handle (synchronises its stream). */
psp_status psp_destroy(psp_handle h);

/* Options (set before psp_symbolic_analyse; they apply to the next analysis):
 *  PSP_OPT_FACTOR_GROUPS  0 (default): automatic; else G in {1, 2, 4}: the factor kernel
 *                         splits each warp into G groups sharing one slab.
 *  PSP_OPT_FACTOR_LANES   0 (default): automatic; else J in {1, 2} adjacent lanes per
 *                         thread (J <= G); a slab holds 32/G*J lanes.
 *                         Results are bitwise independent of G and J.
 *  PSP_OPT_FACTOR_SLAB_WARPS 0 (default): automatic; else P in {1, 2} warps sharing one
 *                         slab (G = J = 1 only), the rows of each pivot split between them.
 *  PSP_OPT_FACTOR_PAIRS   1 (default): fuse supernode pivot pairs (p, p+1 with
 *                         L(:,p) = {p+1} u L(:,p+1)) into one record; 0: off.
 *  PSP_OPT_SKIP_ZERO_ROWS 1 (default): the symbolic analysis marks the multipliers l_{i p} that
 *                         are structural zeros of A's own (unsymmetric) pattern inside the fill of
 *                         the symmetrised pattern, and the capacity-planned batch factor stores
 *                         l = 0 for them instead of the division and the row update
 *                         fma(-0, u, x) = x (the identity the sparse code already relies on for
 *                         entries outside the fill); 0: every row of the fill is computed.
 *                         Takes effect at the next psp_symbolic_analyse.
 *  PSP_OPT_FACTOR_WARPS   0 (default): automatic; else consumer warps per factor CTA
 *                         (1..16, capped by shared memory).
 *  PSP_OPT_FACTOR_TMEM    0 (default): automatic; 1: require, 2: disable the factor
 *                         variant whose warps 0..3 keep their pending slots in tensor
 *                         memory (G = J = P = 1, 2 * slots <= 512).
 *                         Results are bitwise independent of this option.
 *  PSP_OPT_SOLVE_TMEM     0 (default) or 2: off; 1: require the solve
 *                         variant that keeps its live y/x slots in tensor memory
 *                         (DESIGN.md §5).  Results are bitwise independent of it.
 *  PSP_OPT_PHASE_EVENTS   0 (default); 1: record CUDA events around the factor and the
 *                         solve kernel launches (for psp_get_phase_times; any time).
 *  PSP_OPT_GROWTH         0 (default); 1: every factorisation also computes the per-lane
 *                         growth factor (psp_get_lane_growth; any time).
 *  PSP_OPT_COOP           0 (default): automatic — batches of K <= 8 x the SM count use the
 *                         cooperative kernels (one CTA per system, its factor in shared
 *                         memory, etree-level steps); 1: always (when the
 *                         factor fits shared memory); 2: never.  Bitwise-neutral.
 *  PSP_OPT_FACTOR_SPILL   0 (default): automatic — when the pending set exceeds 127 slots
 *                         per lane and the batch needs more than one round of the plain
 *                         launch, factor with the capacity-planned program (<= 127 slots,
 *                         the entries with the furthest next use spilled to a per-lane
 *                         global area and reloaded before their next use):
 *                         2 CTAs x 7 warps per SM instead of 1 x 7-8; 1: always (when a
 *                         launch fits); 2: never.  Bitwise-neutral.
 *  PSP_OPT_COOP_GLOBAL    0 (default): automatic -- when the cooperative kernels' factor
 *                         image does not fit shared memory (large n, e.g. SURVEY §8(d)
 *                         configs 3-4) and K <= 8 x the SM count, factor and solve with the
 *                         global-memory level-scheduled kernels (one CTA per system, the
 *                         factor image lane-major in the handle's factor storage, the same
 *                         etree-level schedule: bitwise the batch kernels); 1: always (when
 *                         built: set before psp_symbolic_analyse); 2: never.  Bitwise-neutral.
 *  PSP_OPT_FACTOR_HYBRID  (capacity-planned factor) 1: every warp keeps its pending slots
 *                         0..63 in tensor memory and 64..127 in shared memory (or all 128 in
 *                         TMEM when alone on its lane quarter) instead of 4 TMEM warps + 3
 *                         shared-memory warps; 3: mixed lanes per thread (4 TMEM warps x 64
 *                         lanes + up to 6 shared-memory warps x 32 lanes); 0 (default) / 2:
 *                         the default layout (measured fastest).  Bitwise-neutral.
 *  PSP_OPT_DATAFLOW       1: psp_factor_solve_batch on a batch that takes the cooperative
 *                         kernels runs ONE fused kernel instead: a CTA per system whose
 *                         factor entries, forward rows and backward rows are dataflow tasks
 *                         walked by one lane per warp (ready flags in shared memory, no level
 *                         barriers); same arithmetic, bitwise; 0 (default): only for small
 *                         systems (nnz_LU <= 1024, where it measured faster); 2: never.
 *  PSP_OPT_TRANSVERSAL    0 (default); 1: the structural pre-pass of P:L304 ("the
 *                         Hopcroft-Karp algorithm (which permutes a matrix by moving
 *                         non-zeros onto the diagonal)"): the analysis computes a maximum
 *                         matching q (columns -> rows, Hopcroft-Karp in a fixed order,
 *                         DESIGN.md R20; psp_get_transversal) and analyses and factors
 *                         A_hat = A[q, :] (zero-free diagonal) instead of A: every later call
 *                         takes A's values and b in the caller's ordering and gathers them
 *                         (A_hat x = b[q] has the same solution x); the perturbation
 *                         eps_k d_j goes on A_hat's diagonal entry (j, j).  The analysis
 *                         fails with PSP_ERR_STRUCT_SINGULAR when no perfect matching
 *                         exists.  Not with a dense D or psp_estimate_rho (UNSUPPORTED).
 *  PSP_OPT_PATH           PSP_PATH_SPARSE (default) or PSP_PATH_DENSE: which kernels the
 *                         next factorisations run (may change at any time; the
 *                         solve follows the last factorisation).  DENSE is the paper's own
 *                         formulation (a dense no-pivot getrf/trsm per
 *                         perturbed copy, "getrf_batched! / trsm_batched!"): every lane's
 *                         P (A + eps_k D) P^T as a dense matrix (n padded to a multiple of
 *                         32, 8 * N^2 bytes per lane), right-looking blocked elimination in
 *                         32-column panels with the trailing updates on the FP64 tensor
 *                         path (DMMA), and dense triangular solves.  Same pivot order
 *                         (perm; PSP_ORDER_NATURAL = the paper-replica mode), statuses,
 *                         tolerance and X layout as the sparse path; the arithmetic is
 *                         blocked (NOT bitwise the canonical order, R19).  Needs
 *                         N x 33 x 8 bytes <= 227 KB of shared memory (n <= 864).  The
 *                         only path for a dense D (psp_set_perturbation_matrix).
 * Errors: ARG (STATE: PSP_OPT_PHASE_EVENTS on a host-only handle). */
enum { PSP_PATH_SPARSE = 0, PSP_PATH_DENSE = 1 };
enum { PSP_OPT_FACTOR_GROUPS = 1, PSP_OPT_FACTOR_WARPS = 2, PSP_OPT_FACTOR_LANES = 3,
       PSP_OPT_FACTOR_SLAB_WARPS = 4, PSP_OPT_FACTOR_PAIRS = 5, PSP_OPT_FACTOR_TMEM = 6,
       PSP_OPT_SOLVE_TMEM = 7, PSP_OPT_PHASE_EVENTS = 8, PSP_OPT_GROWTH = 9,
       PSP_OPT_COOP = 10, PSP_OPT_FACTOR_SPILL = 11, PSP_OPT_PATH = 12, PSP_OPT_COOP_GLOBAL = 13,
       PSP_OPT_TRANSVERSAL = 14, PSP_OPT_DATAFLOW = 15, PSP_OPT_FACTOR_HYBRID = 16,
       PSP_OPT_SKIP_ZERO_ROWS = 17 };
psp_status psp_set_option(psp_handle h, int32_t option, int64_t value);

/* Rebind the handle to another stream of the same device.  Synchronises the old stream
 * first (the handle's programs, factor and staging buffers are reused by the next call,
 * so work still queued on the old stream must not overlap it).  Errors: ARG, CUDA. */
psp_status psp_set_stream(psp_handle h, void* cuda_stream);

const char* psp_status_string(psp_status s);
const char* psp_last_error_detail(psp_handle h);

/* ---- symbolic analysis (a static pivot sequence "computed once, and
 *      perpetually reused"; host-side, once per pattern) ---------------------- */

/* Analyse the pattern of the n x n CSR matrix A (row_ptr_h[n+1], col_idx_h[nnz];
 * column indices strictly increasing within each row, no duplicates).  Computes
 * the elimination order (`ordering`, see enum; user_perm_h[n] for USER, else may
 * be NULL; first_node for MINDEG_FIRST, else ignored), the filled L+U pattern of
 * pattern(A + A^T + I), the batch-major slot layout and the device plans.
 * Discards any previous analysis, perturbations, weights and results.
 * Errors: PSP_ERR_ARG (malformed pattern / permutation), PSP_ERR_ALLOC. */
psp_status psp_symbolic_analyse(psp_handle h, int32_t n, const int32_t* row_ptr_h,
                                const int32_t* col_idx_h, int32_t ordering,
                                const int32_t* user_perm_h, int32_t first_node);

/* PSP_OPT_TRANSVERSAL: q_h[n] receives the matching of the last analysis (row q[j] of A is
 * row j of the analysed A_hat).  Errors: ARG, STATE (no transversal analysed). */
psp_status psp_get_transversal(psp_handle h, int32_t* q_h);

/* Statistics of the analysis; perm_h (may be NULL) receives perm[new] = old. */
psp_status psp_get_symbolic_info(psp_handle h, psp_symbolic_info* info_h, int32_t* perm_h);

/* ---- perturbations (Alg. 1 step 1; Eqs. (5)-(6)) ---------- */

/* Set the K lanes this handle owns: lane k solves (A + eps_h[k] * diag(d_h)) x = b.
 * eps_h[K] are the signed perturbations (e.g. the ladder [+s1,-s1,+s2,-s2,...]
 * with s_j = alpha_j * eps); d_h[n] is D's diagonal in the ORIGINAL
 * ordering (the paper scales ||D||_1 = max|d_i| = 1; the library does not
 * rescale).  The perturbed diagonal entry is a_ii + (eps_k * d_i) (two roundings).
 * Allocates the batch-major factor storage (8 * nnz_LU * K bytes).  A multi-GPU
 * caller passes only its shard of eps.  Errors: ARG, STATE, ALLOC. */
psp_status psp_set_perturbations(psp_handle h, int32_t K, const double* eps_h, const double* d_h);

/* ---- numeric phase ------------------------------------------------------------ */

/* Batched pivot-free LU (Alg. 1 step 2; the getrf_batched of P:L310 made
 * sparse).  A_vals[nnz_A] (device) are A's values in the CSR order given to
 * psp_symbolic_analyse.  pivot_tol > 0: a pivot with |u_pp| <= pivot_tol or a
 * non-finite pivot fails the lane; pivot_tol <= 0 selects n * 2^-52 * ||A||_1
 * (SPEC S:L95), computed on the device from A_vals.  Per-lane status (0 ok, else
 * 1 + first failing permuted pivot position) is kept on the device; if
 * lane_status is non-NULL (device int32[K]) it is also written there.  Failed
 * lanes do not stop the batch.  Asynchronous: returns PSP_OK without checking
 * statuses (use psp_get_lane_status).  Errors: ARG, STATE, CUDA. */
psp_status psp_factor_batch(psp_handle h, const double* A_vals, double pivot_tol,
                            int32_t* lane_status);

/* Batched forward (unit L, ascending) and backward (U, descending) substitution
 * for R right-hand sides shared by all lanes (Alg. 1 step 2; the trsm pair of
 * P:L310).  B (device) is n x R column-major with leading dimension ldb >= n, in
 * the ORIGINAL ordering.  Solutions stay in library memory (see psp_get_solutions).
 * Errors: ARG, STATE, ALLOC, CUDA. */
psp_status psp_solve_batch(psp_handle h, int32_t R, const double* B, int64_t ldb);

/* psp_factor_batch + psp_solve_batch for ONE right-hand side b (device, n values,
 * ORIGINAL ordering) with the forward substitution fused into the factorisation:
 * the factor kernel eliminates the augmented matrix [A | b] (b as a column that is
 * never a pivot), so y = L^{-1} b is produced by the same updates, in the same
 * canonical order (y_i = fma(-l_ip, y_p, y_i), p ascending), as the separate forward
 * pass would, and the solve runs the backward pass only.  Results (factor, lane
 * statuses, solutions) are bitwise those of psp_factor_batch + psp_solve_batch with
 * R = 1.  Saves the forward pass's read of L and its interpretation overhead
 * (DESIGN.md §5).  When the augmented program would need a weaker pending-slot store
 * than the plain one (symbolic info aug_ok != 2) it runs psp_factor_batch +
 * psp_solve_batch instead.  Errors: ARG, STATE, ALLOC, CUDA. */
psp_status psp_factor_solve_batch(psp_handle h, const double* A_vals, const double* b,
                                  double pivot_tol, int32_t* lane_status);

/* Many Jacobians of one pattern in one launch (the Newton-Raphson steps /
 * the 25 voltage starts of P:L302, P:L323 share J's sparsity pattern): the K lanes are split
 * into n_jac equal contiguous groups (n_jac must divide K) and lane k factors
 * A_j + eps_k D with j = k / (K / n_jac).  A_vals (device) holds n_jac value arrays of nnz_A
 * entries back to back (CSR order of the analysed pattern).  pivot_tol <= 0 selects each
 * Jacobian's own n * 2^-52 * ||A_j||_1.  Runs the kernels that take one CTA per system:
 * the cooperative (K <= 8 x SMs, PSP_OPT_COOP), global-memory level-scheduled
 * (PSP_OPT_COOP_GLOBAL) or dense (PSP_OPT_PATH) kernels -- the same arithmetic as
 * psp_factor_batch, bitwise; else PSP_ERR_UNSUPPORTED (factor such batches per Jacobian
 * with psp_factor_batch: values-only refactorisation).  n_jac = 1 is psp_factor_batch.
 * Errors: ARG (n_jac does not divide K), STATE, UNSUPPORTED, ALLOC, CUDA. */
psp_status psp_factor_batch_multi(psp_handle h, int32_t n_jac, const double* A_vals, double pivot_tol,
                                  int32_t* lane_status);

/* Solves after psp_factor_batch_multi with each Jacobian's own R right-hand sides: lane k
 * (Jacobian j) solves for B + j * jac_stride (device; n x R column-major with leading
 * dimension ldb, ORIGINAL ordering).  Solutions as psp_solve_batch.  Errors: ARG
 * (jac_stride < (R - 1) ldb + n), STATE (no multi-Jacobian factorisation), UNSUPPORTED,
 * ALLOC, CUDA. */
psp_status psp_solve_batch_multi(psp_handle h, int32_t R, const double* B, int64_t ldb, int64_t jac_stride);

/* Iterative-refinement baseline (the comparison P:L336 asks for):
 * static pivoting by one perturbation per lane plus fixed-precision iterative refinement
 * against the UNPERTURBED A, every lane k with its own factor F_k = A + eps_k D from the
 * last factorisation:  x^0 = F_k^{-1} b;  x^i = x^{i-1} + F_k^{-1} (b - A x^{i-1}), i = 1..iters
 * (residual one fma per CSR entry in order, the correction by the factor's substitutions,
 * the update one rounded add -- bitwise the oracle's refine).  Converges to x* when
 * |eps_k| rho((A + eps_k D)^{-1} D) < 1: x* - x^i = (eps_k M_k)^{i+1} x*.  A_vals: the
 * (device) values the factorisation used; b: device n values, ORIGINAL ordering; x_out:
 * device K x n (lane-major, ORIGINAL ordering) receives x^iters.  Needs per-lane
 * right-hand sides: the cooperative, global level-scheduled or dense kernels; else
 * PSP_ERR_UNSUPPORTED.  Overwrites the handle's solutions (psp_get_solutions: solve again).
 * Errors: ARG, STATE, UNSUPPORTED, ALLOC, CUDA. */
psp_status psp_refine(psp_handle h, const double* A_vals, const double* b, int32_t iters, double* x_out);

/* Spectral radius rho(A^-1 D) by power iteration (Eq. (4)'s rho; the convergence
 * premise eps_c = m eps < 1 / rho of Theorem 1),
 * reusing the handle's factorisation: A^-1 r is applied as the recovered solution w of
 * the method itself (psp_solve_batch with R = 1 and b = r, psp_recover, row w), so it
 * carries the method's O(eps^2m) truncation error.  v_0 = v0_h (n values, ORIGINAL
 * ordering, nonzero); v_{t+1} = x_hat(D v_t) / ||x_hat(D v_t)||_2, rho_t = ||x_hat(D v_t)||_2
 * (||v_t||_2 = 1); stops when |rho_t - rho_{t-1}| < rtol * rho_t or after max_iter
 * iterations.  Outputs rho_h, iters_h (may be NULL), converged_h (1 / 0, may be NULL).
 * Overwrites the solutions and the recovered rows of the handle (the last iterate).
 * Synchronous.  Errors: ARG, STATE (factor_batch and set_weights first),
 * BATCH_INFEASIBLE (non-finite iterate), CUDA. */
psp_status psp_estimate_rho(psp_handle h, int32_t w, int32_t max_iter, double rtol,
                            const double* v0_h, double* rho_h, int32_t* iters_h,
                            int32_t* converged_h);

/* Per-lane growth factor of the last factorisation made with PSP_OPT_GROWTH = 1
 * (growth monitoring): growth_h[k] = max|U_k| / max|A_k| with
 * A_k = A + eps_k D (its diagonal rounded as in the factorisation: a_ii + (eps_k d_i)),
 * max|U_k| over the lane's upper factor including the pivots.  Synchronises.  For a
 * failed lane (status != 0) the value covers the factor as computed.  Errors: ARG,
 * STATE, CUDA. */
psp_status psp_get_lane_growth(psp_handle h, double* growth_h);

/* With PSP_OPT_PHASE_EVENTS on: the MEAN device time (ms, cudaEventElapsedTime between
 * library events recorded on the handle's stream right before and after each launch) of
 * the factor kernels (ms_h[0]) and of the solve kernels (ms_h[1]) launched since the
 * previous psp_get_phase_times call (or since the option was switched on); 0 for a phase
 * with no launch.  Resets the accumulation.  Synchronises on the recorded events.
 * Errors: ARG, STATE, CUDA. */
psp_status psp_get_phase_times(psp_handle h, float* ms_h);

/* Which kernels the last numeric calls launched (introspection for tests and launch
 * censuses): kernels_h[0] = factor kernel of the last factorisation,
 * kernels_h[1] = 1 if it eliminated the augmented [A | b] (forward substitution fused),
 * kernels_h[2] = solve kernel of the last solve, kernels_h[3] = 1 if that solve ran the
 * forward pass (0: backward only, y came from the fused factor).  Kernel ids: PSP_KERNEL_*
 * (0 = none launched yet).  Errors: ARG. */
enum { PSP_KERNEL_NONE = 0,
       PSP_KERNEL_COOP = 1,        /* cooperative small-batch kernels (CTA per system)      */
       PSP_KERNEL_BATCH = 2,       /* batch kernels, slots in shared (or global) memory      */
       PSP_KERNEL_BATCH_TMEM = 3,  /* batch kernels, slots in tensor memory + shared memory  */
       PSP_KERNEL_BATCH_SPILL = 4, /* batch factor, capacity-planned slots (TMEM + shared)
                                      with idle entries spilled to global memory            */
       PSP_KERNEL_DENSE = 5,       /* dense path (PSP_OPT_PATH): blocked LU / solves, DMMA   */
       PSP_KERNEL_COOP_GLOBAL = 6, /* level-scheduled CTA per system, factor image in global
                                      memory (large n, PSP_OPT_COOP_GLOBAL)                  */
       PSP_KERNEL_DATAFLOW = 7     /* fused factor + solve by dataflow (PSP_OPT_DATAFLOW)     */
};
psp_status psp_get_last_kernels(psp_handle h, int32_t* kernels_h);

/* Copy the per-lane solutions to X (device, K x R x n, lane-major, ORIGINAL
 * ordering): X[(k*R + r)*n + i] = x_k,r[i].  Errors: ARG, STATE. */
psp_status psp_get_solutions(psp_handle h, double* X);

/* Copy lane k's factor to the host (synchronises the stream): vals_h[nnz_LU] in the
 * pivot-major layout of the permuted matrix: first the L region (for p = 0..n-1: l_{i p}
 * for the rows i of L(:, p) ascending), then the DU region (for p = 0..n-1: u_pp, then
 * u_{p i} for the same i).  The row sets are those of the symbolic factorisation of
 * pattern(A + A^T + I) in the order of psp_get_symbolic_info's perm.  Errors: ARG, STATE. */
psp_status psp_get_factor(psp_handle h, int32_t k, double* vals_h);

/* Dense path only: copy lane k's dense factor to the host (synchronises): lu_h[n*n]
 * row-major in the PERMUTED order, strict lower part = L (unit diagonal implied), upper
 * part with the diagonal = U (the layout of a LAPACK-style getrf without pivots, row-major).
 * Errors: ARG, STATE (no dense factorisation), CUDA. */
psp_status psp_get_dense_factor(psp_handle h, int32_t k, double* lu_h);

/* A general perturbation matrix D (footnote P:L72; "all entries of
 * the perturbation matrix ... normally distributed"): lane k then factors
 * A + eps_k * D entry by entry (a_ij + (eps_k * D_ij), a_ij = 0 outside the pattern) instead
 * of A + eps_k * diag(d).  D_h: n x n row-major, ORIGINAL ordering, finite (host; copied,
 * permuted, 8 n^2 bytes on the device); NULL returns to the diagonal d of
 * psp_set_perturbations.  A dense D has no shared sparse pattern: factorisations need
 * PSP_OPT_PATH = PSP_PATH_DENSE (else PSP_ERR_UNSUPPORTED).  psp_estimate_rho uses it.
 * Invalidates the factorisation.  Errors: ARG, STATE (analyse first), UNSUPPORTED
 * (host-only handle), ALLOC, CUDA. */
psp_status psp_set_perturbation_matrix(psp_handle h, const double* D_h);

/* Recombination weights (Remark 2 / Eq. (13), with the pair average of
 * Eq. (avg_hats), folded in: weight beta_j / 2 on each sign).  CSR over
 * W recovered solutions: entries w_ptr_h[w]..w_ptr_h[w+1]-1 list local lanes
 * w_lane_h[] (strictly ascending within a row, 0 <= lane < K) and weights w_val_h[].
 * Exact-zero weights are dropped.  Copied to the device.  Errors: ARG, STATE. */
psp_status psp_set_weights(psp_handle h, int32_t W, const int32_t* w_ptr_h,
                           const int32_t* w_lane_h, const double* w_val_h);

/* x[(w*R + r)*n + i] = sum over the row's lanes k (ascending) of w * x_k,r[i]
 * (ORIGINAL ordering; one fma per term, Alg. 1 steps 3-4).  x is device memory
 * W x R x n.  With lanes sharded across GPUs this is the rank-local partial sum;
 * the caller reduces it (sum) across ranks.  A non-zero weight on a failed lane
 * yields NaN for that solution and raises the batch-infeasible flag
 * (psp_get_lane_status); the flag is cleared at the start of every psp_recover, so it
 * always describes the last combination.  Errors: ARG, STATE, CUDA. */
psp_status psp_recover(psp_handle h, double* x);

/* Synchronise the stream and copy per-lane status to status_h[K] (may be NULL).
 * Returns PSP_ERR_BATCH_INFEASIBLE if the last psp_recover raised its flag, else
 * PSP_ERR_ZERO_PIVOT if any lane failed, else PSP_OK. */
psp_status psp_get_lane_status(psp_handle h, int32_t* status_h);

/* End-to-end call with HOST buffers (the e2e path): copies A_vals_h[nnz_A] and
 * B_h (n x R col-major) to the device, runs factor (pivot_tol as above), solve and
 * recover, copies x_h[W x R x n] back and synchronises.  Pinned host memory gives
 * asynchronous copies; pageable works.  Returns like psp_get_lane_status. */
psp_status psp_solve_host(psp_handle h, const double* A_vals_h, int32_t R, const double* B_h,
                          double pivot_tol, double* x_h);

/* Pipelined form of psp_solve_host for a stream of systems: enqueues the same work
 * (A_vals_h and B_h copied up on a library-owned input stream into a double-buffered
 * staging pair, factor + solve + recover on the handle's stream, x_h copied back on a
 * second library-owned stream from a double-buffered device staging area) and returns
 * without waiting, so the copies of one call overlap the kernels of its neighbours.
 * A_vals_h, B_h and x_h
 * must be pinned and stay valid (x_h unread) until psp_synchronize; lane statuses via
 * psp_get_lane_status afterwards.  Errors: ARG, STATE, ALLOC, CUDA. */
psp_status psp_solve_host_async(psp_handle h, const double* A_vals_h, int32_t R, const double* B_h,
                                double pivot_tol, double* x_h);

/* Synchronise the handle's streams (its stream and the copy stream of
 * psp_solve_host_async). */
psp_status psp_synchronize(psp_handle h);

/* Re-perturbation of failed ladders (a perturbed lane
 * can still meet a (near-)zero pivot; another perturbation size avoids it).  After a
 * factorisation, every weight row of psp_set_weights holding a failed lane (status != 0)
 * has the eps of all its lanes multiplied by `scale`; other lanes keep theirs.  The
 * paper's weights (Remark 2: beta_j depends only on ratios of the squared magnitudes)
 * are invariant under a common scale of a ladder, so the rows' weights stay valid —
 * caller-supplied weights that are not scale-invariant must be reset by the caller.
 * n_rows_h (may be NULL) = rows rescaled.  When a row was rescaled the factorisation is
 * invalidated: the caller factors again (same A_vals).  Synchronous (reads the
 * statuses).  Errors: ARG (scale zero or non-finite), STATE (factor_batch and
 * set_weights first), CUDA. */
psp_status psp_rescale_failed_rows(psp_handle h, double scale, int32_t* n_rows_h);

/* The handle's current eps[K] (after psp_rescale_failed_rows).  Errors: ARG, STATE. */
psp_status psp_get_perturbations(psp_handle h, double* eps_h);

/* Optional error test ("Optionally, test the solution error",
 * P:L323): res_h[w * R + r] = || A x[w][r] - B[:, r] ||_2 for W x R candidate
 * solutions.  A_vals (device, nnz_A, CSR order of the analysed pattern), B (device,
 * n x R col-major, leading dimension n), x (device, W x R x n, ORIGINAL ordering, e.g.
 * psp_recover's output).  Row i: t_i = (sum_q A_q x_{c_q}, ascending q, fma) - b_i;
 * the squares are summed per thread in ascending i and then over a fixed tree, so
 * the result is deterministic (not the oracle's summation order: parity within a
 * relative 1e-12 of ||A|| ||x|| + ||b||).  Non-finite x gives a non-finite residual.
 * Synchronous.  Errors: ARG (W < 1, R < 1, null), STATE (symbolic_analyse first), CUDA. */
psp_status psp_residual(psp_handle h, const double* A_vals, int32_t W, int32_t R, const double* B,
                        const double* x, double* res_h);

/* ---- multi-GPU: one handle per GPU (one process per GPU), the perturbation batch
 *      sharded over the ranks, the partial sums of Alg. 1 steps 3-4 reduced with NCCL
 *      (DESIGN.md §6).  NCCL is loaded at run time
 *      (libnccl.so.2, the process's already-loaded copy when there is one). ---------- */

/* The NCCL unique id (128 bytes) of a new communicator, on one rank; the caller
 * distributes it to every rank (e.g. torch.distributed broadcast).  Errors: ARG,
 * UNSUPPORTED (no libnccl), NCCL. */
psp_status psp_get_unique_id(void* id_h);

/* Join the communicator `id_h` as `rank` of `nranks` (collective over the ranks; the
 * handle's device).  Replaces an earlier communicator of the handle; psp_destroy frees
 * it.  nranks = 1 is valid (the reduce is then a local copy through NCCL).  Errors: ARG,
 * UNSUPPORTED (host-only handle, no libnccl), NCCL. */
psp_status psp_comm_init(psp_handle h, int32_t nranks, int32_t rank, const void* id_h);

/* psp_set_perturbations for a shard: this rank owns the global lanes [k_begin, k_begin +
 * k_count) of a batch of K_global lanes (eps_h has K_global entries; local lane k is global
 * lane k_begin + k).  Contiguous shards keep each ladder's lanes together where the split
 * allows; correctness never depends on it (the weights are global).  Errors: as
 * psp_set_perturbations, ARG for a shard outside [0, K_global). */
psp_status psp_set_perturbations_shard(psp_handle h, int32_t K_global, const double* eps_h,
                                       const double* d_h, int32_t k_begin, int32_t k_count);

/* Pure host helper: the rows of the dense weights_h[W][K_global] (row-major) restricted to
 * the shard [k_begin, k_begin + k_count), as CSR over LOCAL lanes: w_ptr_h[W + 1],
 * w_lane_h / w_val_h (capacity W * k_count; either may be NULL to count only), exact zeros
 * dropped, *nnz_h entries.  Errors: ARG (bad shard, non-finite weight). */
psp_status psp_shard_weights(int32_t W, const double* weights_h, int32_t K_global, int32_t k_begin,
                             int32_t k_count, int32_t* w_ptr_h, int32_t* w_lane_h, double* w_val_h,
                             int32_t* nnz_h);

/* psp_set_weights from dense GLOBAL weights weights_h[W][K_global] (row-major; the
 * combination of Eq. (13) with the pair average folded in): this rank keeps its shard's
 * columns (psp_shard_weights).  Errors: ARG, STATE. */
psp_status psp_set_weights_dense(psp_handle h, int32_t W, const double* weights_h);

/* Collective over the communicator's ranks (all call it): each rank's partial sums
 * x[w][r][i] = sum over its lanes of w * x_k,r[i] (psp_recover, into x), then the sum over
 * the ranks with NCCL on the handle's stream, in place: root >= 0 ncclReduce (the result
 * on `root`; other ranks keep their partial sums), root = -1 ncclAllReduce (every rank).
 * x: device, W x R x n on every rank.  Without psp_comm_init: psp_recover (local sums).
 * The summation order over ranks is NCCL's (R16).  Errors: ARG (root out of
 * range), STATE, CUDA, NCCL. */
psp_status psp_recover_reduce(psp_handle h, double* x, int32_t root);

/* ---- host helper (pure) --------------------------------------------------------- */

/* Paper ladder (Remark 2): for m magnitudes s_h[j] (distinct, non-zero),
 * eps_out_h[2m] = [+s_1, -s_1, ..., +s_m, -s_m] and w_out_h[2m] = beta_j / 2 on both
 * signs, beta_j = prod_{l != j} s_l^2 / (s_l^2 - s_j^2) (the solution of
 * Gamma_m^T beta = e_1, computed in long double without forming Gamma).
 * Errors: ARG (m < 1, m > 256, repeated or zero magnitude). */
psp_status psp_ladder_weights(int32_t m, const double* s_h, double* eps_out_h, double* w_out_h);

#ifdef __cplusplus
}
#endif
#endif /* PSP_H_ */
