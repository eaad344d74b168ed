// Host-side symbolic planning (see psp_plan.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace psp {

struct EtreeResult {
  std::vector<std::vector<int32_t>> lcol;  // strictly-lower rows of each column (sorted)
  std::vector<int32_t> parent, level;
  int32_t height = 0;
};

// Program and layout produced once per pattern; uploaded into a DevicePlan.
struct HostPlan {
  int32_t n = 0, nnz_LU = 0, nnz_L = 0, c_max = 0;
  int64_t factor_fma = 0, solve_fma = 0;
  std::vector<int32_t> perm;   // perm[new] = old
  // per-lane factor layout: L region (column p of L at lofs[p], c_p values) followed
  // by the DU region (u_pp then U row p at nnz_L + dofs[p], 1 + c_p values)
  std::vector<int32_t> lofs, dofs;  // [n+1]
  std::vector<int32_t> adiag;       // [n] CSR index of A's diagonal (permuted numbering) or -1
  // factor program and solve program (forward records, YEND, backward records, END):
  // record streams packed in chunks
  int32_t f_slots = 0, f_births = 0, f_chunk_words = 0, f_pairs = 0;
  bool fuse_pairs = true;          // input: fuse supernode pivot pairs into one record
  // input: mark the L operands that are structural zeros of A's own (unsymmetric) pattern
  // inside the symmetrised fill (listed last in a fused record): the batch factor skips their rows
  bool skip_dead = true;
  int32_t f_dead_rows = 0;         // rows skipped by the program (of nnz_L)
  int32_t f_dead_l = 0;            // structural-zero multipliers found (with skip_dead)
  // input: factor program of the AUGMENTED matrix [A | b] (column n = one right-hand
  // side, never a pivot): every U row gets u_{p b} = y_p, the forward-substitution
  // result, which the factor kernel writes to X instead of the DU region
  bool aug = false;
  // input: capacity of the pending-slot store per lane (0 = unlimited: one slot per
  // simultaneously pending entry, interval colouring).  With a capacity below the peak
  // pending set, the entries with the furthest next use are spilled to a per-lane global
  // area (SPILL records) and reloaded before their next use (RELOAD records): Belady's
  // rule over the record steps.  f_slots is then cap + 1 (the dummy slot), f_gspill the
  // spill-area entries per lane, f_spills / f_reloads the operation counts per lane.
  int32_t cap = 0;
  // input: every operand a pending slot (operands no update touches are born at their
  // pivot): unconditional slot loads in the kernel (the capacity-planned programs)
  bool all_slots = false;
  int32_t f_gspill = 0, f_spills = 0, f_reloads = 0, f_peak = 0;
  bool plan_ok = true;             // output: the emitted program passed the slot self-check
  int32_t c_scr_need = 0;          // output: scratch rows of the large-pivot path (max c + aug
                                   // over pivots with c > kFusedMax or split steps)
  std::vector<int32_t> f_stream;
  // immediates of the factor stream: word position of each 64-bit cell and its source
  // (>= 0: A index, nnz_A = structural zero, nnz_A + 1 + i: b[i] (original numbering);
  // < 0: d[-1 - src], permuted numbering)
  std::vector<int32_t> f_patch_pos, f_patch_src;
  int32_t y_slots = 0, x_slots = 0, s_chunk_words = 0;
  std::vector<int32_t> s_stream;
  // factor-row chunks of the solve (pairs r0, r1 in consumption order; the first s_nfwd
  // are the forward pass's), at most s_rows rows each
  int32_t s_rows = 16, s_nfwd = 0;
  std::vector<int32_t> s_fchunks;
  int32_t s_bwd_chunk = 0;         // first program chunk of the backward records
};

// Level-scheduled plan of the cooperative small-batch kernels (one CTA per system, the
// lane's whole factor image in shared memory).  Every list is grouped by step (CSR-style
// *_ptr over steps); positions index the per-lane factor image (the V layout: L region,
// then DU region).  A contribution to an entry is scheduled at the running maximum of
// its contributors' etree levels, in ascending pivot order, so each entry still gets its
// updates in the canonical order (bitwise the sequential kernels' results).
struct CoopPlan {
  int32_t steps = 0;                         // etree height
  std::vector<int32_t> birth_src;            // [nnz_LU] CSR index of A (permuted entry) or -1
  std::vector<int32_t> birth_diag;           // [nnz_LU] row p for u_pp entries, else -1
  // factor step A (per step: pivots of that level): l positions / their pivot's diag
  std::vector<int32_t> fa_ptr, fa_l, fa_d;   // [steps+1], [.], [.]
  std::vector<int32_t> fp_ptr, fp_d, fp_p;   // pivots per step: diag position, pivot index
  // factor step B: per step, targets; per target, its contributions (l_pos, u_pos)
  std::vector<int32_t> fb_ptr, fb_t, fb_cptr, fb_l, fb_u;
  // forward: per step, target rows; per target, (l_pos, source row p) ascending p
  std::vector<int32_t> ya_ptr, ya_t, ya_cptr, ya_l, ya_p;
  // backward: per step (roots first), rows; per row, (u_pos, column k) descending k
  std::vector<int32_t> xb_ptr, xb_r, xb_d, xb_cptr, xb_u, xb_k;   // xb_d: u_pp position
  int32_t max_fa = 0, max_fb = 0, max_ya = 0, max_xb = 0;   // largest step (sizes)
};
void build_coop(int32_t n, const std::vector<std::vector<int32_t>>& lcol,
                const std::vector<int32_t>& perm, const int32_t* row_ptr_h,
                const int32_t* col_idx_h, const HostPlan& P, CoopPlan& C);

// Dataflow plan of the fused small-batch factor + solve (psp_dataflow.cu): every factor
// entry, forward row and backward row is a task with its contributions in canonical order;
// tasks sorted by dependency depth and dealt round-robin to the CTA's threads.  Packed
// 16-bit fields (ok = false when positions or counts do not fit).  words: [threads + 1]
// segment offsets, then the records (see psp_dataflow.cu).
struct DataflowPlan {
  bool ok = false;
  int32_t threads = 0, depth = 0, tasks = 0;
  std::vector<uint32_t> words;
};
void build_dataflow(int32_t n, const std::vector<std::vector<int32_t>>& lcol, const HostPlan& P,
                    int32_t threads, DataflowPlan& D);
std::vector<int32_t> transversal_hk(int32_t n, const int32_t* row_ptr, const int32_t* col_idx);
std::vector<int32_t> min_degree_order(int32_t n, const std::vector<std::vector<int32_t>>& adj,
                                      int32_t first);
EtreeResult symbolic_etree(int32_t n, const std::vector<std::vector<int32_t>>& adjp);
std::vector<int32_t> postorder_big_first(int32_t n, const EtreeResult& S);
void build_programs(int32_t n, const std::vector<std::vector<int32_t>>& lcol,
                    const std::vector<int32_t>& perm, const int32_t* row_ptr_h,
                    const int32_t* col_idx_h, HostPlan& P);

}  // namespace psp
