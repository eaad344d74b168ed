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
  std::vector<int32_t> blk;    // [n+1] pivot block offsets: [u_pp][L col][U row]
  // factor
  int32_t f_slots = 0, f_births = 0;
  std::vector<int32_t> f_ptr, f_code, f_upd_ptr;
  std::vector<uint16_t> f_upd;
  // forward / backward substitution
  int32_t y_slots = 0, x_slots = 0;
  std::vector<int32_t> y_ptr, y_code, x_ptr, x_code;
};

std::vector<int32_t> min_degree_order(int32_t n, const std::vector<std::vector<int32_t>>& adj,
                                      int32_t first);
EtreeResult symbolic_etree(int32_t n, const std::vector<std::vector<int32_t>>& adjp);
std::vector<int32_t> postorder_big_first(int32_t n, const EtreeResult& S);
void build_programs(int32_t n, const std::vector<std::vector<int32_t>>& lcol,
                    const std::vector<int32_t>& perm, const int32_t* row_ptr_h,
                    const int32_t* col_idx_h, HostPlan& P);

}  // namespace psp
