// Host runtime of libpsp: C ABI (include/psp.h), symbolic analysis, device plans.
//
// Symbolic analysis ("a pivot/permutation
// sequence ... computed once, and perpetually reused"): the elimination order, the
// filled pattern of L+U for the symmetric pattern of A+A^T+I, the batch-major slot
// layout and the kernel plans are computed once per sparsity pattern on the host.
// The numeric work of every step of Alg. 1 runs in the CUDA kernels of
// psp_kernels.cu; nothing here touches a lane's values.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "../../include/psp.h"
#include "psp_internal.h"

using psp::DevicePlan;
using psp::kSlab;

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

}  // namespace

struct psp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string detail;

  // --- symbolic ---
  bool analysed = false;
  int32_t n = 0, nnz_A = 0, nnz_LU = 0, nnz_L = 0, n_levels = 0, n_struct_zero_diag = 0;
  int64_t factor_fma = 0, solve_fma = 0;
  int32_t max_live = 0;
  std::vector<int32_t> perm;
  std::vector<DevBuf> plan_bufs;
  DevicePlan plan;

  // --- perturbations ---
  int32_t K = 0, K_pad = 0;
  DevBuf eps_d, dperm_d, V_d, status_d, tol_d;
  bool factored = false;

  // --- solve ---
  int32_t R = 0;
  DevBuf X_d;
  bool solved = false;

  // --- weights ---
  int32_t W = 0;
  DevBuf wptr_d, wlane_d, wval_d, flag_d;
  bool recovered = false;

  // --- host-API staging ---
  DevBuf stageA_d, stageB_d, stageX_d;
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

// ============================================================================
// Ordering: exact minimum degree on the elimination graph (R13).
// ============================================================================
static std::vector<int32_t> min_degree(int32_t n, const std::vector<std::vector<int32_t>>& adj0,
                                       int32_t first) {
  std::vector<std::vector<int32_t>> adj = adj0;  // sorted neighbour lists
  std::vector<char> alive(n, 1);
  std::set<std::pair<int32_t, int32_t>> pq;      // (degree, vertex)
  for (int32_t v = 0; v < n; ++v) pq.insert({(int32_t)adj[v].size(), v});
  std::vector<int32_t> order;
  order.reserve(n);
  std::vector<int32_t> merged;
  auto eliminate = [&](int32_t v) {
    pq.erase({(int32_t)adj[v].size(), v});
    alive[v] = 0;
    order.push_back(v);
    const std::vector<int32_t> nb = adj[v];
    for (int32_t a : nb) {
      pq.erase({(int32_t)adj[a].size(), a});
      // adj[a] <- (adj[a] U nb) \ {a, v}
      merged.clear();
      std::set_union(adj[a].begin(), adj[a].end(), nb.begin(), nb.end(),
                     std::back_inserter(merged));
      merged.erase(std::remove_if(merged.begin(), merged.end(),
                                  [&](int32_t x) { return x == a || x == v; }),
                   merged.end());
      adj[a].swap(merged);
      pq.insert({(int32_t)adj[a].size(), a});
    }
    adj[v].clear();
  };
  if (first >= 0) eliminate(first);
  while (!pq.empty()) eliminate(pq.begin()->second);
  return order;
}

// ============================================================================
// Symbolic factorisation via the elimination tree (Liu) and column merging.
// ============================================================================
struct SymbolicResult {
  std::vector<std::vector<int32_t>> lcol;  // strictly-lower rows of each column (sorted)
  std::vector<int32_t> parent, level;
  int32_t height = 0;
};

static SymbolicResult symbolic_etree(int32_t n, const std::vector<std::vector<int32_t>>& adjp) {
  // adjp: symmetric adjacency in the permuted numbering (no self loops), sorted.
  SymbolicResult S;
  S.parent.assign(n, -1);
  std::vector<int32_t> anc(n, -1);
  for (int32_t j = 0; j < n; ++j)
    for (int32_t i : adjp[j]) {
      if (i >= j) break;
      int32_t r = i;
      while (anc[r] != -1 && anc[r] != j) {
        int32_t t = anc[r];
        anc[r] = j;
        r = t;
      }
      if (anc[r] == -1) {
        anc[r] = j;
        S.parent[r] = j;
      }
    }
  std::vector<std::vector<int32_t>> children(n);
  for (int32_t j = 0; j < n; ++j)
    if (S.parent[j] >= 0) children[S.parent[j]].push_back(j);
  S.lcol.assign(n, {});
  S.level.assign(n, 0);
  std::vector<int32_t> tmp;
  for (int32_t j = 0; j < n; ++j) {
    std::vector<int32_t>& L = S.lcol[j];
    for (int32_t i : adjp[j])
      if (i > j) L.push_back(i);
    for (int32_t c : children[j]) {
      tmp.clear();
      std::set_union(L.begin(), L.end(), S.lcol[c].begin(), S.lcol[c].end(),
                     std::back_inserter(tmp));
      tmp.erase(std::remove(tmp.begin(), tmp.end(), j), tmp.end());
      L.swap(tmp);
      S.level[j] = std::max(S.level[j], S.level[c] + 1);
    }
    S.height = std::max(S.height, S.level[j] + 1);
  }
  return S;
}

static void release_plan(psp_ctx* h) {
  for (auto& b : h->plan_bufs) b.release();
  h->plan_bufs.clear();
  h->plan = DevicePlan{};
}

static void reset_numeric(psp_ctx* h) {
  h->eps_d.release();
  h->dperm_d.release();
  h->V_d.release();
  h->status_d.release();
  h->X_d.release();
  h->wptr_d.release();
  h->wlane_d.release();
  h->wval_d.release();
  h->K = h->K_pad = h->R = h->W = 0;
  h->factored = h->solved = h->recovered = false;
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
  h->stageX_d.release();
  delete h;
  return PSP_OK;
}

psp_status psp_set_stream(psp_handle h, void* cuda_stream) {
  if (!h) return PSP_ERR_ARG;
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  return PSP_OK;
}

psp_status psp_synchronize(psp_handle h) {
  if (!h) return PSP_ERR_ARG;
  if (h->device < 0) return PSP_OK;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
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
    perm = min_degree(n, adj, ordering == PSP_ORDER_MINDEG_FIRST ? first_node : -1);
  }
  std::vector<int32_t> inv(n);
  for (int32_t i = 0; i < n; ++i) inv[perm[i]] = i;

  std::vector<std::vector<int32_t>> adjp(n);
  for (int32_t i = 0; i < n; ++i) {
    for (int32_t j : adj[perm[i]]) adjp[i].push_back(inv[j]);
    std::sort(adjp[i].begin(), adjp[i].end());
  }
  SymbolicResult S = symbolic_etree(n, adjp);

  // U part of column j = { i < j : j in lcol(i) }
  std::vector<std::vector<int32_t>> ucol(n);
  for (int32_t i = 0; i < n; ++i)
    for (int32_t j : S.lcol[i]) ucol[j].push_back(i);  // i ascending => sorted

  // slot layout: column j = [ucol rows][diag][lcol rows]
  std::vector<int32_t> colptr(n + 1, 0), diag_slot(n), col_end(n);
  for (int32_t j = 0; j < n; ++j) {
    diag_slot[j] = colptr[j] + (int32_t)ucol[j].size();
    colptr[j + 1] = diag_slot[j] + 1 + (int32_t)S.lcol[j].size();
    col_end[j] = colptr[j + 1];
  }
  const int64_t nnzLU64 = colptr[n];
  if (nnzLU64 > INT32_MAX / 2) return fail(h, PSP_ERR_ARG, "pattern too large");
  const int32_t nnzLU = (int32_t)nnzLU64;
  auto slot = [&](int32_t i, int32_t j) -> int32_t {
    if (i == j) return diag_slot[j];
    if (i < j) {
      auto& u = ucol[j];
      auto it = std::lower_bound(u.begin(), u.end(), i);
      return colptr[j] + (int32_t)(it - u.begin());
    }
    auto& l = S.lcol[j];
    auto it = std::lower_bound(l.begin(), l.end(), i);
    return diag_slot[j] + 1 + (int32_t)(it - l.begin());
  };

  // A -> slot scatter map
  std::vector<int32_t> a_src(nnzLU, -1);
  for (int32_t r = 0; r < n; ++r)
    for (int32_t q = row_ptr_h[r]; q < row_ptr_h[r + 1]; ++q)
      a_src[slot(inv[r], inv[col_idx_h[q]])] = q;

  // left-looking factor plan
  std::vector<int32_t> col_gptr(n + 1, 0), g_u, g_ptr(1, 0), pr_l, pr_d;
  for (int32_t j = 0; j < n; ++j) {
    for (int32_t p : ucol[j]) {
      g_u.push_back(slot(p, j));
      for (int32_t i : S.lcol[p]) {
        pr_l.push_back(slot(i, p));
        pr_d.push_back(slot(i, j));
      }
      g_ptr.push_back((int32_t)pr_l.size());
    }
    col_gptr[j + 1] = (int32_t)g_u.size();
  }

  // row-oriented solve plans
  std::vector<int32_t> rl_ptr(n + 1, 0), rl_slot, rl_col, ru_ptr(n + 1, 0), ru_slot, ru_col;
  {
    std::vector<std::vector<int32_t>> lrow(n);
    for (int32_t j = 0; j < n; ++j)
      for (int32_t i : S.lcol[j]) lrow[i].push_back(j);  // j ascending
    for (int32_t i = 0; i < n; ++i) {
      for (int32_t j : lrow[i]) {
        rl_slot.push_back(slot(i, j));
        rl_col.push_back(j);
      }
      rl_ptr[i + 1] = (int32_t)rl_slot.size();
      // row i of U = { j > i : j in lcol(i) } (symmetric pattern), j descending
      for (auto it = S.lcol[i].rbegin(); it != S.lcol[i].rend(); ++it) {
        ru_slot.push_back(slot(i, *it));
        ru_col.push_back(*it);
      }
      ru_ptr[i + 1] = (int32_t)ru_slot.size();
    }
  }

  // CSC grouping of A's entries (original numbering) for the deterministic 1-norm
  std::vector<int32_t> acsc_ptr(n + 1, 0), acsc_q(nnzA);
  for (int32_t q = 0; q < nnzA; ++q) acsc_ptr[col_idx_h[q] + 1]++;
  for (int32_t c = 0; c < n; ++c) acsc_ptr[c + 1] += acsc_ptr[c];
  {
    std::vector<int32_t> fillp(acsc_ptr.begin(), acsc_ptr.end() - 1);
    for (int32_t r = 0; r < n; ++r)
      for (int32_t q = row_ptr_h[r]; q < row_ptr_h[r + 1]; ++q) acsc_q[fillp[col_idx_h[q]]++] = q;
  }

  // max simultaneously-live L values in postorder-free natural elimination order:
  // L(:,p) is live from column p until the last column that reads it (max row).
  {
    std::vector<int32_t> delta(n + 1, 0);
    for (int32_t p = 0; p < n; ++p)
      if (!S.lcol[p].empty()) {
        int32_t last = S.lcol[p].back();
        delta[p] += (int32_t)S.lcol[p].size();
        delta[last + 1] -= (int32_t)S.lcol[p].size();
      }
    int32_t cur = 0, mx = 0;
    for (int32_t j = 0; j < n; ++j) {
      cur += delta[j];
      mx = std::max(mx, cur);
    }
    h->max_live = mx;
  }

  DevicePlan P;
  P.n = n;
  P.nnz_A = nnzA;
  P.nnz_LU = nnzLU;
  psp_status s;
#define UP(vec, field) \
  if (!host_only && (s = upload(h, vec, &P.field))) return s;
  UP(a_src, a_src);
  UP(diag_slot, diag_slot);
  UP(col_end, col_end);
  UP(col_gptr, col_gptr);
  UP(g_u, g_u);
  UP(g_ptr, g_ptr);
  UP(pr_l, pr_l);
  UP(pr_d, pr_d);
  UP(rl_ptr, rl_ptr);
  UP(rl_slot, rl_slot);
  UP(rl_col, rl_col);
  UP(ru_ptr, ru_ptr);
  UP(ru_slot, ru_slot);
  UP(ru_col, ru_col);
  UP(perm, perm);
  UP(acsc_ptr, acsc_ptr);
  UP(acsc_q, acsc_q);
#undef UP
  h->plan = P;
  h->perm = perm;
  h->n = n;
  h->nnz_A = nnzA;
  h->nnz_LU = nnzLU;
  int32_t nnzL = 0;
  for (int32_t j = 0; j < n; ++j) nnzL += (int32_t)S.lcol[j].size();
  h->nnz_L = nnzL;
  h->n_levels = S.height;
  h->n_struct_zero_diag = nzd;
  h->factor_fma = (int64_t)pr_l.size();
  h->solve_fma = (int64_t)rl_slot.size() + (int64_t)ru_slot.size();
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
  info->kernel_variant = 0;
  if (perm_h) std::copy(h->perm.begin(), h->perm.end(), perm_h);
  return PSP_OK;
}

psp_status psp_set_perturbations(psp_handle h, int32_t K, const double* eps_h, const double* d_h) {
  if (!h) return PSP_ERR_ARG;
  if (h->device < 0) return fail(h, PSP_ERR_UNSUPPORTED, "host-only handle (device < 0)");
  if (!h->analysed) return fail(h, PSP_ERR_STATE, "psp_symbolic_analyse first");
  if (K < 1 || !eps_h || !d_h) return fail(h, PSP_ERR_ARG, "K >= 1, eps_h and d_h required");
  cudaSetDevice(h->device);
  const int32_t Kp = (K + kSlab - 1) / kSlab * kSlab;
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
  h->K = K;
  h->K_pad = Kp;
  h->factored = h->solved = h->recovered = false;
  return PSP_OK;
}

psp_status psp_factor_batch(psp_handle h, const double* A_vals, double pivot_tol,
                            int32_t* lane_status) {
  if (!h) return PSP_ERR_ARG;
  if (!h->analysed || h->K == 0) return fail(h, PSP_ERR_STATE, "set_perturbations first");
  if (!A_vals) return fail(h, PSP_ERR_ARG, "A_vals required");
  if (!(pivot_tol == pivot_tol)) return fail(h, PSP_ERR_ARG, "pivot_tol is NaN");
  cudaSetDevice(h->device);
  const double* tol_dev = nullptr;
  if (pivot_tol <= 0) {
    CUDA_TRY(h, psp::launch_pivot_tol(h->plan, A_vals, (double*)h->tol_d.p, h->stream));
    tol_dev = (const double*)h->tol_d.p;
  }
  CUDA_TRY(h, psp::launch_factor(h->plan, A_vals, (const double*)h->eps_d.p,
                                 (const double*)h->dperm_d.p, tol_dev, pivot_tol,
                                 (double*)h->V_d.p, (int32_t*)h->status_d.p, h->K, h->K_pad,
                                 h->stream));
  if (lane_status)
    CUDA_TRY(h, cudaMemcpyAsync(lane_status, h->status_d.p, sizeof(int32_t) * h->K,
                                cudaMemcpyDeviceToDevice, h->stream));
  h->factored = true;
  h->solved = h->recovered = false;
  return PSP_OK;
}

psp_status psp_solve_batch(psp_handle h, int32_t R, const double* B, int64_t ldb) {
  if (!h) return PSP_ERR_ARG;
  if (!h->factored) return fail(h, PSP_ERR_STATE, "factor_batch first");
  if (R < 1 || !B || ldb < h->n) return fail(h, PSP_ERR_ARG, "R >= 1, B, ldb >= n required");
  cudaSetDevice(h->device);
  psp_status s;
  size_t need = sizeof(double) * (size_t)h->K_pad * R * h->n;
  if (h->X_d.bytes < need) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if ((s = ensure(h, h->X_d, need))) return s;
  }
  CUDA_TRY(h, psp::launch_solve(h->plan, (const double*)h->V_d.p, B, ldb, R, (double*)h->X_d.p,
                                h->K_pad, h->stream));
  h->R = R;
  h->solved = true;
  return PSP_OK;
}

psp_status psp_get_solutions(psp_handle h, double* X) {
  if (!h || !X) return PSP_ERR_ARG;
  if (!h->solved) return fail(h, PSP_ERR_STATE, "solve_batch first");
  CUDA_TRY(h, psp::launch_gather_solutions(h->plan, h->K, h->R, (const double*)h->X_d.p, X,
                                           h->stream));
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
  h->W = W;
  return PSP_OK;
}

psp_status psp_recover(psp_handle h, double* x) {
  if (!h || !x) return PSP_ERR_ARG;
  if (!h->solved || h->W == 0) return fail(h, PSP_ERR_STATE, "solve_batch and set_weights first");
  CUDA_TRY(h, psp::launch_recover(h->plan, h->W, h->R, (const int32_t*)h->wptr_d.p,
                                  (const int32_t*)h->wlane_d.p, (const double*)h->wval_d.p,
                                  (const double*)h->X_d.p, (const int32_t*)h->status_d.p, x,
                                  (int32_t*)h->flag_d.p, h->stream));
  h->recovered = true;
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
  if ((s = ensure(h, h->stageA_d, sizeof(double) * h->nnz_A))) return s;
  if ((s = ensure(h, h->stageB_d, sizeof(double) * (size_t)h->n * R))) return s;
  if ((s = ensure(h, h->stageX_d, sizeof(double) * (size_t)h->W * R * h->n))) return s;
  CUDA_TRY(h, cudaMemcpyAsync(h->stageA_d.p, A_vals_h, sizeof(double) * h->nnz_A,
                              cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(h->stageB_d.p, B_h, sizeof(double) * (size_t)h->n * R,
                              cudaMemcpyHostToDevice, h->stream));
  if ((s = psp_factor_batch(h, (const double*)h->stageA_d.p, pivot_tol, nullptr))) return s;
  if ((s = psp_solve_batch(h, R, (const double*)h->stageB_d.p, h->n))) return s;
  if ((s = psp_recover(h, (double*)h->stageX_d.p))) return s;
  CUDA_TRY(h, cudaMemcpyAsync(x_h, h->stageX_d.p, sizeof(double) * (size_t)h->W * R * h->n,
                              cudaMemcpyDeviceToHost, h->stream));
  return psp_get_lane_status(h, nullptr);
}

psp_status psp_ladder_weights(int32_t m, const double* s_h, double* eps_out_h, double* w_out_h) {
  if (m < 1 || m > 64 || !s_h || !eps_out_h || !w_out_h) return PSP_ERR_ARG;
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
