// Symbolic planning (host, once per sparsity pattern): elimination order, filled
// pattern, pivot-major slot layout, and the interpreted "programs" the CUDA kernels
// walk.  SURVEY §8(a) row a0; PAPER P:L82 (a static pivot sequence "computed once,
// and perpetually reused").
//
// Elimination order (R13): exact minimum degree on the elimination graph
// of pattern(A + A^T) (ties to the lowest original index), then the postorder of its
// elimination tree with the heaviest subtree first.  A postorder is a topological
// order of the etree, so the fill is unchanged; it keeps the set of partially
// updated ("pending") entries small, which is what lets a lane's working set live
// in shared memory.
//
// Factor program (right-looking, canonical order): pivot p (ascending) reads its
// final pivot, L column and U row, writes them to the lane's output block
// [u_pp][l_{i_0 p} .. l_{i_{c-1} p}][u_{p i_0} .. u_{p i_{c-1}}] (i_k = rows of L(:,p),
// ascending), then applies a_ij = fma(-l_ip, u_pj, a_ij) to the c x c block
// {i_a} x {i_b}.  Every entry therefore receives its updates in ascending pivot
// order, exactly as in the dense Gaussian elimination of the oracle.  Entries that
// have been updated but are not yet final live in numbered "pending slots"; an
// entry is born (initialised from A, plus eps*d on the diagonal) right before its
// first update and dies when its pivot consumes it.  Slots are reused greedily
// (interval colouring), so the slot count equals the peak pending set.
#include "psp_plan.h"
#include "psp_internal.h"

#include <algorithm>
#include <array>
#include <climits>
#include <cstdint>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <set>

namespace psp {

// Hopcroft-Karp maximum matching columns -> rows (the structural transversal of P:L304),
// every choice in a fixed order (R20): per phase a BFS from the free columns in
// ascending order (rows of a column ascending) computes layer distances, NIL standing for a
// free row; then a DFS from each free column in ascending order along layered edges (an
// explicit stack in the order the recursive form visits).  q[j] = row matched to column j,
// -1 if none.  O(nnz sqrt(n)).
std::vector<int32_t> transversal_hk(int32_t n, const int32_t* row_ptr, const int32_t* col_idx) {
  std::vector<int32_t> cptr(n + 1, 0), crow(row_ptr[n]);
  for (int32_t q = 0; q < row_ptr[n]; ++q) ++cptr[col_idx[q] + 1];
  for (int32_t j = 0; j < n; ++j) cptr[j + 1] += cptr[j];
  {
    std::vector<int32_t> fill(cptr.begin(), cptr.end() - 1);
    for (int32_t i = 0; i < n; ++i)   // rows ascending within each column
      for (int32_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) crow[fill[col_idx[q]]++] = i;
  }
  const int32_t kInf = INT32_MAX;
  std::vector<int32_t> col_match(n, -1), row_match(n, -1), dist(n), queue;
  std::vector<std::pair<int32_t, int32_t>> stk;   // (column, position in its row list)
  for (;;) {
    queue.clear();
    for (int32_t j = 0; j < n; ++j) {
      if (col_match[j] < 0) {
        dist[j] = 0;
        queue.push_back(j);
      } else {
        dist[j] = kInf;
      }
    }
    int32_t dnil = kInf;
    for (size_t h = 0; h < queue.size(); ++h) {
      const int32_t j = queue[h];
      if (dist[j] >= dnil) continue;
      for (int32_t t = cptr[j]; t < cptr[j + 1]; ++t) {
        const int32_t j2 = row_match[crow[t]];
        if (j2 < 0) {
          if (dnil == kInf) dnil = dist[j] + 1;
        } else if (dist[j2] == kInf) {
          dist[j2] = dist[j] + 1;
          queue.push_back(j2);
        }
      }
    }
    if (dnil == kInf) break;
    for (int32_t j0 = 0; j0 < n; ++j0) {
      if (col_match[j0] >= 0) continue;
      stk.assign(1, {j0, cptr[j0]});
      while (!stk.empty()) {
        auto& top = stk.back();
        const int32_t j = top.first;
        if (top.second == cptr[j + 1]) {   // no augmenting path through j
          dist[j] = kInf;
          stk.pop_back();
          if (!stk.empty()) ++stk.back().second;
          continue;
        }
        const int32_t i = crow[top.second];
        const int32_t j2 = row_match[i];
        if (j2 < 0) {
          if (dnil == dist[j] + 1) {   // augment along the stack
            for (const auto& f : stk) {
              const int32_t r = crow[f.second];
              col_match[f.first] = r;
              row_match[r] = f.first;
            }
            break;
          }
          ++top.second;
        } else if (dist[j2] == dist[j] + 1) {
          stk.push_back({j2, cptr[j2]});
        } else {
          ++top.second;
        }
      }
    }
  }
  return col_match;
}

std::vector<int32_t> min_degree_order(int32_t n, const std::vector<std::vector<int32_t>>& adj0,
                                      int32_t first) {
  std::vector<std::vector<int32_t>> adj = adj0;  // sorted neighbour lists
  std::set<std::pair<int32_t, int32_t>> pq;      // (degree, vertex)
  for (int32_t v = 0; v < n; ++v) pq.insert({(int32_t)adj[v].size(), v});
  std::vector<int32_t> order;
  order.reserve(n);
  std::vector<int32_t> merged;
  auto eliminate = [&](int32_t v) {
    pq.erase({(int32_t)adj[v].size(), v});
    order.push_back(v);
    const std::vector<int32_t> nb = adj[v];
    for (int32_t a : nb) {
      pq.erase({(int32_t)adj[a].size(), a});
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

EtreeResult symbolic_etree(int32_t n, const std::vector<std::vector<int32_t>>& adjp) {
  EtreeResult S;
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

// Heaviest-subtree-first postorder of the etree given by parent[] (children have
// smaller indices).  weight(j) = sum over the subtree of |L(:,k)|^2.
std::vector<int32_t> postorder_big_first(int32_t n, const EtreeResult& S) {
  std::vector<int64_t> w(n);
  for (int32_t j = 0; j < n; ++j) w[j] = (int64_t)S.lcol[j].size() * (int64_t)S.lcol[j].size();
  for (int32_t j = 0; j < n; ++j)
    if (S.parent[j] >= 0) w[S.parent[j]] += w[j];
  std::vector<std::vector<int32_t>> children(n);
  std::vector<int32_t> roots;
  for (int32_t j = 0; j < n; ++j) (S.parent[j] >= 0 ? children[S.parent[j]] : roots).push_back(j);
  auto before = [&](int32_t a, int32_t b) { return w[a] != w[b] ? w[a] > w[b] : a < b; };
  std::sort(roots.begin(), roots.end(), before);
  for (auto& c : children) std::sort(c.begin(), c.end(), before);
  std::vector<int32_t> order;
  order.reserve(n);
  // iterative DFS: (node, next child index)
  std::vector<std::pair<int32_t, size_t>> st;
  for (int32_t r : roots) {
    st.push_back({r, 0});
    while (!st.empty()) {
      auto& top = st.back();
      if (top.second < children[top.first].size()) {
        int32_t c = children[top.first][top.second++];
        st.push_back({c, 0});
      } else {
        order.push_back(top.first);
        st.pop_back();
      }
    }
  }
  return order;
}

namespace {

// Greedy interval colouring: items with [birth, death] in step order; returns the
// slot of each item and the number of slots.  `release_same_step` = a slot whose
// item dies at step s may be reused by an item born at step s.
int32_t colour(int32_t n_steps, const std::vector<int32_t>& birth, const std::vector<int32_t>& death,
               bool release_same_step, std::vector<int32_t>& slot) {
  const int32_t m = (int32_t)birth.size();
  std::vector<std::vector<int32_t>> born(n_steps + 1), dies(n_steps + 1);
  for (int32_t e = 0; e < m; ++e) {
    if (birth[e] < 0) continue;
    born[birth[e]].push_back(e);
    dies[death[e]].push_back(e);
  }
  slot.assign(m, -1);
  std::vector<int32_t> free_list;
  int32_t used = 0;
  for (int32_t s = 0; s < n_steps; ++s) {
    if (release_same_step)
      for (int32_t e : dies[s]) free_list.push_back(slot[e]);
    for (int32_t e : born[s]) {
      if (!free_list.empty()) {
        slot[e] = free_list.back();
        free_list.pop_back();
      } else {
        slot[e] = used++;
      }
    }
    if (!release_same_step)
      for (int32_t e : dies[s]) free_list.push_back(slot[e]);
  }
  return used;
}

// Pack 16-byte-aligned records into fixed-size chunks (the kernels stream chunks
// into a CTA-shared shared-memory ring with bulk async copies).  A record never
// straddles a chunk; the rest of a chunk after its last record starts with the
// sentinel -1 (there are always >= 4 words of it).
void pack_chunks(const std::vector<std::vector<int32_t>>& recs, size_t max_rec,
                 int32_t& chunk_words, std::vector<int32_t>& out,
                 const std::vector<std::vector<std::pair<int32_t, int32_t>>>* patches = nullptr,
                 std::vector<int32_t>* patch_pos = nullptr,
                 std::vector<int32_t>* patch_src = nullptr, size_t break_at = SIZE_MAX,
                 int32_t* break_chunk = nullptr) {
  chunk_words = 512;  // 2 KB
  while ((size_t)chunk_words < max_rec + 4) chunk_words *= 2;
  out.assign(chunk_words, -1);
  size_t base = 0, used = 0;
  for (size_t k = 0; k < recs.size(); ++k) {
    const auto& r = recs[k];
    if (used + r.size() + 4 > (size_t)chunk_words || (k == break_at && used > 0)) {
      base += chunk_words;
      used = 0;
      out.resize(base + chunk_words, -1);
    }
    if (k == break_at && break_chunk) *break_chunk = (int32_t)(base / chunk_words);
    std::copy(r.begin(), r.end(), out.begin() + base + used);
    if (patches)
      for (const auto& pr : (*patches)[k]) {
        patch_pos->push_back((int32_t)(base + used + pr.first));
        patch_src->push_back(pr.second);
      }
    used += r.size();
  }
}

}  // namespace

void build_coop(int32_t n, const std::vector<std::vector<int32_t>>& lcol,
                const std::vector<int32_t>& perm, const int32_t* row_ptr_h,
                const int32_t* col_idx_h, const HostPlan& P, CoopPlan& C) {
  const int32_t nnzL = P.nnz_L, nnzLU = P.nnz_LU;
  // etree levels: a pivot's level exceeds its children's (parent = first row of L(:,p))
  std::vector<int32_t> level(n, 0);
  int32_t nl = 0;
  for (int32_t p = 0; p < n; ++p) {
    if (!lcol[p].empty()) level[lcol[p][0]] = std::max(level[lcol[p][0]], level[p] + 1);
    nl = std::max(nl, level[p] + 1);
  }
  C.steps = nl;
  auto pos_in = [&](int32_t col, int32_t row) -> int32_t {
    const auto& v = lcol[col];
    return (int32_t)(std::lower_bound(v.begin(), v.end(), row) - v.begin());
  };
  auto pos = [&](int32_t i, int32_t j) -> int32_t {   // V-image position of entry (i, j)
    if (i == j) return nnzL + P.dofs[i];
    if (i > j) return P.lofs[j] + pos_in(j, i);
    return nnzL + P.dofs[i] + 1 + pos_in(i, j);
  };
  auto a_index = [&](int32_t i, int32_t j) -> int32_t {
    const int32_t r = perm[i], c = perm[j];
    const int32_t* b = col_idx_h + row_ptr_h[r];
    const int32_t* e = col_idx_h + row_ptr_h[r + 1];
    const int32_t* it = std::lower_bound(b, e, c);
    return (it != e && *it == c) ? (int32_t)(it - col_idx_h) : -1;
  };
  C.birth_src.assign(nnzLU, -1);
  C.birth_diag.assign(nnzLU, -1);
  for (int32_t p = 0; p < n; ++p) {
    C.birth_src[pos(p, p)] = a_index(p, p);
    C.birth_diag[pos(p, p)] = p;
    for (int32_t i : lcol[p]) {
      C.birth_src[pos(i, p)] = a_index(i, p);
      C.birth_src[pos(p, i)] = a_index(p, i);
    }
  }
  // factor A: the L column of every pivot of the step; status over the step's pivots
  std::vector<std::vector<int32_t>> by_level(nl);
  for (int32_t p = 0; p < n; ++p) by_level[level[p]].push_back(p);
  C.fa_ptr.assign(1, 0);
  C.fp_ptr.assign(1, 0);
  for (int32_t l = 0; l < nl; ++l) {
    for (int32_t p : by_level[l]) {
      C.fp_d.push_back(pos(p, p));
      C.fp_p.push_back(p);
      for (size_t k = 0; k < lcol[p].size(); ++k) {
        C.fa_l.push_back(P.lofs[p] + (int32_t)k);
        C.fa_d.push_back(pos(p, p));
      }
    }
    C.fa_ptr.push_back((int32_t)C.fa_l.size());
    C.fp_ptr.push_back((int32_t)C.fp_d.size());
    C.max_fa = std::max(C.max_fa, C.fa_ptr[l + 1] - C.fa_ptr[l]);
  }
  // factor B: contributions per target in ascending pivot order, each at the running
  // maximum of its contributors' levels
  {
    std::vector<std::vector<std::array<int32_t, 3>>> contrib(nnzLU);   // (p, l_pos, u_pos)
    for (int32_t p = 0; p < n; ++p) {
      const auto& L = lcol[p];
      for (size_t a = 0; a < L.size(); ++a)
        for (size_t b = 0; b < L.size(); ++b)
          contrib[pos(L[a], L[b])].push_back(
              {p, P.lofs[p] + (int32_t)a, nnzL + P.dofs[p] + 1 + (int32_t)b});
    }
    // step -> list of (target, [contributions])
    std::vector<std::vector<std::pair<int32_t, std::vector<std::array<int32_t, 3>>>>> st(nl);
    for (int32_t t = 0; t < nnzLU; ++t) {
      auto& cl = contrib[t];
      std::sort(cl.begin(), cl.end());
      int32_t run = 0, cur = -1;
      for (const auto& c : cl) {
        run = std::max(run, level[c[0]]);
        if (run != cur) {
          st[run].push_back({t, {}});
          cur = run;
        }
        st[run].back().second.push_back(c);
      }
    }
    C.fb_ptr.assign(1, 0);
    C.fb_cptr.assign(1, 0);
    for (int32_t l = 0; l < nl; ++l) {
      for (const auto& tc : st[l]) {
        C.fb_t.push_back(tc.first);
        for (const auto& c : tc.second) {
          C.fb_l.push_back(c[1]);
          C.fb_u.push_back(c[2]);
        }
        C.fb_cptr.push_back((int32_t)C.fb_l.size());
      }
      C.fb_ptr.push_back((int32_t)C.fb_t.size());
      C.max_fb = std::max(C.max_fb, C.fb_ptr[l + 1] - C.fb_ptr[l]);
    }
  }
  // forward: y_i <- fma(-l_ip, y_p, y_i), p ascending, at running-max steps
  {
    std::vector<std::vector<std::array<int32_t, 2>>> contrib(n);   // (p, l_pos)
    for (int32_t p = 0; p < n; ++p)
      for (size_t a = 0; a < lcol[p].size(); ++a)
        contrib[lcol[p][a]].push_back({p, P.lofs[p] + (int32_t)a});
    std::vector<std::vector<std::pair<int32_t, std::vector<std::array<int32_t, 2>>>>> st(nl);
    for (int32_t i = 0; i < n; ++i) {
      auto& cl = contrib[i];
      std::sort(cl.begin(), cl.end());
      int32_t run = 0, cur = -1;
      for (const auto& c : cl) {
        run = std::max(run, level[c[0]]);
        if (run != cur) {
          st[run].push_back({i, {}});
          cur = run;
        }
        st[run].back().second.push_back(c);
      }
    }
    C.ya_ptr.assign(1, 0);
    C.ya_cptr.assign(1, 0);
    for (int32_t l = 0; l < nl; ++l) {
      for (const auto& tc : st[l]) {
        C.ya_t.push_back(tc.first);
        for (const auto& c : tc.second) {
          C.ya_l.push_back(c[1]);
          C.ya_p.push_back(c[0]);
        }
        C.ya_cptr.push_back((int32_t)C.ya_l.size());
      }
      C.ya_ptr.push_back((int32_t)C.ya_t.size());
      C.max_ya = std::max(C.max_ya, C.ya_ptr[l + 1] - C.ya_ptr[l]);
    }
  }
  // backward: levels from the roots down; row p: U(p, :) columns descending
  C.xb_ptr.assign(1, 0);
  C.xb_cptr.assign(1, 0);
  for (int32_t l = nl - 1; l >= 0; --l) {
    for (int32_t p : by_level[l]) {
      C.xb_r.push_back(p);
      C.xb_d.push_back(pos(p, p));
      const auto& L = lcol[p];
      for (int32_t k = (int32_t)L.size() - 1; k >= 0; --k) {
        C.xb_u.push_back(nnzL + P.dofs[p] + 1 + k);
        C.xb_k.push_back(L[k]);
      }
      C.xb_cptr.push_back((int32_t)C.xb_u.size());
    }
    C.xb_ptr.push_back((int32_t)C.xb_r.size());
    C.max_xb = std::max(C.max_xb, C.xb_ptr[C.xb_ptr.size() - 1] - C.xb_ptr[C.xb_ptr.size() - 2]);
  }
}

void build_dataflow(int32_t n, const std::vector<std::vector<int32_t>>& lcol, const HostPlan& P,
                    int32_t threads, DataflowPlan& D) {
  D = DataflowPlan{};
  const int32_t nnzL = P.nnz_L, nnzLU = P.nnz_LU;
  if (nnzLU >= 0xffff || n >= 0xffff) return;
  auto pos_in = [&](int32_t col, int32_t row) -> int32_t {
    const auto& v = lcol[col];
    return (int32_t)(std::lower_bound(v.begin(), v.end(), row) - v.begin());
  };
  auto pos = [&](int32_t i, int32_t j) -> int32_t {   // V-image position of entry (i, j)
    if (i == j) return nnzL + P.dofs[i];
    if (i > j) return P.lofs[j] + pos_in(j, i);
    return nnzL + P.dofs[i] + 1 + pos_in(i, j);
  };
  // task ids: factor entry t -> t; forward row i -> nnzLU + i; backward row i -> nnzLU + n + i
  const int32_t nt = nnzLU + 2 * n;
  std::vector<std::vector<std::pair<int32_t, int32_t>>> con(nt);   // (a, b) operand ids
  std::vector<int32_t> entry_i(nnzLU), entry_j(nnzLU);
  for (int32_t p = 0; p < n; ++p) {
    entry_i[pos(p, p)] = entry_j[pos(p, p)] = p;
    for (int32_t i : lcol[p]) {
      entry_i[pos(i, p)] = i; entry_j[pos(i, p)] = p;
      entry_i[pos(p, i)] = p; entry_j[pos(p, i)] = i;
    }
  }
  // factor: entry (a, b) of pivot p's block receives (l_ap, u_pb), p ascending
  for (int32_t p = 0; p < n; ++p) {
    const auto& L = lcol[p];
    for (int32_t a : L)
      for (int32_t b : L) con[pos(a, b)].push_back({pos(a, p), pos(p, b)});
  }
  // forward: y_i receives (l_ip, y_p), p ascending; backward: x_i receives (u_ik, x_k), k descending
  for (int32_t p = 0; p < n; ++p)
    for (int32_t i : lcol[p]) con[nnzLU + i].push_back({pos(i, p), p});
  for (int32_t i = 0; i < n; ++i)
    for (int32_t k = (int32_t)lcol[i].size() - 1; k >= 0; --k) con[nnzLU + n + i].push_back({pos(i, lcol[i][k]), lcol[i][k]});
  // ASAP schedule: the earliest finish time of every task with unit cost per contribution
  // (an operand pair's wait + one fma) and 3 for a division; a contribution starts when
  // the task's previous one is done and both operands are final.  Tasks are then dealt to
  // the threads round-robin in order of their earliest finish, so that every thread walks
  // its tasks in the order an ideal schedule completes them.  (Kinds in id order are topologically ordered: factor
  // entries by their smaller index, diagonals first; forward rows ascending; backward
  // rows descending.)
  std::vector<int32_t> fin(nt, 0), start(nt, 0);
  std::vector<int32_t> order(nnzLU);
  for (int32_t t = 0; t < nnzLU; ++t) order[t] = t;
  std::vector<int32_t> diag_of(nnzLU, -1);
  for (int32_t t = 0; t < nnzLU; ++t)
    if (entry_i[t] > entry_j[t]) diag_of[t] = pos(entry_j[t], entry_j[t]);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    const int32_t ma = std::min(entry_i[a], entry_j[a]), mb = std::min(entry_i[b], entry_j[b]);
    if (ma != mb) return ma < mb;
    return (entry_i[a] == entry_j[a]) > (entry_i[b] == entry_j[b]);
  });
  auto run = [&](int32_t t, int32_t t0, auto&& ready_a, auto&& ready_b) {
    int32_t clk = t0, first = -1;
    for (auto& c : con[t]) {
      clk = std::max({clk, ready_a(c.first), ready_b(c.second)}) + 1;
      if (first < 0) first = clk - 1;
    }
    start[t] = first < 0 ? t0 : first;
    return clk;
  };
  auto fe = [&](int32_t e) { return fin[e]; };
  for (int32_t t : order) {
    int32_t clk = run(t, 0, fe, fe);
    if (diag_of[t] >= 0) clk = std::max(clk, fin[diag_of[t]]) + 3;
    fin[t] = clk;
  }
  auto fy = [&](int32_t i) { return fin[nnzLU + i]; };
  auto fx = [&](int32_t i) { return fin[nnzLU + n + i]; };
  for (int32_t i = 0; i < n; ++i) fin[nnzLU + i] = run(nnzLU + i, 0, fe, fy);
  for (int32_t i = n - 1; i >= 0; --i) {
    const int32_t t = nnzLU + n + i;
    const int32_t clk = run(t, fin[nnzLU + i], fe, fx);
    fin[t] = std::max(clk, fin[pos(i, i)]) + 3;
  }
  std::vector<int32_t> all(nt);
  for (int32_t t = 0; t < nt; ++t) all[t] = t;
  // (by finish time: every dependency finishes strictly earlier, so each thread's list is
  // topologically ordered -- the unfinished task of least finish time can always proceed)
  std::stable_sort(all.begin(), all.end(), [&](int32_t a, int32_t b) {
    return fin[a] != fin[b] ? fin[a] < fin[b] : start[a] < start[b];
  });
  for (auto& c : con)
    if (c.size() >= (1u << 13)) return;
  std::vector<std::vector<uint32_t>> seg(threads);
  for (int32_t r = 0; r < nt; ++r) {
    const int32_t t = all[r];
    auto& w = seg[r % threads];
    const uint32_t cnt = (uint32_t)con[t].size();
    if (t < nnzLU) {   // F: [0 | isdiag << 29 | cnt << 16 | p], [t | diag << 16]
      const bool isd = entry_i[t] == entry_j[t];
      w.push_back((0u << 30) | ((isd ? 1u : 0u) << 29) | (cnt << 16) | (uint32_t)entry_i[t]);
      w.push_back((uint32_t)t | ((diag_of[t] >= 0 ? (uint32_t)diag_of[t] : 0xffffu) << 16));
    } else if (t < nnzLU + n) {   // Y: [1 << 30 | cnt << 16], [i]
      w.push_back((1u << 30) | (cnt << 16));
      w.push_back((uint32_t)(t - nnzLU) | (0xffffu << 16));
    } else {   // X: [2 << 30 | cnt << 16], [i | u_ii position << 16]
      const int32_t i = t - nnzLU - n;
      w.push_back((2u << 30) | (cnt << 16));
      w.push_back((uint32_t)i | ((uint32_t)pos(i, i) << 16));
    }
    for (auto& c : con[t]) w.push_back((uint32_t)c.first | ((uint32_t)c.second << 16));
  }
  D.words.assign(threads + 1, 0);
  for (int32_t th = 0; th < threads; ++th) {
    D.words[th + 1] = D.words[th] + (uint32_t)seg[th].size();
  }
  const uint32_t base = (uint32_t)threads + 1;
  for (int32_t th = 0; th <= threads; ++th) D.words[th] += base;
  for (auto& sgm : seg) D.words.insert(D.words.end(), sgm.begin(), sgm.end());
  while (D.words.size() % 4) D.words.push_back(0);
  D.threads = threads;
  D.tasks = nt;
  D.depth = 0;
  for (int32_t t = 0; t < nt; ++t) D.depth = std::max(D.depth, fin[t]);
  D.ok = true;
}

void build_programs(int32_t n, const std::vector<std::vector<int32_t>>& lcol,
                    const std::vector<int32_t>& perm, const int32_t* row_ptr_h,
                    const int32_t* col_idx_h, HostPlan& P) {
  P.n = n;
  P.perm = perm;
  P.lofs.assign(n + 1, 0);
  P.dofs.assign(n + 1, 0);
  P.c_max = 0;
  int64_t nnzL = 0, ffma = 0;
  for (int32_t p = 0; p < n; ++p) {
    const int32_t c = (int32_t)lcol[p].size();
    P.lofs[p + 1] = P.lofs[p] + c;
    P.dofs[p + 1] = P.dofs[p] + 1 + c;
    P.c_max = std::max(P.c_max, c);
    nnzL += c;
    ffma += (int64_t)c * c;
  }
  P.nnz_LU = P.lofs[n] + P.dofs[n];
  P.nnz_L = (int32_t)nnzL;
  P.factor_fma = ffma;
  P.solve_fma = 2 * nnzL;

  const int32_t nnzA = row_ptr_h[n];
  // A lookup in the permuted numbering: (i, j) -> CSR index of A(perm[i], perm[j]) or -1
  auto a_index = [&](int32_t i, int32_t j) -> int32_t {
    const int32_t r = perm[i], c = perm[j];
    const int32_t* b = col_idx_h + row_ptr_h[r];
    const int32_t* e = col_idx_h + row_ptr_h[r + 1];
    const int32_t* it = std::lower_bound(b, e, c);
    return (it != e && *it == c) ? (int32_t)(it - col_idx_h) : -1;
  };
  // entry ids: diag p -> p; L(i,j) (i>j) -> n + off[j] + pos; U(i,j) (i<j) -> n + nnzL + off[i] + pos
  std::vector<int32_t> off(n + 1, 0);
  for (int32_t p = 0; p < n; ++p) off[p + 1] = off[p] + (int32_t)lcol[p].size();
  // augmented: entry n + 2 nnzL + i = (i, b), the right-hand side column
  const bool aug = P.aug;
  const int32_t n_ent = n + 2 * (int32_t)nnzL + (aug ? n : 0);
  auto entry_b = [&](int32_t i) -> int32_t { return n + 2 * (int32_t)nnzL + i; };
  auto pos_in = [&](int32_t col, int32_t row) -> int32_t {
    const auto& v = lcol[col];
    return (int32_t)(std::lower_bound(v.begin(), v.end(), row) - v.begin());
  };
  auto entry = [&](int32_t i, int32_t j) -> int32_t {
    if (i == j) return i;
    if (i > j) return n + off[j] + pos_in(j, i);
    return n + (int32_t)nnzL + off[i] + pos_in(i, j);
  };

  // ---------------- factor ----------------
  std::vector<int32_t> first(n_ent, -1), death(n_ent, -1);
  for (int32_t p = 0; p < n; ++p) {
    const auto& L = lcol[p];
    for (int32_t a : L)
      for (int32_t b : L) {
        const int32_t e = entry(a, b);
        if (first[e] < 0) {
          first[e] = p;
          death[e] = std::min(a, b);
        }
      }
    if (aug)
      for (int32_t a : L) {
        const int32_t e = entry_b(a);
        if (first[e] < 0) {
          first[e] = p;
          death[e] = a;
        }
      }
  }
  // all_slots (the capacity-planned programs): every operand a pending slot — an entry
  // that no update touches is born (its value of A, + eps*d on the diagonal) at the pivot
  // that consumes it and dies there, so the kernel reads operands with unconditional slot
  // loads (no slot-or-immediate selection).  The arithmetic is the same: the birth's
  // a_ii + (eps*d_i) is the pivot path's a_pp + (eps*d_p).
  if (P.all_slots)
    for (int32_t p = 0; p < n; ++p) {
      auto mk = [&](int32_t e) {
        if (first[e] < 0) {
          first[e] = p;
          death[e] = p;
        }
      };
      mk(entry(p, p));
      for (int32_t a : lcol[p]) {
        mk(entry(a, p));
        mk(entry(p, a));
      }
      if (aug) mk(entry_b(p));
    }
  P.f_births = 0;
  // inverse entry -> (i, j) for births
  std::vector<int32_t> ent_i(n_ent), ent_j(n_ent);
  for (int32_t p = 0; p < n; ++p) {
    ent_i[p] = ent_j[p] = p;
    for (size_t k = 0; k < lcol[p].size(); ++k) {
      const int32_t i = lcol[p][k];
      ent_i[n + off[p] + k] = i;  // L(i, p)
      ent_j[n + off[p] + k] = p;
      ent_i[n + nnzL + off[p] + k] = p;  // U(p, i)
      ent_j[n + nnzL + off[p] + k] = i;
    }
    if (aug) {
      ent_i[entry_b(p)] = p;  // (p, b): j = n marks the right-hand side
      ent_j[entry_b(p)] = n;
    }
  }
  std::vector<std::vector<int32_t>> births_at(n);
  for (int32_t e = 0; e < n_ent; ++e)
    if (first[e] >= 0) births_at[first[e]].push_back(e);
  // Structural liveness under A's own pattern.  The fill above is that of the symmetrised
  // pattern A + A^T (one elimination tree for rows and columns); an entry of it that is
  // absent from A and receives no update l_{i k} u_{k j} with both factors structurally
  // non-zero is exactly +0 in every lane when it is consumed.  For such an L operand
  // a_{i p} the multiplier is l_{i p} = 0 and its whole row update fma(-0, u, x) = x is
  // the identity (as for the entries outside the fill, which no sparse code touches):
  // the row is dead: the capacity-planned fused records list it after the live rows,
  // without its tile row, and the batch factor only stores l = 0.
  std::vector<char> live(n_ent, 1);
  if (P.skip_dead) {
    for (int32_t e = n; e < n + 2 * (int32_t)nnzL; ++e) live[e] = a_index(ent_i[e], ent_j[e]) >= 0;
    for (int32_t p = 0; p < n; ++p) {
      const auto& L = lcol[p];
      for (size_t a = 0; a < L.size(); ++a) {
        if (!live[n + off[p] + a]) continue;            // L(L[a], p)
        for (size_t b = 0; b < L.size(); ++b)
          if (live[n + nnzL + off[p] + b]) live[entry(L[a], L[b])] = 1;   // U(p, L[b])
      }
    }
  }
  P.f_dead_rows = 0;
  P.f_dead_l = 0;
  for (int32_t e = n; e < n + (int32_t)nnzL; ++e) P.f_dead_l += !live[e];
  // Slot-store capacity (HostPlan::cap): the peak pending set of the unlimited plan
  // (interval colouring) decides whether the capacity-planned program is needed.
  std::vector<int32_t> fslot;
  P.f_peak = colour(n, first, death, false, fslot);
  bool capped = P.cap > 0 && P.f_peak > P.cap;
  const int32_t C = P.cap;
  // Per pivot: the pending entries of its update block (targets, + the right-hand side
  // column) and the pending entries it consumes (pivot, L column, U row, y_p).  Disjoint:
  // block entries have both indices > p, consumed ones one index = p.
  auto block_of = [&](int32_t p, std::vector<int32_t>& u) {
    const auto& L = lcol[p];
    for (int32_t a : L) {
      for (int32_t b : L) u.push_back(entry(a, b));
      if (aug) u.push_back(entry_b(a));
    }
  };
  auto consumed_of = [&](int32_t p, std::vector<int32_t>& u) {
    auto add = [&](int32_t e) {
      if (first[e] >= 0) u.push_back(e);
    };
    add(entry(p, p));
    for (int32_t a : lcol[p]) {
      add(entry(a, p));
      add(entry(p, a));
    }
    if (aug) add(entry_b(p));
  };
  auto need_of = [&](int32_t p) {
    std::vector<int32_t> u;
    block_of(p, u);
    consumed_of(p, u);
    return (int32_t)u.size();
  };
  // Supernode pairs: pivot p and q = p + 1 with L(:, p) = {q} u L(:, q) (a fundamental
  // supernode link, q the etree parent of p) share one record: q's update block is the
  // trailing part of p's, so the kernel applies both updates to it with one load/store
  // (in the canonical order: p's, then q's).  Entries first touched at q: none.  With a
  // capacity, only pairs whose step fits it.
  std::vector<char> paired(n, 0);
  P.f_pairs = 0;
  if (P.fuse_pairs)
    for (int32_t p = 0; p + 1 < n; ++p) {
      const auto& Lp = lcol[p];
      const auto& Lq = lcol[p + 1];
      if (Lp.empty() || Lp[0] != p + 1 || (int32_t)Lp.size() + (aug ? 1 : 0) > kPairMax) continue;
      if (Lp.size() != Lq.size() + 1 || !std::equal(Lq.begin(), Lq.end(), Lp.begin() + 1)) continue;
      if (!births_at[p + 1].empty()) continue;
      if (capped && need_of(p) > C) continue;
      paired[p] = 1;
      ++P.f_pairs;
      ++p;   // q is not the first of another pair
    }
  // Steps = the record groups the kernel executes in order: one per pivot or pair.  With
  // a capacity, a pivot whose block + consumed entries exceed it is SPLIT into step A
  // (pivot record: L column and U row read into scratch, consumed entries die) and step B
  // (its births in BIRTH records, then UPDATE records): the large-pivot path.
  // Step B is itself split into row chunks of rpc[p] rows (one step each: the chunk's
  // block rows are all the step needs resident), so a capacity below a whole update block
  // (c x cu entries) stays feasible: a chunk needs rpc x cu slots.
  std::vector<int32_t> stepA(n, -1), stepB(n, -1), rpc(n, 0);
  std::vector<char> split(n, 0);
  int32_t n_steps = 0;
  for (int32_t p = 0; p < n; ++p) {
    split[p] = capped && !paired[p] && need_of(p) > C;
    stepA[p] = n_steps++;
    if (split[p]) {
      const int32_t c = (int32_t)lcol[p].size(), cu = c + (aug ? 1 : 0);
      rpc[p] = std::max<int32_t>(1, std::min<int32_t>(c, C / std::max<int32_t>(1, cu)));
      stepB[p] = n_steps;
      n_steps += (c + rpc[p] - 1) / rpc[p];
    } else {
      stepB[p] = stepA[p];
    }
    if (paired[p]) {
      stepA[p + 1] = stepB[p + 1] = stepA[p];
      ++p;
    }
  }
  // the step of row a of split pivot p's update block
  auto step_row = [&](int32_t p, int32_t a) { return split[p] ? stepB[p] + a / rpc[p] : stepB[p]; };
  // the block entries of rows [a0, a1) of pivot p's update (+ the right-hand side column)
  auto block_rows = [&](int32_t p, int32_t a0, int32_t a1, std::vector<int32_t>& u) {
    const auto& L = lcol[p];
    for (int32_t a = a0; a < a1; ++a) {
      for (int32_t b : L) u.push_back(entry(L[a], b));
      if (aug) u.push_back(entry_b(L[a]));
    }
  };
  P.c_scr_need = 0;
  for (int32_t p = 0; p < n; ++p) {
    const int32_t cu = (int32_t)lcol[p].size() + (aug ? 1 : 0);
    if (split[p] || cu > kFusedMax) P.c_scr_need = std::max(P.c_scr_need, cu);
  }
  // capped: per entry its (from step, slot) residency intervals; spill / reload ops per step
  std::vector<std::vector<std::pair<int32_t, int32_t>>> slot_hist;
  std::vector<std::vector<std::pair<int32_t, int32_t>>> spill_at, reload_at;   // (slot, gidx)
  P.f_gspill = P.f_spills = P.f_reloads = 0;
  if (capped) {
    std::vector<std::vector<int32_t>> uses(n_steps);
    for (int32_t p = 0; p < n; ++p) {
      if (p > 0 && paired[p - 1] && stepA[p] == stepA[p - 1]) continue;   // q of a pair
      consumed_of(p, uses[stepA[p]]);
      if (split[p]) {
        const int32_t c = (int32_t)lcol[p].size();
        for (int32_t a0 = 0; a0 < c; a0 += rpc[p])
          block_rows(p, a0, std::min(c, a0 + rpc[p]), uses[step_row(p, a0)]);
      } else {
        block_of(p, uses[stepB[p]]);
      }
    }
    for (auto& u : uses) {
      std::sort(u.begin(), u.end());
      u.erase(std::unique(u.begin(), u.end()), u.end());
    }
    std::vector<std::vector<int32_t>> use_steps(n_ent);
    for (int32_t st = 0; st < n_steps; ++st)
      for (int32_t e : uses[st]) use_steps[e].push_back(st);
    std::vector<int32_t> where(n_ent, -1), gwhere(n_ent, -1), nxt(n_ent, 0), mark(n_ent, -1);
    slot_hist.assign(n_ent, {});
    spill_at.assign(n_steps, {});
    reload_at.assign(n_steps, {});
    std::vector<int32_t> free_slot, free_g, resident;
    for (int32_t k = C - 1; k >= 0; --k) free_slot.push_back(k);
    int32_t next_g = 0;
    for (int32_t st = 0; st < n_steps && capped; ++st) {
      const auto& N = uses[st];
      for (int32_t e : N) mark[e] = st;
      int32_t need = 0;
      for (int32_t e : N) need += where[e] < 0;
      const int32_t over = (int32_t)resident.size() + need - C;
      if (over > 0) {   // Belady: evict the residents (not used now) with the furthest next use
        std::vector<std::pair<int32_t, int32_t>> cand;   // (-next use, entry)
        for (int32_t e : resident)
          if (mark[e] != st) cand.push_back({-use_steps[e][nxt[e]], e});
        if ((int32_t)cand.size() < over) {   // one step alone needs more than C slots:
          capped = false;                       // no capped plan (unlimited slots instead)
          break;
        }
        std::partial_sort(cand.begin(), cand.begin() + over, cand.end());
        for (int32_t k = 0; k < over; ++k) {
          const int32_t e = cand[k].second;
          int32_t g;
          if (!free_g.empty()) {
            g = free_g.back();
            free_g.pop_back();
          } else {
            g = next_g++;
          }
          spill_at[st].push_back({where[e], g});
          free_slot.push_back(where[e]);
          where[e] = -1;
          gwhere[e] = g;
          ++P.f_spills;
        }
        resident.erase(std::remove_if(resident.begin(), resident.end(),
                                      [&](int32_t e) { return where[e] < 0; }),
                       resident.end());
      }
      for (int32_t e : N) {
        if (where[e] >= 0) continue;
        const int32_t sl = free_slot.back();
        free_slot.pop_back();
        if (gwhere[e] >= 0) {   // spilled: reload before this step
          reload_at[st].push_back({sl, gwhere[e]});
          free_g.push_back(gwhere[e]);
          gwhere[e] = -1;
          ++P.f_reloads;
        }
        where[e] = sl;
        slot_hist[e].push_back({st, sl});
        resident.push_back(e);
      }
      for (int32_t e : N) ++nxt[e];
      bool died = false;
      for (int32_t e : N)
        if (stepA[death[e]] == st) {   // consumed at its death pivot's (first) step
          free_slot.push_back(where[e]);
          where[e] = -1;
          died = true;
        }
      if (died)
        resident.erase(std::remove_if(resident.begin(), resident.end(),
                                      [&](int32_t e) { return where[e] < 0; }),
                       resident.end());
    }
    P.f_gspill = next_g;
  }
  if (capped) {
    P.f_slots = C;
  } else {   // unlimited slots: interval colouring (no split steps are needed then)
    slot_hist.clear();
    spill_at.clear();
    reload_at.clear();
    P.f_gspill = P.f_spills = P.f_reloads = 0;
    P.f_slots = P.f_peak;
    if (P.cap > 0 && P.f_peak > P.cap) P.f_peak = -P.f_peak;   // (capacity infeasible)
    for (int32_t p = 0; p < n; ++p) {
      if (split[p]) {
        split[p] = 0;
        stepB[p] = stepA[p];
      }
    }
  }
  const int32_t dummy_slot = P.f_slots++;   // target of the padding births (never read)
  const int32_t dummy_g = P.f_gspill;       // spill-area entry of the padding spill ops
  if (capped) ++P.f_gspill;
  int32_t cur_step = 0;
  auto slot_of = [&](int32_t e) -> int32_t {
    if (!capped) return fslot[e];
    const auto& hst = slot_hist[e];
    for (int32_t k = (int32_t)hst.size() - 1; k >= 0; --k)
      if (hst[k].first <= cur_step) return hst[k].second;
    return dummy_slot;   // (unreachable: every used entry has a residency at its step)
  };
  // Self-check of the slot plan while the records are emitted, in kernel execution order:
  // slot / spill-entry contents are simulated (births, spills, reloads), and every slot a
  // record reads (operands, update targets) must hold the entry the record means.
  std::vector<int32_t> sim_slot(P.f_slots + 1, -1), sim_g(P.f_gspill + 1, -1);
  std::vector<std::pair<int32_t, int32_t>> checks;   // (slot, entry) read by the current record
  P.plan_ok = true;
  // Factor stream (v4): one record per pivot, 16-byte aligned, packed into fixed-size
  // chunks that the kernel pulls into a CTA-shared ring with bulk async copies.  Values
  // of A and d are IMMEDIATES: 64-bit cells patched into a device copy of the stream
  // before every factorisation (patch list f_patch_pos / f_patch_src below), so the
  // kernel never looks A up.  An OPERAND is 4 words [slot, 0, lo, hi]: the pending slot
  // (slot >= 0) or the immediate (lo, hi) when slot = -1.
  //   PIVOT  [2<<28 | c, p, nbd, nba, flags, ws, d_p (2 words)]
  //          + pivot operand (4 words)
  //          + nbd diagonal births  [slot, 0, a_ii (2), d_i (2), 0, 0]: a_ii + eps*d_i
  //          + nba births           [slot, 0, a_ij (2)] (structural zeros: a_ij = 0);
  //            nba is a multiple of 4 (padding births write a dummy slot never read)
  //            (all-slot programs: births in groups of 4, see put_births)
  //          + c L operands, cu U operands (4 words each; cu = c (+ 1: y_p of [A | b]),
  //            padded to a multiple of 4 with immediate zeros)
  //          + (flags & 2 == 0) c rows x ws target slots of the c x c update block
  //          flags: 1 = the pivot was never updated (add eps*d_p); 2 = c > kFusedMax,
  //          the update comes in UPDATE records; 4 = supernode pair: the record also
  //          carries pivot q = p + 1 (row 0 of the block is q's row, column 0 its column);
  //          bits 8..15 = number of dead rows (l_{i p} a structural zero, below): listed
  //          last among the L operands, without tile rows; L operand word 1 = the row's
  //          position in the stored L column;
  //          ws = row stride (8 * ceil(cu / 8)); padding columns hold the dummy slot
  //   BIRTH  [1<<28, 0, nbd, nba, 0, 0, 0, 0] + births: those of the next pivot that do
  //          not fit its record
  //   UPDATE [3<<28 | c, a0, na, ws, 0, 0, 0, 0] + na rows x ws target slots (rows
  //          a0 .. a0+na-1 of a pivot with c > kFusedMax)
  //   END    [4<<28, ...]
  //   SPILL  [6<<28 | cnt, 0, 0, 0] + cnt x [slot, gidx]: slot -> the lane's spill entry gidx
  //   RELOAD [7<<28 | cnt, 0, 0, 0] + cnt x [slot, gidx]: spill entry gidx -> slot
  //          (capacity-planned programs only; before the BIRTH/PIVOT records of a step:
  //          the evictions that make room for the step, then its reloads)
  // Births of pivot p are the entries first touched by p's update; the pivot's output
  // position (lofs[p], dofs[p]) is implicit: pivots come in order.
  constexpr size_t kMaxRec = 508;   // words: records stay within one 2 KB chunk
  std::vector<std::vector<int32_t>> recs;
  std::vector<std::vector<std::pair<int32_t, int32_t>>> rec_patch;  // (word offset, src)
  size_t max_rec = 0;
  P.f_births = 0;
  auto pad4 = [](std::vector<int32_t>& r) {
    while (r.size() % 4) r.push_back(0);
  };
  auto push = [&](std::vector<int32_t>&& r, std::vector<std::pair<int32_t, int32_t>>&& pt) {
    for (const auto& ck : checks)
      if (ck.first < 0 || ck.first >= (int32_t)sim_slot.size() || sim_slot[ck.first] != ck.second)
        P.plan_ok = false;
    checks.clear();
    pad4(r);
    max_rec = std::max(max_rec, r.size());
    recs.push_back(std::move(r));
    rec_patch.push_back(std::move(pt));
  };
  // immediate cell sources: >= 0 A index (nnz_A = the structural zero), < 0: d[-1 - src]
  auto imm = [](std::vector<int32_t>& r, std::vector<std::pair<int32_t, int32_t>>& pt, int32_t src) {
    pt.push_back({(int32_t)r.size(), src});
    r.push_back(0);
    r.push_back(0);
  };
  // A value (or b_i for j = n) of entry (i, j) as an immediate source
  auto a_src = [&](int32_t i, int32_t j) -> int32_t {
    if (j == n) return nnzA + 1 + perm[i];
    const int32_t q = a_index(i, j);
    return q >= 0 ? q : nnzA;
  };
  auto operand = [&](std::vector<int32_t>& r, std::vector<std::pair<int32_t, int32_t>>& pt,
                     int32_t i, int32_t j) {
    const int32_t e = j == n ? entry_b(i) : entry(i, j);
    if (first[e] >= 0) {
      checks.push_back({slot_of(e), e});
      r.insert(r.end(), {slot_of(e), 0, 0, 0});
    } else {
      r.insert(r.end(), {-1, 0});
      imm(r, pt, a_src(i, j));
    }
  };
  auto birth = [&](std::vector<int32_t>& r, std::vector<std::pair<int32_t, int32_t>>& pt, int32_t e) {
    const int32_t i = ent_i[e], j = ent_j[e];
    r.insert(r.end(), {slot_of(e), 0});
    sim_slot[slot_of(e)] = e;
    imm(r, pt, a_src(i, j));
    if (i == j) {
      imm(r, pt, -1 - i);
      r.insert(r.end(), {0, 0});
    }
    ++P.f_births;
  };
  // Births of d[d0, d1) (diagonal entries) and o[o0, o1) (the others) appended to record r;
  // returns the record's (nbd, nba) counts.  Plain programs: per birth [slot, 0, a (2)
  // (, d_i (2), 0, 0)], nba padded to 4.  All-slot programs (the capacity-planned kernel):
  // groups of 4, [4 slots] + 4 x [a_ii, d_i] (20 words) or 4 x [a] (12 words), both
  // counts padded to 4 (the dummy slot): 5 + 3 instead of 8 + 4 words per birth (the
  // program ring's chunks go further; its waits are a measured cost of this kernel).
  auto ceil4 = [](size_t k) { return (k + 3) & ~(size_t)3; };
  auto birth_words = [&](size_t nd, size_t no) {
    return P.all_slots ? 5 * ceil4(nd) + 3 * ceil4(no) : 8 * nd + 4 * ceil4(no);
  };
  auto put_births = [&](std::vector<int32_t>& r, std::vector<std::pair<int32_t, int32_t>>& pt,
                        const std::vector<int32_t>& d, size_t d0, size_t d1, const std::vector<int32_t>& o,
                        size_t o0, size_t o1) -> std::pair<int32_t, int32_t> {
    if (!P.all_slots) {
      for (size_t k = d0; k < d1; ++k) birth(r, pt, d[k]);
      for (size_t k = o0; k < o1; ++k) birth(r, pt, o[k]);
      for (size_t k = o1 - o0; k < ceil4(o1 - o0); ++k) r.insert(r.end(), {dummy_slot, 0, 0, 0});
      return {(int32_t)(d1 - d0), (int32_t)ceil4(o1 - o0)};
    }
    auto groups = [&](const std::vector<int32_t>& v, size_t b0, size_t b1, bool diag) {
      for (size_t g = b0; g < b1; g += 4) {
        for (size_t k = g; k < g + 4; ++k) r.push_back(k < b1 ? slot_of(v[k]) : dummy_slot);
        for (size_t k = g; k < g + 4; ++k) {
          if (k >= b1) {
            r.insert(r.end(), {0, 0});
            if (diag) r.insert(r.end(), {0, 0});
            continue;
          }
          const int32_t e = v[k], i = ent_i[e], j = ent_j[e];
          sim_slot[slot_of(e)] = e;
          imm(r, pt, a_src(i, j));
          if (diag) imm(r, pt, -1 - i);
          ++P.f_births;
        }
      }
    };
    groups(d, d0, d1, true);
    groups(o, o0, o1, false);
    return {(int32_t)ceil4(d1 - d0), (int32_t)ceil4(o1 - o0)};
  };
  P.adiag.assign(n, -1);
  for (int32_t i = 0; i < n; ++i) P.adiag[i] = a_index(i, i);
  // SPILL / RELOAD  [type<<28 | cnt, 0, 0, 0] + cnt x [slot, gidx] (cnt a multiple of 4:
  // padding ops move the dummy slot to / from the dummy spill entry)
  auto emit_moves = [&](uint32_t type, const std::vector<std::pair<int32_t, int32_t>>& ops) {
    constexpr size_t kPer = (kMaxRec - 4) / 2 / 4 * 4;
    for (size_t o0 = 0; o0 < ops.size(); o0 += kPer) {
      const size_t o1 = std::min(ops.size(), o0 + kPer);
      size_t cnt = o1 - o0;
      const size_t cnt4 = (cnt + 3) & ~(size_t)3;
      std::vector<int32_t> r = {(int32_t)((type << 28) | (uint32_t)cnt4), 0, 0, 0};
      for (size_t o = o0; o < o1; ++o) {
        r.insert(r.end(), {ops[o].first, ops[o].second});
        if (type == kRecSpill) {
          sim_g[ops[o].second] = sim_slot[ops[o].first];
          sim_slot[ops[o].first] = -1;
        } else {
          sim_slot[ops[o].first] = sim_g[ops[o].second];
        }
      }
      for (; cnt < cnt4; ++cnt) r.insert(r.end(), {dummy_slot, dummy_g});
      push(std::move(r), {});
    }
  };
  // births in BIRTH records (those that do not fit a pivot's record, or all of a split
  // pivot's, emitted after its PIVOT record)
  auto birth_records = [&](const std::vector<int32_t>& bd, const std::vector<int32_t>& bo, size_t& qd,
                           size_t& qo, size_t budget) {
    while (budget + birth_words(bd.size() - qd, bo.size() - qo) > kMaxRec &&
           (qd < bd.size() || qo < bo.size())) {
      std::vector<int32_t> b = {(int32_t)(kRecBirth << 28), 0, 0, 0, 0, 0, 0, 0};
      std::vector<std::pair<int32_t, int32_t>> pt;
      size_t nd = 0, no = 0;   // as many as fit one record: diagonal ones first
      while (qd + nd < bd.size() && 8 + birth_words(nd + 1, 0) <= kMaxRec) ++nd;
      while (qo + no < bo.size() && 8 + birth_words(nd, no + 1) <= kMaxRec) ++no;
      const auto cnt = put_births(b, pt, bd, qd, qd + nd, bo, qo, qo + no);
      qd += nd;
      qo += no;
      b[2] = cnt.first;
      b[3] = cnt.second;
      push(std::move(b), std::move(pt));
    }
  };
  for (int32_t p = 0; p < n; ++p) {
    cur_step = stepA[p];
    if (capped) {
      emit_moves(kRecSpill, spill_at[cur_step]);
      emit_moves(kRecReload, reload_at[cur_step]);
    }
    const auto& L = lcol[p];
    const int32_t c = (int32_t)L.size();
    const int32_t cu = c + (aug ? 1 : 0);   // U-row columns (+ the right-hand side)
    const int32_t ws = 8 * ((cu + 7) / 8);
    const bool sp = split[p];
    const bool fused = cu <= kFusedMax && !sp;
    std::vector<int32_t> bd, bo;   // diagonal / other births (entry ids)
    for (int32_t e : births_at[p]) (ent_i[e] == ent_j[e] ? bd : bo).push_back(e);
    const int32_t cu4 = (cu + 3) & ~3;   // U operands padded to a multiple of 4 (immediate 0)
    const size_t fixed = 8 + 4 + 12 + 4 * (size_t)(c + cu4) + (fused ? (size_t)c * ws : 0);
    size_t qd = 0, qo = 0;
    std::vector<int32_t> bdB, boB;   // split pivot: the block's births (step B)
    if (sp) {   // the operands born at p (all_slots) stay in the pivot record (step A)
      auto part = [&](std::vector<int32_t>& v, std::vector<int32_t>& vb) {
        std::vector<int32_t> keep;
        for (int32_t e : v) (death[e] == p ? keep : vb).push_back(e);
        v.swap(keep);
      };
      part(bd, bdB);
      part(bo, boB);
    }
    birth_records(bd, bo, qd, qo, fixed);   // births that do not fit the record go first
    const int32_t e_pp = entry(p, p);
    const int32_t flags = (first[e_pp] < 0 ? 1 : 0) | (fused ? 0 : 2) | (paired[p] ? 4 : 0);
    std::vector<int32_t> r = {(int32_t)((kRecPivot << 28) | (uint32_t)c), p, 0, 0, flags, ws};
    std::vector<std::pair<int32_t, int32_t>> pt;
    imm(r, pt, -1 - p);
    operand(r, pt, p, p);
    {
      const auto cnt = put_births(r, pt, bd, qd, bd.size(), bo, qo, bo.size());
      qd = bd.size();
      qo = bo.size();
      r[2] = cnt.first;
      r[3] = cnt.second;
    }
    // Row order of the record: the stored order (ascending rows), or -- capacity-planned
    // fused records -- the live rows first and the dead rows (see `live` above; a pair's
    // row also needs a dead a_{i q}, and row 0 of a pair, q's own row, stays first) last,
    // without tile rows.  Operand word 1 = the row's position in the stored L column.
    std::vector<int32_t> rord;
    int32_t n_dead = 0;
    {
      std::vector<int32_t> deadr;
      for (int32_t k = 0; k < c; ++k) {
        const bool dead = P.skip_dead && P.all_slots && fused && !live[entry(L[k], p)] &&
                          (!paired[p] || (k > 0 && !live[entry(L[k], p + 1)]));
        (dead ? deadr : rord).push_back(k);
      }
      n_dead = (int32_t)deadr.size();
      rord.insert(rord.end(), deadr.begin(), deadr.end());
      P.f_dead_rows += n_dead;
      r[4] |= n_dead << 8;   // flags bits 8..15: dead rows
    }
    for (int32_t k : rord) {
      operand(r, pt, L[k], p);
      r[r.size() - 3] = k;
    }
    for (int32_t k = 0; k < c; ++k) operand(r, pt, p, L[k]);
    if (aug) operand(r, pt, p, n);   // y_p
    for (int32_t k = cu; k < cu4; ++k)   // (all_slots: the dummy slot, else an immediate 0)
      r.insert(r.end(), {P.all_slots ? dummy_slot : -1, 0, 0, 0});
    auto row = [&](std::vector<int32_t>& out, int32_t a) {
      for (int32_t b = 0; b < ws; ++b)
        if (b < cu) {
          const int32_t e = b < c ? entry(L[a], L[b]) : entry_b(L[a]);
          checks.push_back({slot_of(e), e});
          out.push_back(slot_of(e));
        } else {
          out.push_back(dummy_slot);   // padding columns: the dummy slot (never read)
        }
    };
    if (fused)
      for (int32_t a = 0; a < c - n_dead; ++a) row(r, rord[a]);
    push(std::move(r), std::move(pt));
    if (paired[p]) ++p;   // q's work is in p's record
    if (!fused) {
      const int32_t rows_per = std::max<int32_t>(1, (int32_t)((kMaxRec - 8) / ws));
      auto updates = [&](int32_t r0, int32_t r1) {
        for (int32_t a0 = r0; a0 < r1; a0 += rows_per) {
          const int32_t na = std::min(rows_per, r1 - a0);
          std::vector<int32_t> u = {(int32_t)((kRecUpdate << 28) | (uint32_t)c), a0, na, ws, 0, 0, 0, 0};
          for (int32_t a = a0; a < a0 + na; ++a) row(u, a);
          push(std::move(u), {});
        }
      };
      if (sp) {   // step B, chunk by chunk: make room, reload, the chunk's births, its rows
        // (the block's births by row: entry (L[a], .) belongs to row a)
        std::vector<int32_t> row_of(n + 1, -1);
        for (int32_t a = 0; a < c; ++a) row_of[L[a]] = a;
        for (int32_t r0 = 0; r0 < c; r0 += rpc[p]) {
          const int32_t r1 = std::min(c, r0 + rpc[p]);
          cur_step = step_row(p, r0);
          emit_moves(kRecSpill, spill_at[cur_step]);
          emit_moves(kRecReload, reload_at[cur_step]);
          std::vector<int32_t> cd, co;
          for (int32_t e : bdB)
            if (row_of[ent_i[e]] >= r0 && row_of[ent_i[e]] < r1) cd.push_back(e);
          for (int32_t e : boB)
            if (row_of[ent_i[e]] >= r0 && row_of[ent_i[e]] < r1) co.push_back(e);
          size_t zd = 0, zo = 0;
          birth_records(cd, co, zd, zo, 20);
          if (zd < cd.size() || zo < co.size()) {   // the rest (fits one record)
            std::vector<int32_t> b = {(int32_t)(kRecBirth << 28), 0, 0, 0, 0, 0, 0, 0};
            std::vector<std::pair<int32_t, int32_t>> pt2;
            const auto cnt = put_births(b, pt2, cd, zd, cd.size(), co, zo, co.size());
            zd = cd.size();
            zo = co.size();
            b[2] = cnt.first;
            b[3] = cnt.second;
            push(std::move(b), std::move(pt2));
          }
          updates(r0, r1);
        }
      } else {
        updates(0, c);
      }
    }
  }
  push({(int32_t)(kRecEnd << 28), 0, 0, 0}, {});
  pack_chunks(recs, max_rec, P.f_chunk_words, P.f_stream, &rec_patch, &P.f_patch_pos,
              &P.f_patch_src);

  // ---------------- solve program ----------------
  // Forward substitution (column-oriented, pivots ascending):
  //   YBIRTH [1<<28 | nb, 0, 0, 0] + nb x (slot, original row): pending y_i <- b[row]
  //   YPIVOT [2<<28 | c, ys, lofs, perm[j]] + c target slots: y_j final (slot ys, or
  //          b[perm[j]] if never updated); y_i = fma(-l_ij, y_j, y_i) for the c rows of L(:, j)
  //   YEND   [5<<28, 0, 0, 0]
  // Backward substitution (row-oriented, pivots descending, the sum in descending
  // column order, the division last):
  //   XROW   [3<<28 | c, xs, dofs, i] + c slots of x_{i_k}; xs = slot keeping x_i for
  //          the rows above that need it (or -1)
  //   END    [4<<28, 0, 0, 0]
  std::vector<std::vector<int32_t>> srec;
  size_t smax = 0;
  auto spush = [&](std::vector<int32_t>&& r) {
    while (r.size() % 4) r.push_back(0);
    smax = std::max(smax, r.size());
    srec.push_back(std::move(r));
  };
  {
    std::vector<int32_t> yb(n, -1), yd(n, -1);
    for (int32_t j = 0; j < n; ++j)
      for (int32_t i : lcol[j])
        if (yb[i] < 0) {
          yb[i] = j;
          yd[i] = i;
        }
    std::vector<int32_t> ys;
    P.y_slots = colour(n, yb, yd, false, ys);
    std::vector<std::vector<int32_t>> yborn(n);
    for (int32_t i = 0; i < n; ++i)
      if (yb[i] >= 0) yborn[yb[i]].push_back(i);
    for (int32_t j = 0; j < n; ++j) {
      const auto& bl = yborn[j];
      for (size_t b0 = 0; b0 < bl.size(); b0 += 64) {
        const size_t b1 = std::min(bl.size(), b0 + 64);
        std::vector<int32_t> r = {(int32_t)((kRecBirth << 28) | (uint32_t)(b1 - b0)), 0, 0, 0};
        for (size_t q = b0; q < b1; ++q) {
          r.push_back(ys[bl[q]]);
          r.push_back(perm[bl[q]]);
        }
        spush(std::move(r));
      }
      std::vector<int32_t> r = {(int32_t)((kRecPivot << 28) | (uint32_t)lcol[j].size()),
                                yb[j] >= 0 ? ys[j] : -1, P.lofs[j], perm[j]};
      for (int32_t i : lcol[j]) r.push_back(ys[i]);
      spush(std::move(r));
    }
    spush({(int32_t)(kRecYEnd << 28), 0, 0, 0});
  }
  const size_t bwd_first = srec.size();   // the backward records start a chunk
  {
    // step s = n-1-i; x_i born at the step of i, dies at the step of the smallest q with
    // i in lcol(q)
    std::vector<int32_t> xb(n, -1), xd(n, -1);
    for (int32_t q = 0; q < n; ++q)
      for (int32_t i : lcol[q])
        if (xd[i] < 0 || n - 1 - q > xd[i]) xd[i] = n - 1 - q;
    for (int32_t i = 0; i < n; ++i)
      if (xd[i] >= 0) xb[i] = n - 1 - i;
    std::vector<int32_t> xs;
    P.x_slots = colour(n, xb, xd, true, xs);
    for (int32_t i = n - 1; i >= 0; --i) {
      std::vector<int32_t> r = {(int32_t)((kRecUpdate << 28) | (uint32_t)lcol[i].size()),
                                xb[i] >= 0 ? xs[i] : -1, P.dofs[i], i};
      for (int32_t k : lcol[i]) r.push_back(xs[k]);
      spush(std::move(r));
    }
    spush({(int32_t)(kRecEnd << 28), 0, 0, 0});
  }
  pack_chunks(srec, smax, P.s_chunk_words, P.s_stream, nullptr, nullptr, nullptr, bwd_first,
              &P.s_bwd_chunk);

  // Factor-row chunks of the solve, in consumption order: the L region ascending
  // (forward), then the DU region descending (backward).  A chunk holds <= s_rows rows
  // and never splits the rows one record consumes (a pivot's c rows of L; a row's 1 + c
  // rows of DU), so the kernel checks the ring once per record, not per element.
  P.s_rows = std::min<int32_t>(32, std::max<int32_t>(16, (P.c_max + 2) & ~1));
  if (const char* env = std::getenv("PSP_SOLVE_ROWS"))   // tuning experiments only
    P.s_rows = std::max<int32_t>((P.c_max + 2) & ~1, std::atoi(env));
  P.s_fchunks.clear();
  {
    // (a record longer than s_rows is split across chunks; the kernel then reads it
    // element by element)
    const int32_t S = P.s_rows;
    int32_t r0 = 0, r1 = 0;
    for (int32_t j = 0; j < n; ++j) {
      const int32_t a = P.lofs[j], b = P.lofs[j + 1];
      if (b == a) continue;
      if (b - r0 > S) {
        if (r1 > r0) P.s_fchunks.insert(P.s_fchunks.end(), {r0, r1});
        r0 = a;
        while (b - r0 > S) {
          P.s_fchunks.insert(P.s_fchunks.end(), {r0, r0 + S});
          r0 += S;
        }
      }
      r1 = b;
    }
    if (r1 > r0) P.s_fchunks.insert(P.s_fchunks.end(), {r0, r1});
    P.s_nfwd = (int32_t)P.s_fchunks.size() / 2;
    int32_t hi = P.nnz_LU, lo = P.nnz_LU;
    for (int32_t i = n - 1; i >= 0; --i) {
      const int32_t b0 = P.nnz_L + P.dofs[i];
      if (hi - b0 > S) {
        if (hi > lo) P.s_fchunks.insert(P.s_fchunks.end(), {lo, hi});
        hi = lo;
        while (hi - b0 > S) {
          P.s_fchunks.insert(P.s_fchunks.end(), {hi - S, hi});
          hi -= S;
        }
      }
      lo = b0;
    }
    P.s_fchunks.insert(P.s_fchunks.end(), {lo, hi});
  }
}

}  // namespace psp
