// Host emulator of the factor program (debugging aid, test infrastructure only):
// interprets the record stream of psp_plan.cpp for one lane with the G-group split of
// factor_kernel, groups run one after another inside each record.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>
#include "../../paper_2311_11833_b200/csrc/psp_plan.h"
#include "../../paper_2311_11833_b200/csrc/psp_internal.h"
using namespace psp;
extern "C" int emu_factor(int n, const int* rp, const int* ci, const double* A, const int* perm_in,
                          double eps, const double* d_orig, int G, double* out, int* nnzlu) {
  std::vector<int> perm(perm_in, perm_in + n), inv(n);
  for (int i = 0; i < n; ++i) inv[perm[i]] = i;
  std::vector<std::vector<int>> adjp(n);
  for (int r = 0; r < n; ++r)
    for (int q = rp[r]; q < rp[r + 1]; ++q) {
      int c = ci[q];
      if (c == r) continue;
      adjp[inv[r]].push_back(inv[c]);
      adjp[inv[c]].push_back(inv[r]);
    }
  for (auto& a : adjp) { std::sort(a.begin(), a.end()); a.erase(std::unique(a.begin(), a.end()), a.end()); }
  EtreeResult S = symbolic_etree(n, adjp);
  HostPlan P;
  build_programs(n, S.lcol, perm, rp, ci, P);
  *nnzlu = P.nnz_LU;
  std::vector<double> dperm(n);
  for (int i = 0; i < n; ++i) dperm[i] = d_orig[perm[i]];
  std::vector<double> pend(P.f_slots, NAN), sl(P.c_max), su(P.c_max);
  const int32_t* w = P.f_stream.data();
  size_t pos = 0;
  int lo = 0, dd = 0;
  double* du = out + P.nnz_L;
  auto src = [&](int code) { return code >= 0 ? pend[code] : (code == kZero ? 0.0 : A[-1 - code]); };
  for (;;) {
    if (w[pos] == -1) { pos = (pos / P.f_chunk_words + 1) * P.f_chunk_words; continue; }
    const int32_t* r = w + pos;
    uint32_t h0 = (uint32_t)r[0], type = h0 >> 28;
    if (type == kRecBirth) {
      int nb = h0 & 0xffff;
      for (int g = 0; g < G; ++g)
        for (int b = g; b < nb; b += G) {
          int x = r[4 + 2 * b], y = r[5 + 2 * b];
          uint32_t slot = (uint32_t)x & 0x7fffffffu;
          double v;
          if (x < 0) { int q = P.adiag[y]; v = (q >= 0 ? A[q] : 0.0) + eps * dperm[y]; }
          else v = y >= 0 ? A[y] : 0.0;
          pend[slot] = v;
        }
      pos += (4 + 2 * nb + 3) & ~3;
    } else if (type == kRecPivot) {
      int c = h0 & 0xffff, ps = r[1], piv = r[2];
      double pv = ps >= 0 ? pend[ps] : ((ps == kZero ? 0.0 : A[-1 - ps]) + eps * dperm[piv]);
      du[dd] = pv;
      for (int k = 0; k < c; ++k) { sl[k] = src(r[4 + k]) / pv; out[lo + k] = sl[k]; }
      for (int k = 0; k < c; ++k) { su[k] = src(r[4 + c + k]); du[dd + 1 + k] = su[k]; }
      lo += c; dd += 1 + c;
      pos += (4 + 2 * c + 3) & ~3;
    } else if (type == kRecUpdate) {
      int wdt = h0 & 0xff, a0 = r[1], na = r[2], j0 = r[3];
      for (int g = 0; g < G; ++g)
        for (int a = g; a < na; a += G)
          for (int b = 0; b < wdt; ++b) {
            int s = r[4 + 8 * a + b];
            pend[s] = std::fma(-sl[a0 + a], su[j0 + b], pend[s]);
          }
      pos += 4 + 8 * na;
    } else break;
  }
  return 0;
}
