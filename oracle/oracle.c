/*
 * ORACLE (test infrastructure only) — plain, slow, obviously-correct CPU FP64
 * implementation of the perturbation-induced static-pivoting hot path of
 * arXiv 2311.11833 (PAPER.md, "Towards Perturbation-Induced Static Pivoting on
 * GPU-Based Linear Solvers").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference leg
 * may load this library.  It shares no code, header, table or generator with the
 * CUDA path in paper_2311_11833_b200/ and includes nothing from it.
 *
 * Floating-point conventions (reading R12): IEEE binary64, round to
 * nearest; every multiply-add that the algorithm states as "a - l*u" is ONE fused
 * fma(-l, u, a); divisions are true divisions; compiled with -ffp-contract=off so
 * that no other contraction happens.  Update order (R11): each entry's updates are
 * applied in ascending pivot order p (Gaussian elimination as written), forward
 * substitution ascending j, backward substitution descending j with the division
 * last, combination ascending k.
 *
 * Status convention: 0 = ok, else 1 + first (permuted) pivot position p with
 * |u_pp| <= tol or u_pp non-finite (SPEC S:L46 ZeroPivot{row}; PAPER P:L304 the
 * NaN/Inf failure mode, reported instead of propagated).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

/* ------------------------------------------------------------------------- */
/* OR1: dense pivot-free Gaussian elimination (PAPER §II-C: "Gaussian
 * elimination ... sequentially dividing rows of a matrix by a leading diagonal
 * entrant"; no row exchanges = static pivoting).  A is n x n row-major and is
 * overwritten by L (strict lower, unit diagonal implied) and U (upper).
 * Returns 0 or 1 + first failing pivot position.                              */
int oracle_lu_nopivot(int n, double* A, double tol) {
  for (int p = 0; p < n; ++p) {
    double piv = A[(size_t)p * n + p];
    if (!(fabs(piv) > tol) || !isfinite(piv)) return p + 1;
    for (int i = p + 1; i < n; ++i) {
      double l = A[(size_t)i * n + p] / piv;
      A[(size_t)i * n + p] = l;
      for (int j = p + 1; j < n; ++j)
        A[(size_t)i * n + j] = fma(-l, A[(size_t)p * n + j], A[(size_t)i * n + j]);
    }
  }
  return 0;
}

/* Forward (unit L, ascending j) then backward (U, descending j) substitution on
 * one right-hand side y (overwritten by x).  Alg. 1 step 2, the
 * trsm pair of P:L310.                                                          */
void oracle_lu_solve(int n, const double* LU, double* y) {
  for (int j = 0; j < n; ++j)
    for (int i = j + 1; i < n; ++i) y[i] = fma(-LU[(size_t)i * n + j], y[j], y[i]);
  for (int j = n - 1; j >= 0; --j) {
    y[j] = y[j] / LU[(size_t)j * n + j];
    for (int i = 0; i < j; ++i) y[i] = fma(-LU[(size_t)i * n + j], y[j], y[i]);
  }
}

/* Partial-pivot GE (SPEC S:L52-59 lu_partial_pivot: the reference solution x*
 * = A^{-1} b of P:L89).  piv[p] = row swapped into position p.  Returns 0 or
 * 1 + column with an exactly zero pivot.                                        */
int oracle_lu_partial_pivot(int n, double* A, int* piv) {
  for (int p = 0; p < n; ++p) {
    int r = p;
    double best = fabs(A[(size_t)p * n + p]);
    for (int i = p + 1; i < n; ++i) {
      double v = fabs(A[(size_t)i * n + p]);
      if (v > best) { best = v; r = i; }
    }
    piv[p] = r;
    if (best == 0.0) return p + 1;
    if (r != p)
      for (int j = 0; j < n; ++j) {
        double t = A[(size_t)p * n + j];
        A[(size_t)p * n + j] = A[(size_t)r * n + j];
        A[(size_t)r * n + j] = t;
      }
    double pv = A[(size_t)p * n + p];
    for (int i = p + 1; i < n; ++i) {
      double l = A[(size_t)i * n + p] / pv;
      A[(size_t)i * n + p] = l;
      for (int j = p + 1; j < n; ++j)
        A[(size_t)i * n + j] = fma(-l, A[(size_t)p * n + j], A[(size_t)i * n + j]);
    }
  }
  return 0;
}

void oracle_lu_pp_solve(int n, const double* LU, const int* piv, double* y) {
  for (int p = 0; p < n; ++p)
    if (piv[p] != p) { double t = y[p]; y[p] = y[piv[p]]; y[piv[p]] = t; }
  oracle_lu_solve(n, LU, y);
}

/* Dense A from CSR (duplicates summed). */
static void csr_to_dense(int n, const int32_t* rp, const int32_t* ci, const double* v, double* A) {
  memset(A, 0, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int q = rp[i]; q < rp[i + 1]; ++q) A[(size_t)i * n + ci[q]] += v[q];
}

/* One perturbed lane of Alg. 1: A_k = P (A + eps_k D) P^T formed
 * densely (Eqs. (5)-(6), D = diag(d)), pivot-free LU, then R solves.
 * perm[new] = old (the elimination order); B is n x R column-major in the
 * ORIGINAL ordering; X receives R x n (row r = solution r, original ordering).   */
int oracle_dense_lane(int n, const int32_t* rp, const int32_t* ci, const double* v,
                      const int32_t* perm, const double* d, double eps, int R,
                      const double* B, double tol, double* X) {
  double* A = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* Ak = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  csr_to_dense(n, rp, ci, v, A);
  for (int i = 0; i < n; ++i) A[(size_t)i * n + i] = A[(size_t)i * n + i] + eps * d[i];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Ak[(size_t)i * n + j] = A[(size_t)perm[i] * n + perm[j]];
  int st = oracle_lu_nopivot(n, Ak, tol);
  for (int r = 0; r < R; ++r) {
    if (st) {
      for (int i = 0; i < n; ++i) X[(size_t)r * n + i] = NAN;
      continue;
    }
    for (int i = 0; i < n; ++i) y[i] = B[(size_t)r * n + perm[i]];
    oracle_lu_solve(n, Ak, y);
    for (int i = 0; i < n; ++i) X[(size_t)r * n + perm[i]] = y[i];
  }
  free(A); free(Ak); free(y);
  return st;
}

/* Alg. 1 steps 1-2 over a batch of K lanes (independent; OpenMP over lanes).
 * X is K x R x n.                                                               */
void oracle_dense_batch(int n, const int32_t* rp, const int32_t* ci, const double* v,
                        const int32_t* perm, const double* d, int K, const double* eps,
                        int R, const double* B, double tol, double* X, int32_t* status) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int k = 0; k < K; ++k)
    status[k] = oracle_dense_lane(n, rp, ci, v, perm, d, eps[k], R, B, tol,
                                  X + (size_t)k * R * n);
}

/* Reference solve x* = A^{-1} b by partial-pivot GE (unperturbed A).            */
int oracle_reference_solve(int n, const int32_t* rp, const int32_t* ci, const double* v,
                           int R, const double* B, double* X) {
  double* A = (double*)malloc(sizeof(double) * (size_t)n * n);
  int* piv = (int*)malloc(sizeof(int) * (size_t)n);
  csr_to_dense(n, rp, ci, v, A);
  int st = oracle_lu_partial_pivot(n, A, piv);
  for (int r = 0; r < R; ++r) {
    for (int i = 0; i < n; ++i) X[(size_t)r * n + i] = B[(size_t)r * n + i];
    if (!st) oracle_lu_pp_solve(n, A, piv, X + (size_t)r * n);
  }
  free(A); free(piv);
  return st;
}

/* ------------------------------------------------------------------------- */
/* OR2: sparse left-looking pivot-free LU on a given filled pattern (the same
 * Gaussian elimination; for entry (i,j) the updates from pivots p are applied in
 * ascending p, so it is bitwise equal to OR1 whenever all values are finite).
 * Used where dense O(n^3) is infeasible.  Inputs, all in the PERMUTED ordering:
 *   acp/ari/av : CSC of P A P^T (no duplicates)
 *   fcp/fri    : CSC of the filled pattern of L+U (rows ascending, diagonal incl.)
 *   dp         : permuted d
 * Output LU values in fv (aligned with fri).                                    */
int oracle_sparse_lu(int n, const int32_t* acp, const int32_t* ari, const double* av,
                     const int32_t* fcp, const int32_t* fri, const double* dp, double eps,
                     double tol, double* fv) {
  double* w = (double*)calloc((size_t)n, sizeof(double));
  int32_t* diag = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int st = 0;
  for (int j = 0; j < n; ++j) {
    diag[j] = -1;
    for (int q = fcp[j]; q < fcp[j + 1]; ++q) if (fri[q] == j) diag[j] = q;
  }
  for (int j = 0; j < n && !st; ++j) {
    for (int q = fcp[j]; q < fcp[j + 1]; ++q) w[fri[q]] = 0.0;
    for (int q = acp[j]; q < acp[j + 1]; ++q) w[ari[q]] = w[ari[q]] + av[q];
    w[j] = w[j] + eps * dp[j];
    for (int q = fcp[j]; q < fcp[j + 1]; ++q) {
      int p = fri[q];
      if (p >= j) break;
      double u = w[p];
      for (int t = diag[p] + 1; t < fcp[p + 1]; ++t) w[fri[t]] = fma(-fv[t], u, w[fri[t]]);
    }
    double piv = w[j];
    if (!(fabs(piv) > tol) || !isfinite(piv)) st = j + 1;
    for (int q = fcp[j]; q < fcp[j + 1]; ++q) {
      int i = fri[q];
      fv[q] = (i > j) ? w[i] / piv : w[i];
    }
  }
  free(w); free(diag);
  return st;
}

/* Sparse forward/backward substitution on the filled CSC factor; b and x in the
 * original ordering (perm[new] = old).                                          */
void oracle_sparse_solve(int n, const int32_t* fcp, const int32_t* fri, const double* fv,
                         const int32_t* perm, const double* b, double* x) {
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
  for (int j = 0; j < n; ++j)
    for (int q = fcp[j]; q < fcp[j + 1]; ++q)
      if (fri[q] > j) y[fri[q]] = fma(-fv[q], y[j], y[fri[q]]);
  for (int j = n - 1; j >= 0; --j) {
    double ujj = 0.0;
    for (int q = fcp[j]; q < fcp[j + 1]; ++q) if (fri[q] == j) ujj = fv[q];
    y[j] = y[j] / ujj;
    for (int q = fcp[j + 1] - 1; q >= fcp[j]; --q)   /* order irrelevant: distinct y_i */
      if (fri[q] < j) y[fri[q]] = fma(-fv[q], y[j], y[fri[q]]);
  }
  for (int i = 0; i < n; ++i) x[perm[i]] = y[i];
  free(y);
}

void oracle_sparse_batch(int n, const int32_t* acp, const int32_t* ari, const double* av,
                         const int32_t* fcp, const int32_t* fri, const double* dp,
                         const int32_t* perm, int K, const double* eps, int R,
                         const double* B, double tol, double* X, int32_t* status) {
  int nnzf = fcp[n];
#pragma omp parallel for schedule(dynamic, 1)
  for (int k = 0; k < K; ++k) {
    double* fv = (double*)malloc(sizeof(double) * (size_t)(nnzf > 0 ? nnzf : 1));
    int st = oracle_sparse_lu(n, acp, ari, av, fcp, fri, dp, eps[k], tol, fv);
    status[k] = st;
    for (int r = 0; r < R; ++r) {
      double* xo = X + ((size_t)k * R + r) * n;
      if (st) { for (int i = 0; i < n; ++i) xo[i] = NAN; continue; }
      oracle_sparse_solve(n, fcp, fri, fv, perm, B + (size_t)r * n, xo);
    }
    free(fv);
  }
}

/* ------------------------------------------------------------------------- */
/* Alg. 1 steps 3-4 / Eq. (13)-(14):
 * x_hat[w] = sum_k weights[w][k] * x_k, ascending k, one fma per term.  The pair
 * average of Eq. (avg_hats) is folded into the weights (w = beta_j / 2 per sign). */
void oracle_combine(int K, int R, int n, int W, const double* weights, const double* X,
                    double* out) {
  for (int w = 0; w < W; ++w)
    for (int r = 0; r < R; ++r)
      for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int k = 0; k < K; ++k) {
          double c = weights[(size_t)w * K + k];
          if (c != 0.0) acc = fma(c, X[((size_t)k * R + r) * n + i], acc);
        }
        out[((size_t)w * R + r) * n + i] = acc;
      }
}

/* ------------------------------------------------------------------------- */
/* Iterative-refinement baseline ("compared with
 * existing iterative refinement-based approaches"): the residual of one iterate,
 * r = b - A x, row by row over the CSR entries in order, one fma per term:
 * r_i = b_i; for q: r_i = fma(-a_iq, x_{col q}, r_i).                            */
void oracle_residual_fma(int n, const int32_t* rp, const int32_t* ci, const double* v,
                         const double* x, const double* b, double* r) {
  for (int i = 0; i < n; ++i) {
    double acc = b[i];
    for (int q = rp[i]; q < rp[i + 1]; ++q) acc = fma(-v[q], x[ci[q]], acc);
    r[i] = acc;
  }
}
