// Host build of dense.h / recycle.h (one "thread") for CPU unit tests of the
// device dense kernel's numerics (tests/test_dense_host.py). Not a product
// path: the solver only ever runs these routines inside k_dense on the GPU.
#include <cstdlib>
#include <cstring>
#include <vector>

#include "recycle.h"

using namespace skrd;

namespace {
struct HostArena {
  std::vector<double> d;
  std::vector<int> i;
  Arena a;
  HostArena() : d(arena_doubles(1, LDD), 0.0), i(arena_ints(LDD), 0) {
    a = make_arena(d.data(), i.data(), 1, LDD);
  }
};
}  // namespace

extern "C" {

int skrh_eig(const double* A, int lda, int n, double* wr, double* wi) {
  if (n < 1 || n > DMAX) return -1;
  HostArena h;
  Ctx c = ctx();
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) DA(h.a.M1, LDD, i, j) = DA(A, lda, i, j);
  return eig_schur(c, h.a.M1, LDD, n, h.a.M3, LDD, wr, wi, h.a.vec + 2 * LDD, h.a.M2,
                   LDD * LDD / ZREC);
}

// eigen-decomposition with the selection: returns ncols, P (n x ncols) NOT
// orthonormalised (raw [Re v, Im v] columns) for direct span tests.
int skrh_select(const double* A, int lda, int n, int k, int max_cols, double* P, int ldp,
                double* wr, double* wi) {
  HostArena h;
  Ctx c = ctx();
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) DA(h.a.M1, LDD, i, j) = DA(A, lda, i, j);
  if (eig_schur(c, h.a.M1, LDD, n, h.a.M3, LDD, wr, wi, h.a.vec + 2 * LDD, h.a.M2,
                   LDD * LDD / ZREC) != 0)
    return -2;
  int nc = select_basis(c, h.a.M1, LDD, n, h.a.M3, LDD, wr, wi, k, max_cols, h.a.M4, LDD,
                        h.a.iw + LDD, h.a.xwork, h.a.red);
  for (int j = 0; j < nc; ++j)
    for (int i = 0; i < n; ++i) DA(P, ldp, i, j) = DA(h.a.M4, LDD, i, j);
  return nc;
}

int skrh_qrcp(const double* A, int lda, int m, int n, double rtol, double* Q, int ldq, double* R,
              int ldr, int* jpvt) {
  HostArena h;
  Ctx c = ctx();
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) DA(h.a.M1, LDD, i, j) = DA(A, lda, i, j);
  double tau[LDD];
  int r = qrcp(c, h.a.M1, LDD, m, n, jpvt, h.a.M2, LDD, rtol, h.a.vec, tau);
  for (int j = 0; j < r; ++j)
    for (int i = 0; i < m; ++i) DA(Q, ldq, i, j) = DA(h.a.M2, LDD, i, j);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < (m < n ? m : n); ++i) DA(R, ldr, i, j) = (i <= j) ? DA(h.a.M1, LDD, i, j) : 0.0;
  return r;
}

int skrh_hr_first(const double* H, int ldh, int m, int k, double* P, int ldp, int* warn) {
  HostArena h;
  Ctx c = ctx();
  int r = hr_first(c, h.a, H, ldh, m, k, warn);
  for (int j = 0; j < r; ++j)
    for (int i = 0; i < m; ++i) DA(P, ldp, i, j) = DA(h.a.M2, LDD, i, j);
  return r;
}

int skrh_hr_next(const double* G, int ldg, const double* cross, int ldx, int mm, int k, double* P,
                 int ldp, int* warn) {
  HostArena h;
  Ctx c = ctx();
  for (int j = 0; j < mm; ++j)
    for (int i = 0; i <= mm; ++i) DA(h.a.G, LDD, i, j) = DA(G, ldg, i, j);
  int r = hr_next(c, h.a, mm, cross, ldx, k, warn);
  for (int j = 0; j < r; ++j)
    for (int i = 0; i < mm; ++i) DA(P, ldp, i, j) = DA(h.a.M2, LDD, i, j);
  return r;
}

int skrh_recycle_first(const double* H, int ldh, int j, int k, double* coefU, int ldu,
                       double* coefC, int ldcc, int* warn) {
  HostArena h;
  Ctx c = ctx();
  return recycle_first(c, h.a, H, ldh, j, k, coefU, ldu, coefC, ldcc, warn);
}

int skrh_recycle_next(const double* H, int ldh, const double* B, int ldb, const double* dk, int kc,
                      int j, const double* cross, int ldx, int k, double* coefU, int ldu,
                      double* coefC, int ldcc, int* warn) {
  HostArena h;
  Ctx c = ctx();
  return recycle_next(c, h.a, H, ldh, B, ldb, dk, kc, j, cross, ldx, k, coefU, ldu, coefC, ldcc,
                      warn);
}

// CholQR2 on a host tall matrix X (n x k, ld): returns r2 and writes
// Q = X T (n x r2) into Q, kept pivots and Rinv.
int skrh_cholqr2(const double* X, int ldx, int n, int k, double* Q, int ldq, int* kept) {
  HostArena h;
  Ctx c = ctx();
  std::vector<double> G(LDD * LDD), T1(LDD * LDD), R1(LDD * LDD), X1((size_t)n * k), G2(LDD * LDD),
      T2(LDD * LDD), Rinv(LDD * LDD);
  for (int a = 0; a < k; ++a)
    for (int b = 0; b < k; ++b) {
      double s = 0.0;
      for (int r = 0; r < n; ++r) s += X[r + (size_t)a * ldx] * X[r + (size_t)b * ldx];
      G[a + b * LDD] = s;
    }
  int r = cholqr_pass1(c, h.a, G.data(), LDD, k, T1.data(), LDD, R1.data(), LDD);
  if (r <= 0) return 0;
  for (int q = 0; q < r; ++q)
    for (int row = 0; row < n; ++row) {
      double s = 0.0;
      for (int a = 0; a < k; ++a) s += X[row + (size_t)a * ldx] * T1[a + q * LDD];
      X1[row + (size_t)q * n] = s;
    }
  for (int a = 0; a < r; ++a)
    for (int b = 0; b < r; ++b) {
      double s = 0.0;
      for (int row = 0; row < n; ++row) s += X1[row + (size_t)a * n] * X1[row + (size_t)b * n];
      G2[a + b * LDD] = s;
    }
  int r2 = cholqr_pass2(c, h.a, G2.data(), LDD, r, R1.data(), LDD, k, T2.data(), LDD, kept,
                        Rinv.data(), LDD);
  for (int q = 0; q < r2; ++q)
    for (int row = 0; row < n; ++row) {
      double s = 0.0;
      for (int a = 0; a < r; ++a) s += X1[row + (size_t)a * n] * T2[a + q * LDD];
      Q[row + (size_t)q * ldq] = s;
    }
  return r2;
}

}  // extern "C"
