// Recycle-space "programs" run by the single-CTA dense kernel (and, for unit
// tests, on the host): harmonic-Ritz recycle updates and the tall-skinny QR
// steps of the between-system refresh. Built on dense.h.
//
// Reference steps restated (kryrec/gcrodr.py):
//   first cycle  _first_cycle_recycle           gcrodr.py:280-292
//   later cycles recycle update in gcrodr_solve  gcrodr.py:444-460
//   refresh      refresh_recycle                gcrodr.py:80-113 (via CholQR2 + QRCP(R))
//
// The tall (N-row) products are NOT done here: these programs emit small
// coefficient matrices that the row-parallel combine kernel applies
// (U_new = [U | V] coefU, C_new = [C | V] coefC), so the span algebra is
// identical to the reference while every N-length pass stays one HBM sweep.
#pragma once
#include "dense.h"

namespace skrd {

struct Arena {
  int ld;      // leading dimension of the matrices (odd, >= m + 1; <= LDD)
  double* G;   // ld x ld
  double* M1;  // ld x ld
  double* M2;  // ld x ld
  double* M3;  // ld x ld (M3, M4 adjacent: hr_next solves 2 mm right-hand sides)
  double* M4;  // ld x ld
  double* vec;    // 12 * ld
  double* xwork;  // nw * 3 * DMAX
  double* red;    // 64
  int* iw;        // 8 * ld
  long long* prof;  // optional phase clocks (device profiling), may be null
};

// phase clock accumulation (thread 0 only): [0] products [1] LU
// [2] solve + kappa (+ the singular fallback) [3] eig (Hessenberg + QR) [4] select + eigenvectors [5] QRCP(P)
// [6] GP tail [7] QR iterations [8] bulge steps [9] calls
#define SKR_PHASE(ar, c, idx, t0)                                  \
  do {                                                            \
    if ((ar).prof && (c).tid == 0) {                              \
      long long _t = SKR_CLK();                                   \
      (ar).prof[idx] += _t - (t0);                                \
      (t0) = _t;                                                  \
    }                                                             \
  } while (0)

// arena leading dimension for Arnoldi length m: the matrices are at most
// (m + 1) x (m + 1); odd for fewer shared-memory bank conflicts
SKR_HD int arena_ld(int m) { return (m + 1) | 1; }
SKR_HD size_t arena_doubles(int nw, int ld) {
  return (size_t)5 * ld * ld + 12 * ld + (size_t)nw * 3 * DMAX + 64;
}
SKR_HD size_t arena_ints(int ld) { return 8 * (size_t)ld; }

SKR_HD Arena make_arena(double* d, int* iw, int nw, int ld) {
  Arena a;
  size_t M = (size_t)ld * ld;
  a.ld = ld;
  a.G = d;
  a.M1 = d + M;
  a.M2 = d + 2 * M;
  a.M3 = d + 3 * M;
  a.M4 = d + 4 * M;
  a.vec = d + 5 * M;
  a.xwork = a.vec + 12 * ld;
  a.red = a.xwork + (size_t)nw * 3 * DMAX;
  a.iw = iw;
  a.prof = 0;
  return a;
}

// exact reference singularity test: sigma_max == 0 or sigma_min < 1e-14 sigma_max
SKR_HD bool svd_singular(const Ctx& c, Arena& ar, const double* A, int lda, int n, double* work) {
  copy_mat(c, A, lda, work, ar.ld, n, n);
  bsync();
  double* sv = ar.vec + 8 * ar.ld;
  jacobi_svd(c, work, ar.ld, n, n, 0, 0, sv, ar.red);
  double mx = 0.0, mn = INFINITY;
  for (int i = 0; i < n; ++i) {
    mx = sv[i] > mx ? sv[i] : mx;
    mn = sv[i] < mn ? sv[i] : mn;
  }
  bsync();
  return mx == 0.0 || mn < SING_RTOL * mx;
}

// harmonic_ritz_first_cycle (gcrodr.py:173-206). H: (m+1) x m raw Arnoldi
// Hessenberg (only H[:m,:m] and H[m, m-1] are used). Result P_o (m x r1,
// orthonormal) in ar.M2; returns r1 >= 1, or -status.
SKR_HD int hr_first(const Ctx& c, Arena& ar, const double* H, int ldh, int m, int k, int* warn) {
  if (m <= 0 || m > DMAX) return -D_LINALG_ERROR;
  int kk = k < m ? k : m;
  int* piv = ar.iw;
  double hsub = DA(H, ldh, m, m - 1);
  for (Flat2 f_(c, m, m); f_.ok(); f_.next()) {
    int i = f_.i, j = f_.j;
    DA(ar.M2, ar.ld, i, j) = DA(H, ldh, j, i);  // Hs^T
    DA(ar.M1, ar.ld, i, j) = DA(H, ldh, i, j);  // Hs
  }
  bsync();
  double fn = fro_norm(c, ar.M1, ar.ld, m, m, ar.red);
  int info = 0;
  lu_factor(c, ar.M2, ar.ld, m, piv, &info);
  bool singular = info != 0;
  if (!singular) {
    // [e_m | I]
    for (Flat2 f_(c, m, (m + 1)); f_.ok(); f_.next()) {
      int i = f_.i, j = f_.j;
      DA(ar.M3, ar.ld, i, j) = (j == 0) ? (i == m - 1 ? 1.0 : 0.0) : (i == j - 1 ? 1.0 : 0.0);
    }
    bsync();
    lu_solve(c, ar.M2, ar.ld, m, piv, ar.M3, ar.ld, m + 1);
    double gn = fro_norm(c, ar.M3 + ar.ld, ar.ld, m, m, ar.red);
    if (!(fn * gn < KAPPA_CERT)) {
      *warn |= W_JACOBI_SVD;
      singular = svd_singular(c, ar, ar.M1, ar.ld, m, ar.M4);
    }
  }
  if (singular) {
    // gcrodr.py:196-203: the generalized problem (H^T H + h^2 e e^T) z =
    // theta H^T z (the reference: QZ, scipy eig(lhs, H^T)). Solved here as the
    // ordinary problem of (A - sigma H^T)^-1 H^T, A = H^T H + h^2 e e^T, whose
    // eigenvalues are nu = 1 / (theta - sigma) with the same eigenvectors; the
    // pencil's infinite eigenvalues (H^T singular) become nu = 0 and are never
    // among the k smallest |theta|; the selection runs on theta = sigma + 1/nu.
    // sigma = 0 unless A is singular or badly conditioned (a null vector of H
    // orthogonal to e_m makes theta = 0 an eigenvalue), then small shifts.
    *warn |= W_SINGULAR_H;
    const double h2 = hsub * hsub;
    double sigma = 0.0;
    bool ok = false;
    for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
      gemm(c, true, ar.M1, ar.ld, ar.M1, ar.ld, ar.M2, ar.ld, m, m, m);  // Hs^T Hs
      bsync();
      if (attempt > 0) {
        const double an = fro_norm(c, ar.M2, ar.ld, m, m, ar.red) + h2;
        const double fac[3] = {1.0e-3, -7.3e-3, 3.1e-2};
        sigma = fac[attempt - 1] * an / (fn > 0.0 ? fn : 1.0);
      }
      for (Flat2 f_(c, m, m); f_.ok(); f_.next()) {
        const int i = f_.i, j = f_.j;
        DA(ar.M2, ar.ld, i, j) -= sigma * DA(ar.M1, ar.ld, j, i);  // - sigma H^T
        DA(ar.M4, ar.ld, i, j) = DA(ar.M1, ar.ld, j, i);            // H^T
      }
      bsync();
      if (c.tid == 0) DA(ar.M2, ar.ld, m - 1, m - 1) += h2;
      bsync();
      const double an2 = fro_norm(c, ar.M2, ar.ld, m, m, ar.red);
      int info2 = 0;
      lu_factor(c, ar.M2, ar.ld, m, piv, &info2);
      if (info2 != 0) continue;
      // conditioning certificate ||S||_F ||S^-1||_F from S^-1 (identity RHS in M3)
      for (Flat2 f_(c, m, m); f_.ok(); f_.next())
        DA(ar.M3, ar.ld, f_.i, f_.j) = f_.i == f_.j ? 1.0 : 0.0;
      bsync();
      lu_solve(c, ar.M2, ar.ld, m, piv, ar.M3, ar.ld, m);
      const double gn2 = fro_norm(c, ar.M3, ar.ld, m, m, ar.red);
      if (!(an2 * gn2 < KAPPA_CERT)) continue;
      lu_solve(c, ar.M2, ar.ld, m, piv, ar.M4, ar.ld, m);  // M4 = (A - sigma H^T)^-1 H^T
      bsync();
      ok = true;
    }
    if (!ok) return -D_LINALG_ERROR;
    double* wr = ar.vec;
    double* wi = ar.vec + ar.ld;
    // Z log in M2 (the LU factors of A are dead)
    if (eig_schur(c, ar.M4, ar.ld, m, ar.M3, ar.ld, wr, wi, ar.vec + 2 * ar.ld, ar.M2,
                  ar.ld * ar.ld / ZREC) != 0)
      return -D_QR_NOCONV;
    double* kr = ar.vec + 9 * ar.ld;  // theta = sigma + 1 / nu (inf for nu = 0)
    double* ki = ar.vec + 10 * ar.ld;
    for (int i = c.tid; i < m; i += c.nt) {
      const double d2 = wr[i] * wr[i] + wi[i] * wi[i];
      kr[i] = d2 > 0.0 ? sigma + wr[i] / d2 : INFINITY;
      ki[i] = d2 > 0.0 ? -wi[i] / d2 : 0.0;
    }
    bsync();
    int ncols = select_basis(c, ar.M4, ar.ld, m, ar.M3, ar.ld, wr, wi, kk, m, ar.M1, ar.ld,
                             ar.iw + ar.ld, ar.xwork, ar.red, kr, ki);
    if (ncols < 0) return -D_LINALG_ERROR;
    int* jp = ar.iw + 6 * ar.ld;
    return qrcp(c, ar.M1, ar.ld, m, ncols, jp, ar.M2, ar.ld, RANK_RTOL, ar.vec + 2 * ar.ld,
                ar.vec + 5 * ar.ld);
  }
  // modified = Hs + h^2 f e_m^T
  double h2 = hsub * hsub;
  for (int i = c.tid; i < m; i += c.nt) DA(ar.M1, ar.ld, i, m - 1) += h2 * DA(ar.M3, ar.ld, i, 0);
  bsync();
  double* wr = ar.vec;
  double* wi = ar.vec + ar.ld;
  // Z log in M2 (the LU factors are dead; qrcp writes M2 only after select)
  if (eig_schur(c, ar.M1, ar.ld, m, ar.M3, ar.ld, wr, wi, ar.vec + 2 * ar.ld, ar.M2,
                ar.ld * ar.ld / ZREC) != 0)
    return -D_QR_NOCONV;
  int ncols = select_basis(c, ar.M1, ar.ld, m, ar.M3, ar.ld, wr, wi, kk, m, ar.M4, ar.ld, ar.iw + ar.ld,
                           ar.xwork, ar.red);
  if (ncols < 0) return -D_LINALG_ERROR;
  int* jp = ar.iw + 6 * ar.ld;
  int r1 = qrcp(c, ar.M4, ar.ld, m, ncols, jp, ar.M2, ar.ld, RANK_RTOL, ar.vec + 2 * ar.ld,
                ar.vec + 5 * ar.ld);
  return r1;
}

// harmonic_ritz_subsequent (gcrodr.py:209-240). G in ar.G ((mm+1) x mm),
// cross: mm x mm (leading block of What^T Vhat). P_o (mm x r1) in ar.M2.
SKR_HD int hr_next(const Ctx& c, Arena& ar, int mm, const double* cross, int ldx, int k, int* warn) {
  if (mm <= 0 || mm > DMAX) return -D_LINALG_ERROR;
  int kk = k < mm ? k : mm;
  int* piv = ar.iw;
  long long t0 = SKR_CLK();
  gemm(c, true, ar.G, ar.ld, ar.G, ar.ld, ar.M1, ar.ld, mm, mm, mm + 1);   // lhs = G^T G
  gemm(c, true, ar.G, ar.ld, cross, ldx, ar.M2, ar.ld, mm, mm, mm);      // rhs = G[:mm]^T cross
  bsync();
  SKR_PHASE(ar, c, 0, t0);
  double fn = fro_norm(c, ar.M2, ar.ld, mm, mm, ar.red);
  int info = 0;
  lu_factor(c, ar.M2, ar.ld, mm, piv, &info);
  SKR_PHASE(ar, c, 1, t0);
  bool singular = info != 0;
  // one LU solve for [I | lhs]: I at M3 columns [ar.ld-mm, ar.ld), lhs at M4[:, 0:mm)
  // (M3 and M4 are adjacent, so the 2 mm right-hand sides are contiguous)
  double* X = ar.M3 + (size_t)(ar.ld - mm) * ar.ld;
  if (!singular) {
    for (Flat2 f_(c, mm, mm); f_.ok(); f_.next()) {
      int i = f_.i, j = f_.j;
      DA(X, ar.ld, i, j) = (i == j) ? 1.0 : 0.0;
      DA(ar.M4, ar.ld, i, j) = DA(ar.M1, ar.ld, i, j);
    }
    bsync();
    lu_solve(c, ar.M2, ar.ld, mm, piv, X, ar.ld, 2 * mm);
    double gn = fro_norm(c, X, ar.ld, mm, mm, ar.red);
    if (!(fn * gn < KAPPA_CERT)) {
      *warn |= W_JACOBI_SVD;
      gemm(c, true, ar.G, ar.ld, cross, ldx, ar.M3, ar.ld, mm, mm, mm);  // rhs again
      bsync();
      singular = svd_singular(c, ar, ar.M3, ar.ld, mm, ar.M2);
    }
  }
  if (singular) {
    *warn |= W_SINGULAR_CROSS;
    // pinv(rhs) via Jacobi SVD: M3 <- U S, M2 <- V, M4 <- pinv, A = pinv lhs -> M4
    gemm(c, true, ar.G, ar.ld, cross, ldx, ar.M3, ar.ld, mm, mm, mm);
    bsync();
    double* sv = ar.vec + 8 * ar.ld;
    jacobi_svd(c, ar.M3, ar.ld, mm, mm, ar.M2, ar.ld, sv, ar.red);
    double mx = 0.0;
    for (int i = 0; i < mm; ++i) mx = sv[i] > mx ? sv[i] : mx;
    double cut = 1e-15 * mx;  // numpy pinv default rcond
    for (Flat2 f_(c, mm, mm); f_.ok(); f_.next()) {
      int i = f_.i, j = f_.j;
      double sacc = 0.0;
      for (int q = 0; q < mm; ++q)
        if (sv[q] > cut) sacc += DA(ar.M2, ar.ld, i, q) * DA(ar.M3, ar.ld, j, q) / (sv[q] * sv[q]);
      DA(ar.M4, ar.ld, i, j) = sacc;
    }
    bsync();
    gemm(c, false, ar.M4, ar.ld, ar.M1, ar.ld, ar.M3, ar.ld, mm, mm, mm);  // pinv @ lhs
    bsync();
    copy_mat(c, ar.M3, ar.ld, ar.M4, ar.ld, mm, mm);
    bsync();
  }
  SKR_PHASE(ar, c, 2, t0);
  double* wr = ar.vec;
  double* wi = ar.vec + ar.ld;
  hessenberg(c, ar.M4, ar.ld, mm, ar.M3, ar.ld, ar.vec + 2 * ar.ld);
  SKR_PHASE(ar, c, 10, t0);
  // Z log in M1..M2 (adjacent; lhs and the LU factors are dead until select)
  int est = hqr(c, ar.M4, ar.ld, mm, ar.M3, ar.ld, wr, wi, ar.vec + 2 * ar.ld, ar.M1,
                2 * ar.ld * ar.ld / ZREC);
  if (ar.prof && c.tid == 0) {
    ar.prof[7] += (long long)ar.vec[2 * ar.ld + 1];
    ar.prof[8] += (long long)ar.vec[2 * ar.ld + 2];
    ar.prof[9] += 1;
    for (int q = 0; q < 4; ++q) ar.prof[11 + q] += (long long)ar.vec[2 * ar.ld + 3 + q];
  }
  SKR_PHASE(ar, c, 3, t0);
  if (est != 0) return -D_QR_NOCONV;
  int ncols = select_basis(c, ar.M4, ar.ld, mm, ar.M3, ar.ld, wr, wi, kk, mm, ar.M1, ar.ld,
                           ar.iw + ar.ld, ar.xwork, ar.red);
  SKR_PHASE(ar, c, 4, t0);
  if (ncols < 0) return -D_LINALG_ERROR;
  int* jp = ar.iw + 6 * ar.ld;
  int r1 = qrcp(c, ar.M1, ar.ld, mm, ncols, jp, ar.M2, ar.ld, RANK_RTOL, ar.vec + 2 * ar.ld,
                ar.vec + 5 * ar.ld);
  SKR_PHASE(ar, c, 5, t0);
  return r1;
}

// Common tail: GP = G P_o ((rows) x r1) -> QRCP -> Q, R, kept; Z = P_o[:,kept] R^-1.
// Writes coefC (rows x r2) = Q and Zc (cols x r2) = Z. Returns r2.
SKR_HD int gp_tail(const Ctx& c, Arena& ar, int rows, int cols, int r1, double* Zc, int ldz,
                   double* Qc, int ldq) {
  gemm(c, false, ar.G, ar.ld, ar.M2, ar.ld, ar.M1, ar.ld, rows, r1, cols);
  bsync();
  int* jp = ar.iw + 6 * ar.ld;
  int r2 = qrcp(c, ar.M1, ar.ld, rows, r1, jp, ar.M3, ar.ld, RANK_RTOL, ar.vec + 2 * ar.ld,
                ar.vec + 5 * ar.ld);
  if (r2 <= 0) return 0;
  inv_upper(c, ar.M1, ar.ld, r2, ar.M4, ar.ld);
  for (Flat2 f_(c, cols, r2); f_.ok(); f_.next()) {
    int i = f_.i, j = f_.j;
    double s = 0.0;
    for (int q = 0; q <= j; ++q) s += DA(ar.M2, ar.ld, i, jp[q]) * DA(ar.M4, ar.ld, q, j);
    DA(Zc, ldz, i, j) = s;
  }
  for (Flat2 f_(c, rows, r2); f_.ok(); f_.next()) {
    int i = f_.i, j = f_.j;
    DA(Qc, ldq, i, j) = DA(ar.M3, ar.ld, i, j);
  }
  bsync();
  return r2;
}

// First-cycle recycle pair (gcrodr.py:280-292). H: (j+1) x j.
// U = V[:, :j] coefU (coefU: j x r), C = V[:, :j+1] coefC ((j+1) x r).
// Returns r >= 1, 0 when the rank collapsed, or -status (U stays None).
SKR_HD int recycle_first(const Ctx& c, Arena& ar, const double* H, int ldh, int j, int k,
                         double* coefU, int ldu, double* coefC, int ldcc, int* warn) {
  int kk = k < j ? k : j;
  int r1 = hr_first(c, ar, H, ldh, j, kk, warn);
  if (r1 <= 0) return r1 < 0 ? r1 : 0;
  for (Flat2 f_(c, j + 1, j); f_.ok(); f_.next()) {
    int i = f_.i, q = f_.j;
    DA(ar.G, ar.ld, i, q) = DA(H, ldh, i, q);
  }
  bsync();
  return gp_tail(c, ar, j + 1, j, r1, coefU, ldu, coefC, ldcc);
}

// Subsequent-cycle update (gcrodr.py:444-460). mm = kc + j. G built from dk,
// B (kc x j) and H ((j+1) x j). coefU rows: [U cols 0..kc) (dk folded in:
// Vhat = [U diag(dk), V]) | V_0..V_{j-1}]; coefC rows: [C cols | V_0..V_j].
SKR_HD int recycle_next(const Ctx& c, Arena& ar, const double* H, int ldh, const double* B,
                        int ldb, const double* dk, int kc, int j, const double* cross, int ldx,
                        int k, double* coefU, int ldu, double* coefC, int ldcc, int* warn) {
  int mm = kc + j;
  if (mm + 1 > ar.ld) return -D_LINALG_ERROR;
  for (Flat2 f_(c, mm + 1, mm); f_.ok(); f_.next()) {
    int i = f_.i, q = f_.j;
    double v = 0.0;
    if (i < kc && q < kc)
      v = (i == q) ? dk[i] : 0.0;
    else if (i < kc)
      v = DA(B, ldb, i, q - kc);
    else if (q >= kc)
      v = DA(H, ldh, i - kc, q - kc);
    DA(ar.G, ar.ld, i, q) = v;
  }
  bsync();
  int r1 = hr_next(c, ar, mm, cross, ldx, k, warn);
  if (r1 <= 0) return r1 < 0 ? r1 : 0;
  long long t0 = SKR_CLK();
  int r2 = gp_tail(c, ar, mm + 1, mm, r1, coefU, ldu, coefC, ldcc);
  SKR_PHASE(ar, c, 6, t0);
  if (r2 <= 0) return 0;
  for (Flat2 f_(c, kc, r2); f_.ok(); f_.next()) {
    int i = f_.i, q = f_.j;
    DA(coefU, ldu, i, q) *= dk[i];
  }
  bsync();
  return r2;
}

// ---------------------------------------------------------------------------
// CholQR building blocks for the refresh (orth(U) and QRCP(op U)).
// Pass 1: diagonally-scaled pivoted Cholesky of the Gram matrix Gm (k x k).
// Columns whose scaled Schur diagonal falls below drop_tol are numerically
// dependent at Gram precision and dropped. Outputs T1 (k x r: X T1 has
// orthonormal columns spanning X[:, perm[:r]]) and R1 (r x k, original column
// order, X ~= (X T1) R1). Returns r.
// ---------------------------------------------------------------------------
SKR_HD int cholqr_pass1(const Ctx& c, Arena& ar, const double* Gm, int ldg, int k, double* T1,
                        int ldt, double* R1, int ldr) {
  double* S = ar.M1;
  double* R = ar.M2;
  double* dsq = ar.vec;       // sqrt(diag)
  int* perm = ar.iw;          // k
  int* meta = ar.iw + ar.ld;    // [0] = rank, [1] = pivot
  const double drop_tol = 1e-13;
  for (int i = c.tid; i < k; i += c.nt) {
    double d = DA(Gm, ldg, i, i);
    dsq[i] = d > 0.0 ? sqrt(d) : 0.0;
    perm[i] = i;
  }
  bsync();
  for (Flat2 f_(c, k, k); f_.ok(); f_.next()) {
    int i = f_.i, j = f_.j;
    double den = dsq[i] * dsq[j];
    DA(S, ar.ld, i, j) = den > 0.0 ? DA(Gm, ldg, i, j) / den : 0.0;
    DA(R, ar.ld, i, j) = 0.0;
  }
  bsync();
  int rank = k;
  for (int i = 0; i < k; ++i) {
    if (c.tid == 0) {
      int p = i;
      double best = DA(S, ar.ld, i, i);
      for (int q = i + 1; q < k; ++q)
        if (DA(S, ar.ld, q, q) > best) {
          best = DA(S, ar.ld, q, q);
          p = q;
        }
      meta[1] = p;
      meta[0] = (best > drop_tol) ? 1 : 0;
    }
    bsync();
    if (!meta[0]) {
      rank = i;
      break;
    }
    int p = meta[1];
    if (p != i) {
      // symmetric swap of rows/cols i,p of S, columns of R (rows < i), perm
      for (int q = c.tid; q < k; q += c.nt) {
        double t = DA(S, ar.ld, i, q);
        DA(S, ar.ld, i, q) = DA(S, ar.ld, p, q);
        DA(S, ar.ld, p, q) = t;
      }
      bsync();
      for (int q = c.tid; q < k; q += c.nt) {
        double t = DA(S, ar.ld, q, i);
        DA(S, ar.ld, q, i) = DA(S, ar.ld, q, p);
        DA(S, ar.ld, q, p) = t;
        if (q < i) {
          double u = DA(R, ar.ld, q, i);
          DA(R, ar.ld, q, i) = DA(R, ar.ld, q, p);
          DA(R, ar.ld, q, p) = u;
        }
      }
      if (c.tid == 0) {
        int t = perm[i];
        perm[i] = perm[p];
        perm[p] = t;
      }
      bsync();
    }
    double rii = sqrt(DA(S, ar.ld, i, i));
    for (int q = i + c.tid; q < k; q += c.nt)
      DA(R, ar.ld, i, q) = (q == i) ? rii : DA(S, ar.ld, i, q) / rii;
    bsync();
    int rem = k - i - 1;
    for (Flat2 f_(c, rem, rem); f_.ok(); f_.next()) {
      int a = i + 1 + f_.i, b = i + 1 + f_.j;
      DA(S, ar.ld, a, b) -= DA(R, ar.ld, i, a) * DA(R, ar.ld, i, b);
    }
    bsync();
  }
  // unscale: R_true(:, q) = R(:, q) * dsq[perm[q]]
  for (Flat2 f_(c, rank, k); f_.ok(); f_.next()) {
    int i = f_.i, q = f_.j;
    DA(R, ar.ld, i, q) *= dsq[perm[q]];
  }
  bsync();
  if (rank > 0) inv_upper(c, R, ar.ld, rank, ar.M3, ar.ld);
  for (Flat2 f_(c, k, rank); f_.ok(); f_.next()) {
    int i = f_.i, q = f_.j;
    DA(T1, ldt, i, q) = 0.0;
  }
  bsync();
  for (Flat2 f_(c, rank, rank); f_.ok(); f_.next()) {
    int i = f_.i, q = f_.j;
    DA(T1, ldt, perm[i], q) = DA(ar.M3, ar.ld, i, q);
  }
  for (Flat2 f_(c, rank, k); f_.ok(); f_.next()) {
    int i = f_.i, q = f_.j;
    DA(R1, ldr, i, perm[q]) = DA(R, ar.ld, i, q);
  }
  bsync();
  return rank;
}

// Pass 2 + rank decision: Gram G2 (r x r) of X1 = X T1, R1 (r x k) from pass 1.
// R_tot = R2 R1 and QRCP(R_tot) gives the reference's QRCP(X) pivots / rank
// (|R'_ii| >= 1e-12 |R'_00|). Outputs T2 (r x r2): X1 T2 = Q[:, :r2] of
// QRCP(X); kept[0..r2) = pivots into X's columns; Rinv (r2 x r2) = R'^-1.
// Returns r2 (0 = collapsed).
SKR_HD int cholqr_pass2(const Ctx& c, Arena& ar, const double* G2, int ldg, int r, const double* R1,
                        int ldr, int k, double* T2, int ldt, int* kept, double* Rinv, int ldri) {
  if (r <= 0) return 0;
  // pass-2 Cholesky (pivoted routine: G2 ~ I, so it keeps every column)
  double* T2a = ar.G;  // r x r2a
  double* R2 = ar.M4;  // r2a x r (original order)
  int r2a = cholqr_pass1(c, ar, G2, ldg, r, T2a, ar.ld, R2, ar.ld);
  if (r2a <= 0) return 0;
  // R_tot = R2 R1 (r2a x k) -> M1
  gemm(c, false, R2, ar.ld, R1, ldr, ar.M1, ar.ld, r2a, k, r);
  bsync();
  int* jp = ar.iw + 6 * ar.ld;
  int r2 = qrcp(c, ar.M1, ar.ld, r2a, k, jp, ar.M3, ar.ld, RANK_RTOL, ar.vec + 2 * ar.ld,
                ar.vec + 5 * ar.ld);
  if (r2 <= 0) return 0;
  // T2 = T2a Q'[:, :r2]  (r x r2)
  gemm(c, false, T2a, ar.ld, ar.M3, ar.ld, T2, ldt, r, r2, r2a);
  inv_upper(c, ar.M1, ar.ld, r2, Rinv, ldri);
  for (int i = c.tid; i < r2; i += c.nt) kept[i] = jp[i];
  bsync();
  return r2;
}

}  // namespace skrd
