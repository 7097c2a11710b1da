// General left preconditioners on the device (kryrec/precond.py:80-145, :251-312):
// SOR, ILU(0), IC(0) as level-scheduled sparse triangular sweeps, block Jacobi
// as per-block dense LU solves. "apply" = solve M z = v in place.
//
// Triangular kinds keep their factor on the CSR pattern of the matrix they
// were built from (rows sorted): fval[q] is the factor entry at pattern
// position q, dpos[i] the position of row i's diagonal. The lower sweep uses
// the entries left of the diagonal, the upper sweep those right of it (IC(0)
// stores L^T there, mirrored at build time). Rows are grouped into dependency
// levels (all rows of a level are independent). A sweep walks the levels;
// runs of narrow levels are swept by CTA 0 alone with a block barrier per
// level, wide levels by the whole grid with one grid barrier each. Each row is
// one sequential sum (separate multiply and subtract), so the result does not
// depend on how a level's rows are spread over threads.
#pragma once
#include "skr_device.cuh"

namespace skr {

enum PcKind { PC_NONE = 0, PC_SOR = 1, PC_ILU0 = 2, PC_ICC0 = 3, PC_BJACOBI = 4 };
enum PcDiv { PCD_UNIT = 0, PCD_FACTOR = 1 };
enum PcStatus { PCS_OK = 0, PCS_ZERO_PIVOT = 1, PCS_NOT_SYMMETRIC = 2, PCS_ABORTED = 3 };

constexpr int PC_NARROW = 2 * NT;  // rows up to which a level is swept by one CTA
constexpr int PC_ELL = 3;           // entries per row kept in the slot-major arrays

struct PcView {
  int kind;        // PcKind
  int n;
  int nsweep;      // triangular sweeps per apply (1: SOR, 2: ILU0 / ICC0)
  int upper[2];    // sweep s uses the upper (1) or lower (0) part
  int dmode[2];    // PcDiv of sweep s
  int nlev[2];     // levels of the lower [0] / upper [1] schedule
  const int* rp;   // pattern the factor lives on (the caller's CSR arrays)
  const int* ci;
  const double* fval;
  const int* dpos;
  const int* lptr[2];   // level l of schedule h: rows lrows[h][lptr[h][l] .. lptr[h][l+1])
  const int* lrows[2];
  // the sweeps' operands packed in level order (position e of schedule h is row
  // lrows[h][e]): its off-diagonal factor entries pval / pci [prp[e], prp[e+1])
  // and its divisor pdiv[e] (1 for the unit-diagonal sweep). A level's operands
  // are contiguous and do not depend on the solution, so they are prefetched
  // while the previous level is solved.
  const int* prp[2];
  const int* pci[2];
  const double* pval[2];
  const double* pdiv[2];
  // the first PC_ELL entries of every position again, slot-major (slot k of
  // position e at [k n + e]; unused slots: the row itself with a zero value):
  // addresses that depend on e only, so a whole level's operands are one
  // round trip and can be loaded while the previous level is solved
  const int* eci[2];
  const double* eval[2];
  double scale;         // ICC0: sign (1 otherwise)
  int bs, nb;           // block Jacobi: block size, number of blocks
  const double* lu;     // nb x (bs x bs) column-major LU factors (unit L below the diagonal)
  const int* perm;      // n: row (within its block) gathered into position i
};

// Device-resident head of a preconditioner buffer (skr_precond_build).
struct PcHeader {
  PcView v;
  int status;           // PcStatus
  int err_row;          // first row with a zero / nonpositive pivot (n: none)
  double err_value;
  int any_nonneg_diag;  // ICC0 sign test
  int maxlev[2];
  int chg[3];
  int pad0[32];
  unsigned long long bar_count;  // the build / standalone-apply kernels' grid barrier
  unsigned bar_pad[62];
  int abort_flag;
};

// One triangular sweep over `ncols` columns of v (leading dimension ldv),
// grid-cooperative: sync() is the caller's grid barrier (false = aborted).
// operands of one position of a schedule (solution-independent)
struct PcRowOps {
  int i, q0, cnt;
  double dv;
  int c[PC_ELL];
  double a[PC_ELL];
};

template <class Sync>
__device__ __forceinline__ bool pc_tri_sweep(const PcView& pc, int s, double* v, int ncols,
                                             size_t ldv, Sync&& sync) {
  const int up = pc.upper[s];
  const int* lptr = pc.lptr[up];
  const int* lrows = pc.lrows[up];
  const int* prp = pc.prp[up];
  const int* pci = pc.pci[up];
  const double* pval = pc.pval[up];
  const double* pdiv = pc.pdiv[up];
  const int* eci = pc.eci[up];
  const double* eval = pc.eval[up];
  const int nlev = pc.nlev[up];
  const int n = pc.n;
  auto load_ops = [&](int e) -> PcRowOps {
    PcRowOps o;
    o.i = __ldg(lrows + e);
    o.q0 = __ldg(prp + e);
    o.cnt = __ldg(prp + e + 1) - o.q0;
    o.dv = __ldg(pdiv + e);
#pragma unroll
    for (int k = 0; k < PC_ELL; ++k) {
      o.c[k] = __ldg(eci + (size_t)k * n + e);
      o.a[k] = __ldg(eval + (size_t)k * n + e);
    }
    return o;
  };
  auto solve_row = [&](const PcRowOps& o, double* col) {
    double x[PC_ELL];
#pragma unroll
    for (int k = 0; k < PC_ELL; ++k) x[k] = col[o.c[k]];  // (unused slots read the row itself)
    double acc = col[o.i];
#pragma unroll
    for (int k = 0; k < PC_ELL; ++k)
      if (k < o.cnt) acc = __dsub_rn(acc, __dmul_rn(o.a[k], x[k]));
    for (int q = o.q0 + PC_ELL; q < o.q0 + o.cnt; ++q)
      acc = __dsub_rn(acc, __dmul_rn(__ldg(pval + q), col[__ldg(pci + q)]));
    col[o.i] = __ddiv_rn(acc, o.dv);
  };
  auto do_rows = [&](int lo, int nr, int first, int stride) {
    for (int it = first; it < nr * ncols; it += stride) {
      const int cidx = ncols == 1 ? 0 : it / nr;
      solve_row(load_ops(lo + it - cidx * nr), v + (size_t)cidx * ldv);
    }
  };
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int gthreads = gridDim.x * blockDim.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  int l = 0;
  int lo = __ldg(lptr);
  while (l < nlev) {
    int hi = __ldg(lptr + l + 1);
    if ((hi - lo) * ncols <= PC_NARROW) {
      // a run of narrow levels: CTA 0 alone, a block barrier per level. With one
      // column a thread's first row of the NEXT level is loaded (operands
      // only) before this level's solution-dependent loads, so a level costs
      // one L2 round trip instead of a chain of them.
      int l1 = l;
      PcRowOps nxt;
      bool have = false;
      if (blockIdx.x == 0 && ncols == 1 && tid < hi - lo) {
        nxt = load_ops(lo + tid);
        have = true;
      }
      while (true) {
        const int nhi = l1 + 1 < nlev ? __ldg(lptr + l1 + 2) : hi;
        const bool nnarrow = l1 + 1 < nlev && (nhi - hi) * ncols <= PC_NARROW;
        if (blockIdx.x == 0) {
          if (ncols == 1) {
            const PcRowOps cur = nxt;
            const bool hcur = have;
            have = nnarrow && tid < nhi - hi;
            if (have) nxt = load_ops(hi + tid);
            if (hcur) solve_row(cur, v);
            for (int it = tid + nt; it < hi - lo; it += nt) solve_row(load_ops(lo + it), v);
          } else {
            do_rows(lo, hi - lo, tid, nt);
          }
          __syncthreads();
        }
        lo = hi;
        ++l1;
        if (!nnarrow) break;
        hi = nhi;
      }
      l = l1;
    } else {
      do_rows(lo, hi - lo, gtid, gthreads);
      lo = hi;
      ++l;
    }
    if (!sync()) return false;
  }
  return true;
}

// Block Jacobi: block b's slice of every column <- U^-1 L^-1 P (slice), one
// warp per (block, column); RB = ceil(bs / 32) entries per lane in registers.
// The factor's columns stream through registers D columns ahead of the
// substitution step that uses them (they do not depend on the solution), so
// the sequential steps do not each wait for their own memory round trip.
template <int RB>
__device__ __forceinline__ void pc_block_solve(const PcView& pc, double* v, int ncols, size_t ldv,
                                               int n) {
  constexpr int D = RB <= 2 ? 8 : 1;  // columns in flight (blocks of up to 64 rows: 8)
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int bs = pc.bs;
  for (int it = gw; it < pc.nb * ncols; it += nw) {
    const int b = it % pc.nb;
    double* col = v + (size_t)(it / pc.nb) * ldv;
    const int start = b * bs, bsz = min(bs, n - start);
    const double* lu = pc.lu + (size_t)b * bs * bs;
    double x[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int i = 32 * r + lane;
      x[r] = i < bsz ? col[start + __ldg(pc.perm + start + i)] : 0.0;
    }
    __syncwarp();  // every gather is done before the slice is overwritten
    double cur[D][RB], nxt[D][RB];
    auto load_chunk = [&](double (&dst)[D][RB], int k0) {  // columns k0 .. k0 + D - 1
#pragma unroll
      for (int d = 0; d < D; ++d)
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const int i = 32 * r + lane, k = k0 + d;
          dst[d][r] = (k >= 0 && k < bsz && i < bsz) ? __ldg(lu + i + (size_t)k * bs) : 0.0;
        }
    };
    auto x_at = [&](int k) -> double {  // x[k] of the block, broadcast
      double src = x[0];
#pragma unroll
      for (int r = 1; r < RB; ++r)
        if (r == (k >> 5)) src = x[r];
      return __shfl_sync(0xffffffffu, src, k & 31);
    };
    // forward, unit lower
    load_chunk(nxt, 0);
    for (int k0 = 0; k0 < bsz; k0 += D) {
#pragma unroll
      for (int d = 0; d < D; ++d)
#pragma unroll
        for (int r = 0; r < RB; ++r) cur[d][r] = nxt[d][r];
      if (k0 + D < bsz) load_chunk(nxt, k0 + D);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int k = k0 + d;
        if (k < bsz) {
          const double xk = x_at(k);
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            const int i = 32 * r + lane;
            if (i > k && i < bsz) x[r] = __dsub_rn(x[r], __dmul_rn(cur[d][r], xk));
          }
        }
      }
    }
    // backward, upper: chunks of columns from the last one down
    const int klast = ((bsz - 1) / D) * D;
    load_chunk(nxt, klast);
    for (int k0 = klast; k0 >= 0; k0 -= D) {
#pragma unroll
      for (int d = 0; d < D; ++d)
#pragma unroll
        for (int r = 0; r < RB; ++r) cur[d][r] = nxt[d][r];
      if (k0 - D >= 0) load_chunk(nxt, k0 - D);
#pragma unroll
      for (int d = D - 1; d >= 0; --d) {
        const int k = k0 + d;
        if (k < bsz) {
          // the diagonal entry lives in the lane that owns row k
#pragma unroll
          for (int r = 0; r < RB; ++r)
            if (r == (k >> 5) && lane == (k & 31)) x[r] = __ddiv_rn(x[r], cur[d][r]);
          const double xk = x_at(k);
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            const int i = 32 * r + lane;
            if (i < k) x[r] = __dsub_rn(x[r], __dmul_rn(cur[d][r], xk));
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int i = 32 * r + lane;
      if (i < bsz) col[start + i] = x[r];
    }
  }
}

// v[:, c] <- M^-1 v[:, c] for c < ncols, by every CTA of a cooperative grid.
// The caller has made v visible grid-wide (a barrier after it was written);
// on return (true) the result is visible grid-wide as well.
// FAMILY: 1 = triangular kinds only, 2 = block Jacobi only (the cycle kernel
// is instantiated per family so that neither's registers crowd the other),
// 0 = either (standalone kernels, run-time dispatch).
template <int FAMILY = 0, class Sync>
__device__ __forceinline__ bool pc_apply_grid(const PcView& pc, double* v, int ncols, size_t ldv,
                                              Sync&& sync) {
  const int n = pc.n;
  if (FAMILY == 2 || (FAMILY == 0 && pc.kind == PC_BJACOBI)) {
    if (pc.bs <= 32)
      pc_block_solve<1>(pc, v, ncols, ldv, n);
    else if (pc.bs <= 64)
      pc_block_solve<2>(pc, v, ncols, ldv, n);
    else if (pc.bs <= 128)
      pc_block_solve<4>(pc, v, ncols, ldv, n);
    else
      pc_block_solve<8>(pc, v, ncols, ldv, n);
    return sync();
  }
  for (int s = 0; s < pc.nsweep; ++s)
    if (!pc_tri_sweep(pc, s, v, ncols, ldv, sync)) return false;
  if (pc.scale != 1.0) {
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int gthreads = gridDim.x * blockDim.x;
    for (size_t e = gtid; e < (size_t)n * ncols; e += gthreads) {
      double* q = v + (e / n) * ldv + (e % n);
      *q = __dmul_rn(pc.scale, *q);
    }
    return sync();
  }
  return true;
}

}  // namespace skr
