// GCRO-DR solve for one sparse fp64 system on a B200, with the recycle pair
// carried between systems (kryrec/gcrodr.py:295-496 restated for the GPU).
//
// Kernels (one stream, no host sync inside a cycle):
//   k_setup / k_init           scalars, x0, r = M^-1 b, norms (gcrodr.py:332-353)
//   refresh chain              CholQR2 of U_in, W = op(Yo), CholQR2 + QRCP of W,
//                              U = Yo[:, kept] R^-1, projection (gcrodr.py:80-113, 360-378)
//   k_cycle (cooperative)      ONE launch per restart cycle: the whole deflated (or
//                              first GMRES) Arnoldi cycle with lagged one-reduction
//                              CGS2 (DCGS2: sweep 1 = SpMV + multi-dot, one grid
//                              reduction, sweep 2 = finishing AXPYs), Givens LS in
//                              every CTA, x update, explicit residual and the
//                              cross-Gram for the recycle update (gcrodr.py:398-448)
//   k_dense (1 CTA)            harmonic Ritz + QRCP recycle update, state machine
//                              (gcrodr.py:444-470, 280-292, dense.h / recycle.h)
//   k_combine                  U, C <- [U | C | V] coefficients, in place, row-parallel
// The host loop enqueues cycles ahead and polls a mapped flag the dense kernel
// writes, so the GPU never waits for the CPU.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "precond.cuh"
#include "recycle.h"
#include "skr_device.cuh"

namespace skr {

// ---------------------------------------------------------------------------
// device state
// ---------------------------------------------------------------------------
constexpr int LDH = MMAX + 1;          // ld of H (rows <= m+1)
constexpr int LDR = MMAX;              // ld of rotated R
constexpr int LDB = KMAX;              // ld of B
constexpr int LDX = MMAX;              // ld of cross
constexpr int LDC = KMAX + MMAX + 1;   // ld of coefficient matrices
constexpr int LDK = KMAX;              // ld of small k x k matrices

enum Prog {
  P_INIT = 0,
  P_CHOL1 = 1,   // CholQR pass 1 on a tall block (arg: 0 = U block, 1 = C block)
  P_CHOL2 = 2,   // pass 2 + QRCP(R) ; arg 0 = orth(U) ; arg 1 = QR(W) -> C, U
  P_PROJ_FIN = 3,
  P_CYCLE = 4,
  P_FINAL = 5,
};

enum CombineMode {
  CM_CYCLE = 0,     // U, C <- [U|V] coefU, [C|V] coefC (recycle update)
  CM_U_ONLY = 1,    // U[:, :nout] <- U[:, :nin] T
  CM_C_ONLY = 2,    // C <- C T
  CM_REFRESH = 3,   // C <- C Tc ; U <- U Tu
};

struct State {
  // config
  int n, ld, m, k, kcap, max_iter, jacobi, nblk, rpb, k_in, has_x0,
      comb_part,  // cycle-start partials: 0 = rows [0, 2kc) (k_project), 1 = COMB_PART0 rows
      comb_nblk,  // CTAs of the k_combine launch that wrote the COMB_PART0 rows
      ndiag,         // diagnostics records logged (SKR_COLLECT_DIAGNOSTICS)
      comb_pending;  // P_CYCLE left a recycle update (coefU / coefC) for the next
                     // k_cycle launch (or the final k_combine) to apply
  double tol;
  // scalars
  double bnorm, bprec, abs_tol, rnorm, true_rel;
  int iters, kc, kc_prev, k_new, converged, done, brk, ran, upd, j, cycles, defl_steps;
  int hist_len, nchecks, warn, status, abort_flag, zero_rhs, fallback, ncol_a, ncol_b, r_tmp,
      cm_mode, cm_nin_u, cm_nin_c, cm_nv, cm_nout_u, cm_nout_c, ncol_orig;
  unsigned long long bar_count;      // grid-barrier arrivals (never reset within a solve),
  unsigned bar_pad0[62];             // alone on its 256-byte line
  unsigned bar_pad1[64];
  int* host_flag;  // mapped pinned: [0] = last processed cycle, [1] = done
  // k_cycle neighbour epochs (stencil form): CTA b publishes at
  // nb_epoch[b * NB_STRIDE] how many Arnoldi sweeps 2 it has finished in this
  // solve; zeroed by k_init
  unsigned nb_epoch[GRID_MAX * 16];
  double step_bytes;  // algorithmic SpMV+ortho bytes accumulated
  int steps, v0proj;  // Arnoldi steps executed; cycles whose V_0 was formed from r - C c_r
  long long prof[32]; // [0,16) dense-kernel phase clocks (recycle.h SKR_PHASE),
                      // [16,24) k_cycle phase clocks of CTA 0
  int kept[KMAX];
  // per-cycle small data
  double H[LDH * MMAX];
  double B[LDB * MMAX];
  double R[LDR * MMAX];
  double g[MMAX + 1];
  double y[KMAX + MMAX];
  double dk[KMAX];
  double cr[KMAX];
  double cross[LDX * MMAX];
  double coefU[LDC * KMAX];
  double coefC[LDC * KMAX];
  double gram[LDK * KMAX];
  double R1[LDK * KMAX];
  double alpha[KMAX];
  double red[PV_STEP];
};

struct Layout {
  size_t state, basis, r, z, part, sred, hist, checks, dlog, total;
  int ld, kcap, ncols, hist_cap;
};

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static Layout make_layout(int n, int m, int k, int max_iter) {
  Layout L;
  L.ld = (int)align_up((size_t)std::max(n, 1), 64);
  L.kcap = k + 1;
  L.ncols = 2 * L.kcap + m + 1;
  L.hist_cap = max_iter + 2 * L.kcap + 8;
  size_t off = 0;
  L.state = off;
  off = align_up(off + sizeof(State), 256);
  L.basis = off;
  off = align_up(off + (size_t)L.ld * L.ncols * sizeof(double), 256);
  L.r = off;
  off = align_up(off + (size_t)L.ld * sizeof(double), 256);
  L.z = off;
  off = align_up(off + (size_t)L.ld * sizeof(double), 256);
  L.part = off;
  off = align_up(off + (size_t)(PV_MAX + 16 + 2 * KMAX) * GRID_MAX * sizeof(double), 256);
  L.sred = off;
  off = align_up(off + (size_t)2 * GRID_MAX * PV_STEP * sizeof(double), 256);
  L.hist = off;
  off = align_up(off + (size_t)L.hist_cap * sizeof(double), 256);
  L.checks = off;
  off = align_up(off + (size_t)2 * L.hist_cap * sizeof(double), 256);
  L.dlog = off;  // diagnostics: 4 doubles per record, one per deflated cycle + refresh
  off = align_up(off + (size_t)4 * (max_iter + 2) * sizeof(double), 256);
  L.total = off;
  return L;
}

// p.part rows: [0, 16) per-cycle scalar partials, [16, 16 + mm^2) cross-Gram,
// [COMB_PART0, COMB_PART0 + 2 KMAX) next-cycle partials written by k_combine
// (one slot per combine CTA, st->comb_nblk of them). Every cross-CTA sum in
// this file is a fixed-order sum of per-CTA slots: results are bitwise
// reproducible run to run (no floating-point atomics).
constexpr int GRAM_PART0 = 16;
constexpr int COMB_PART0 = GRAM_PART0 + PV_MAX;
// diagnostics partials (k_diag): inside the cross-Gram rows but past the
// refresh projection's rows [0, 2 kc] (still live when the refresh record is taken)
constexpr int DIAG_PART0 = 2 * KMAX + 1;
static_assert(DIAG_PART0 + 1 + KMAX * KMAX <= COMB_PART0, "diagnostics rows");

struct Ptrs {
  int sm_R, sm_B, sm_csr, sm_cmb;  // k_cycle dynamic smem offsets (doubles), cycle_smem_layout
  State* st;
  const int32_t* rp;
  const int32_t* ci;
  const double* av;
  const double* dg;  // Jacobi diagonal or nullptr
  StenView sv;       // optional symmetric 7-diagonal form (sv.hdr == nullptr: none)
  const double* b;
  double* x;
  double* r;
  double* z;
  double* basis;
  double* part;
  double* sred;  // k_cycle per-step partials: [2 buffers][GRID_MAX CTAs][PV_STEP values]
  double* hist;
  double* checks;
  double* dlog;
  int n, ld, kcap, nblk, rpb;
  double v0_rtol;  // |C^T r| / beta above which V_0 is formed from r - C C^T r (V0_PROJ_RTOL)
  int fuse_comb;  // 1: k_cycle applies the recycle update at its start (large row slices);
                  // 0: a separate k_combine launch after every dense update
  int gram_half;  // 1: the DMMA cross-Gram computes What^T U only (What^T V = [0; I])
  int upd_direct;  // k_update: B fragments straight from global memory (no shared tile)
  PcHeader* pch;  // general preconditioner (SOR / ILU0 / IC0 / block Jacobi) or nullptr; with
                  // it dg is nullptr and op(v) = M^-1 (A v) runs as an SpMV phase followed by
                  // the level-scheduled sweeps of precond.cuh
};

__device__ __forceinline__ double* colU(const Ptrs& p, int c) { return p.basis + (size_t)c * p.ld; }
// C block column c in [0, kcap): global column kcap + c; active C = last kc.
__device__ __forceinline__ double* colC(const Ptrs& p, int c) {
  return p.basis + (size_t)(p.kcap + c) * p.ld;
}
__device__ __forceinline__ double* colV(const Ptrs& p, int v) {
  return p.basis + (size_t)(2 * p.kcap + v) * p.ld;
}

// row of A x through the stencil form when it qualified, else the CSR
__device__ __forceinline__ double op_row(const Ptrs& p, bool sten, const double* x, int row) {
  return sten ? sten_row(p.sv, x, row) : csr_row(p.rp, p.ci, p.av, x, row);
}

__device__ __forceinline__ void flag_host(State* st, int cycle, int done) {
  if (st->host_flag) {
    volatile int* hf = st->host_flag;
    hf[1] = done;
    __threadfence_system();
    hf[0] = cycle;
    __threadfence_system();
  }
}

// ---------------------------------------------------------------------------
// setup / init
// ---------------------------------------------------------------------------
__global__ void k_setup(State* st, int n, int ld, int m, int k, int max_iter, double tol,
                        int jacobi, int nblk, int rpb, int k_in, int has_x0, int* host_flag) {
  // zero the scalar header (everything before kept[])
  char* p = reinterpret_cast<char*>(st);
  size_t hdr = offsetof(State, kept);
  for (size_t i = threadIdx.x; i < hdr; i += blockDim.x) p[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    st->n = n;
    st->ld = ld;
    st->m = m;
    st->k = k;
    st->kcap = k + 1;
    st->max_iter = max_iter;
    st->tol = tol;
    st->jacobi = jacobi;
    st->nblk = nblk;
    st->rpb = rpb;
    st->prof[30] = nblk;  // launch shape, reported by skr_gcrodr_profile
    st->prof[31] = rpb;
    st->k_in = k_in;
    st->has_x0 = has_x0;
    st->host_flag = host_flag;
    if (host_flag) {
      host_flag[0] = -1;
      host_flag[1] = 0;
    }
  }
}

// x = x0 or 0; r = M^-1 (b - A x) or M^-1 b; partials: |b|^2, |M^-1 b|^2, |r|^2
__global__ void __launch_bounds__(NT) k_init(Ptrs p, const double* x0) {
  __shared__ double s_red[NW];
  int r0 = blockIdx.x * p.rpb, r1 = min(p.n, r0 + p.rpb);
  double sb = 0.0, sbp = 0.0, sr = 0.0;
  for (int row = r0 + threadIdx.x; row < r1; row += NT) {
    double bv = __ldg(p.b + row);
    double xv = x0 ? x0[row] : 0.0;
    p.x[row] = xv;
    double bp = p.dg ? __ddiv_rn(bv, __ldg(p.dg + row)) : bv;
    sb += bv * bv;
    sbp += bp * bp;
  }
  const bool sten = sten_ok(p.sv);
  for (int row = r0 + threadIdx.x; row < r1; row += NT) {
    double bv = __ldg(p.b + row);
    double rv;
    if (x0) {
      double t = op_row(p, sten, x0, row);
      rv = __dsub_rn(bv, t);
    } else {
      rv = bv;
    }
    if (p.dg) rv = __ddiv_rn(rv, __ldg(p.dg + row));
    p.r[row] = rv;
    sr += rv * rv;
  }
  double t0 = block_sum(sb, s_red);
  double t1 = block_sum(sbp, s_red);
  double t2 = block_sum(sr, s_red);
  if (threadIdx.x == 0) {
    p.part[0 * GRID_MAX + blockIdx.x] = t0;
    p.part[1 * GRID_MAX + blockIdx.x] = t1;
    p.part[2 * GRID_MAX + blockIdx.x] = t2;
  }
  for (int v = threadIdx.x; v < 2 * KMAX; v += NT)
    p.part[(size_t)(COMB_PART0 + v) * GRID_MAX + blockIdx.x] = 0.0;
  if (threadIdx.x == 0) p.st->nb_epoch[blockIdx.x * 16] = 0u;
}

// ---------------------------------------------------------------------------
// generic partial producers for the refresh
// ---------------------------------------------------------------------------
// Gram partials X^T X of nc columns starting at column pointer base (stride
// ld) -> part[(i*nc + j) * GRID_MAX + blk]
__global__ void __launch_bounds__(NT) k_gram(Ptrs p, int which, int ncols_from_state) {
  State* st = p.st;
  if (st->done) return;
  int nc = ncols_from_state == 0 ? st->ncol_a : st->ncol_b;
  if (nc <= 0) return;
  const double* base = which == 0 ? colU(p, 0) : colC(p, p.kcap - nc);
  __shared__ double tile[32][KMAX + 1];
  int r0 = blockIdx.x * p.rpb, r1 = min(p.n, r0 + p.rpb);
  int ne = nc * nc;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // ne <= 1024 = 4 * NT
  for (int t0 = r0; t0 < r1; t0 += 32) {
    for (int e = threadIdx.x; e < 32 * nc; e += NT) {
      int rr = e % 32, c = e / 32;
      int row = t0 + rr;
      tile[rr][c] = row < r1 ? base[(size_t)c * p.ld + row] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int e = threadIdx.x + q * NT;
      if (e < ne) {
        int i = e % nc, j = e / nc;
        double s = 0.0;
        for (int rr = 0; rr < 32; ++rr) s += tile[rr][i] * tile[rr][j];
        acc[q] += s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int e = threadIdx.x + q * NT;
    if (e < ne) p.part[(size_t)e * GRID_MAX + blockIdx.x] = acc[q];
  }
}

// The same Gram partials on the fp64 tensor cores (the refresh runs four of
// them per system): every warp owns 32-row tiles, loads the DMMA fragments
// straight from global memory (lane (ln, lk): column 8 b + ln, row 4 ks + lk;
// the A fragment of column block bi is the B fragment of block bi), half a
// tile ahead in registers, and accumulates the upper block triangle; no block
// barrier inside the sweep. Warps are added in a fixed order at the end.
__global__ void __launch_bounds__(NT, 2) k_gram_dmma(Ptrs p, int which, int ncols_from_state) {
  State* st = p.st;
  if (st->done) return;
  const int nc = ncols_from_state == 0 ? st->ncol_a : st->ncol_b;
  if (nc <= 0) return;
  const double* base = which == 0 ? colU(p, 0) : colC(p, p.kcap - nc);
  __shared__ double sg[KMAX * KMAX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ln = lane >> 2, lk = lane & 3;
  const int r0 = blockIdx.x * p.rpb, r1 = min(p.n, r0 + p.rpb);
  const int nb = (nc + 7) >> 3;  // <= 4 column blocks
  constexpr int NB = KMAX / 8, HS = 4;  // k-steps (4 rows each) per half tile
  const double* colp[NB];
  bool cin[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    cin[b] = 8 * b + ln < nc;
    colp[b] = base + (size_t)min(8 * b + ln, nc - 1) * p.ld + lk;
  }
  double acc[NB][NB][2];
#pragma unroll
  for (int x = 0; x < NB; ++x)
#pragma unroll
    for (int y = 0; y < NB; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  double cur[HS][NB], nxt[HS][NB];
  auto load_half = [&](double (&dst)[HS][NB], int row0) {
#pragma unroll
    for (int ks = 0; ks < HS; ++ks) {
      const int row = row0 + 4 * ks + lk;
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (b < nb) dst[ks][b] = (cin[b] && row < r1) ? colp[b][row0 + 4 * ks] : 0.0;
    }
  };
  // this warp's half tiles: rows r0 + 16 h, h = warp, warp + NW, ...
  const int nh = (r1 - r0 + 15) >> 4;
  if (warp < nh) load_half(nxt, r0 + 16 * warp);
  for (int h = warp; h < nh; h += NW) {
#pragma unroll
    for (int ks = 0; ks < HS; ++ks)
#pragma unroll
      for (int b = 0; b < NB; ++b) cur[ks][b] = nxt[ks][b];
    if (h + NW < nh) load_half(nxt, r0 + 16 * (h + NW));
#pragma unroll
    for (int ks = 0; ks < HS; ++ks)
#pragma unroll
      for (int x = 0; x < NB; ++x)
#pragma unroll
        for (int y = 0; y < NB; ++y)
          if (x <= y && y < nb)
            asm volatile(
                "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc[x][y][0]), "+d"(acc[x][y][1])
                : "d"(cur[ks][x]), "d"(cur[ks][y]));
  }
  for (int e = tid; e < KMAX * KMAX; e += NT) sg[e] = 0.0;
  __syncthreads();
  for (int q = 0; q < NW; ++q) {  // warps in order: a fixed summation order
    if (warp == q)
#pragma unroll
      for (int x = 0; x < NB; ++x)
#pragma unroll
        for (int y = 0; y < NB; ++y)
          if (x <= y && y < nb) {
            // D[m = ln][n = 2 lk + e] of block (x, y)
            const int i = 8 * x + ln, j = 8 * y + 2 * lk;
            sg[i + j * KMAX] += acc[x][y][0];
            sg[i + (j + 1) * KMAX] += acc[x][y][1];
          }
    __syncthreads();
  }
  for (int e = tid; e < nc * nc; e += NT) {
    const int i = e % nc, j = e / nc;
    // blocks below the diagonal were not computed: mirror (the Gram is symmetric)
    const bool upper = (i >> 3) <= (j >> 3);
    p.part[(size_t)e * GRID_MAX + blockIdx.x] = upper ? sg[i + j * KMAX] : sg[j + i * KMAX];
  }
}

// C^T r partials (kc values) for the projection after the refresh
__global__ void __launch_bounds__(NT) k_ctr(Ptrs p) {
  State* st = p.st;
  if (st->done || st->kc == 0) return;
  int kc = st->kc;
  __shared__ double s_red[NW];
  int r0 = blockIdx.x * p.rpb, r1 = min(p.n, r0 + p.rpb);
  for (int c = 0; c < kc; ++c) {
    const double* C = colC(p, p.kcap - kc + c);
    double s = 0.0;
    for (int row = r0 + threadIdx.x; row < r1; row += NT) s += C[row] * p.r[row];
    double t = block_sum(s, s_red);
    if (threadIdx.x == 0) p.part[(size_t)c * GRID_MAX + blockIdx.x] = t;
  }
}

// Deterministic reduction of nv partial values into dst (state arrays).
__global__ void __launch_bounds__(NT) k_reduce(Ptrs p, int nv_from, int dst) {
  State* st = p.st;
  if (st->done) return;
  int nv;
  double* out;
  switch (nv_from) {
    case 0: nv = st->ncol_a * st->ncol_a; out = st->gram; break;       // gram of U block
    case 1: nv = st->ncol_b * st->ncol_b; out = st->gram; break;       // gram of C block
    default: nv = st->kc; out = st->alpha; break;                      // C^T r
  }
  (void)dst;
  if (nv <= 0) return;
  int lane = threadIdx.x & 31;
  int gw = (blockIdx.x * NT + threadIdx.x) >> 5;
  int nwt = (gridDim.x * NT) >> 5;
  for (int v = gw; v < nv; v += nwt) {
    const double* q = p.part + (size_t)v * GRID_MAX;
    double s = 0.0;
    for (int b = lane; b < p.nblk; b += 32) s += q[b];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (nv_from <= 1) {
        int nc = (nv_from == 0) ? st->ncol_a : st->ncol_b;
        out[(v % nc) + (v / nc) * LDK] = s;
      } else {
        out[v] = s;
      }
    }
  }
}

// W = op(Yo): C block (last r columns) <- M^-1 A U[:, :r]
__global__ void __launch_bounds__(NT) k_spmm(Ptrs p) {
  State* st = p.st;
  if (st->done) return;
  int r = st->ncol_a;
  if (r <= 0) return;
  int r0 = blockIdx.x * p.rpb, r1 = min(p.n, r0 + p.rpb);
  const bool sten = sten_ok(p.sv);
  for (int row = r0 + threadIdx.x; row < r1; row += NT) {
    int s = sten ? 0 : __ldg(p.rp + row), e = sten ? 0 : __ldg(p.rp + row + 1);
    double d = p.dg ? __ldg(p.dg + row) : 1.0;
    for (int c = 0; c < r; ++c) {
      const double* Y = colU(p, c);
      double acc = 0.0;
      if (sten)
        acc = sten_row(p.sv, Y, row);
      else
        for (int q = s; q < e; ++q) acc = __dadd_rn(acc, __dmul_rn(__ldg(p.av + q), Y[__ldg(p.ci + q)]));
      if (p.dg) acc = __ddiv_rn(acc, d);
      colC(p, p.kcap - r + c)[row] = acc;
    }
  }
}

// x += U alpha ; r -= C alpha ; partials: C^T r_new (kc), |U_c|^2 (kc), |r_new|^2
__global__ void __launch_bounds__(NT) k_project(Ptrs p) {
  State* st = p.st;
  if (st->done || st->kc == 0) return;
  int kc = st->kc;
  __shared__ double s_al[KMAX];
  __shared__ double s_red[NW];
  if (threadIdx.x < kc) s_al[threadIdx.x] = st->alpha[threadIdx.x];
  __syncthreads();
  int r0 = blockIdx.x * p.rpb, r1 = min(p.n, r0 + p.rpb);
  double rr = 0.0;
  for (int row = r0 + threadIdx.x; row < r1; row += NT) {
    double ua = 0.0, ca = 0.0;
    for (int c = 0; c < kc; ++c) {
      ua += colU(p, c)[row] * s_al[c];
      ca += colC(p, p.kcap - kc + c)[row] * s_al[c];
    }
    p.x[row] = p.x[row] + ua;
    double rv = p.r[row] - ca;
    p.r[row] = rv;
    rr += rv * rv;
  }
  __syncthreads();
  for (int c = 0; c < kc; ++c) {
    const double* C = colC(p, p.kcap - kc + c);
    const double* U = colU(p, c);
    double s1 = 0.0, s2 = 0.0;
    for (int row = r0 + threadIdx.x; row < r1; row += NT) {
      s1 += C[row] * p.r[row];
      double u = U[row];
      s2 += u * u;
    }
    double t1 = block_sum(s1, s_red);
    double t2 = block_sum(s2, s_red);
    if (threadIdx.x == 0) {
      p.part[(size_t)c * GRID_MAX + blockIdx.x] = t1;
      p.part[(size_t)(kc + c) * GRID_MAX + blockIdx.x] = t2;
    }
  }
  double t = block_sum(rr, s_red);
  if (threadIdx.x == 0) p.part[(size_t)(2 * kc) * GRID_MAX + blockIdx.x] = t;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->comb_part = 0;
}


// ---------------------------------------------------------------------------
// general preconditioner outside the cycle kernel (cooperative, nblk CTAs, the
// solve's own barrier words): M^-1 applied in place to
//   target 0  r (and M^-1 b into z when x0 is given), then the |M^-1 b|^2 and
//             |r|^2 partials k_init left unpreconditioned (gcrodr.py:348-351)
//   target 1  W = op(Yo): the C block columns k_spmm wrote (gcrodr.py:96)
//   target 2  op(U) into the V block for the diagnostics record (gcrodr.py:116-123)
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool diag_skip(const State* st, int stage);
__global__ void __launch_bounds__(NT) k_pc_cols(Ptrs p, int target, int stage) {
  State* st = p.st;
  __shared__ PcView s_pc;
  __shared__ int s_flag;
  __shared__ double s_red[NW];
  const int tid = threadIdx.x, blk = blockIdx.x;
  if (tid == 0) s_pc = p.pch->v;
  __syncthreads();
  unsigned long long seen =
      tid == 0 ? ld_relaxed_gpu64(&st->bar_count) / (unsigned long long)p.nblk : 0ull;
  auto sync = [&]() -> bool {
    return grid_sync(&st->bar_count, &st->abort_flag, p.nblk, &s_flag, seen);
  };
  auto fail = [&]() {
    if (tid == 0) {
      st->done = 1;
      if (blk == 0) flag_host(st, -1, 1);
    }
  };
  const int r0 = blk * p.rpb, r1 = min(p.n, r0 + p.rpb);
  if (target == 0) {
    const bool hx = st->has_x0 != 0;
    if (hx) {
      for (int row = r0 + tid; row < r1; row += NT) p.z[row] = __ldg(p.b + row);
      if (!sync()) return fail();
      if (!pc_apply_grid(s_pc, p.z, 1, 0, sync)) return fail();
    }
    if (!pc_apply_grid(s_pc, p.r, 1, 0, sync)) return fail();
    double sr = 0.0, sbp = 0.0;
    for (int row = r0 + tid; row < r1; row += NT) {
      const double rv = p.r[row], bp = hx ? p.z[row] : rv;
      sr += rv * rv;
      sbp += bp * bp;
    }
    const double t1 = block_sum(sbp, s_red);
    const double t2 = block_sum(sr, s_red);
    if (tid == 0) {
      p.part[1 * GRID_MAX + blk] = t1;
      p.part[2 * GRID_MAX + blk] = t2;
    }
  } else if (target == 1) {
    const int r = st->ncol_a;
    if (st->done || r <= 0) return;
    if (!pc_apply_grid(s_pc, colC(p, p.kcap - r), r, p.ld, sync)) return fail();
  } else {
    if (diag_skip(st, stage)) return;
    const int kc = st->kc;
    const bool sten = sten_ok(p.sv);
    for (int row = r0 + tid; row < r1; row += NT)
      for (int q = 0; q < kc; ++q) colV(p, q)[row] = op_row(p, sten, colU(p, q), row);
    if (!sync()) return fail();
    if (!pc_apply_grid(s_pc, colV(p, 0), kc, p.ld, sync)) return fail();
  }
}

// true residual partials |b - A x|^2
__global__ void __launch_bounds__(NT) k_final_resid(Ptrs p) {
  __shared__ double s_red[NW];
  int r0 = blockIdx.x * p.rpb, r1 = min(p.n, r0 + p.rpb);
  double s = 0.0;
  const bool sten = sten_ok(p.sv);
  for (int row = r0 + threadIdx.x; row < r1; row += NT) {
    double t = __dsub_rn(__ldg(p.b + row), op_row(p, sten, p.x, row));
    s += t * t;
  }
  double t = block_sum(s, s_red);
  if (threadIdx.x == 0) p.part[blockIdx.x] = t;
}

// ---------------------------------------------------------------------------
// combine: row-parallel small-coefficient update of U / C, in place
// ---------------------------------------------------------------------------
template <int KT>
__global__ void __launch_bounds__(NT, 2) k_combine(Ptrs p, int cycle_mode) {
  State* st = p.st;
  if (cycle_mode) {
    // fused mode: only the last cycle's update when no k_cycle launch applied
    // it (k_cycle clears the flag after applying it; k_setup resets it);
    // otherwise after every dense update that followed a cycle
    if (p.fuse_comb ? !st->comb_pending : !st->ran) return;
  } else if (st->done) {
    return;
  }
  extern __shared__ double sm[];
  int mode = cycle_mode ? CM_CYCLE : st->cm_mode;
  int nin_u, nin_c, nv, nout_u, nout_c;
  const double* cu;
  const double* cc;
  int ldcu, ldcc;
  if (mode == CM_CYCLE) {
    nin_u = st->kc_prev;
    nin_c = st->kc_prev;
    nv = st->j;  // U uses V_0..V_{j-1}; C uses V_0..V_j
    nout_u = st->upd ? st->k_new : 0;
    nout_c = nout_u;
    cu = st->coefU;
    cc = st->coefC;
    ldcu = LDC;
    ldcc = LDC;
  } else {
    nin_u = st->cm_nin_u;
    nin_c = st->cm_nin_c;
    nv = 0;
    nout_u = st->cm_nout_u;
    nout_c = st->cm_nout_c;
    cu = st->coefU;
    cc = st->coefC;
    ldcu = LDC;
    ldcc = LDC;
  }
  int rows_u = nin_u + nv, rows_c = nin_c + (mode == CM_CYCLE ? nv + 1 : 0);
  double* s_cu = sm;                       // rows_u x nout_u
  double* s_cc = sm + (size_t)LDC * KT;    // rows_c x nout_c
  __shared__ double s_red[NW];
  for (int e = threadIdx.x; e < rows_u * nout_u; e += NT)
    s_cu[(e % rows_u) + (e / rows_u) * LDC] = cu[(e % rows_u) + (e / rows_u) * ldcu];
  for (int e = threadIdx.x; e < rows_c * nout_c; e += NT)
    s_cc[(e % rows_c) + (e / rows_c) * LDC] = cc[(e % rows_c) + (e / rows_c) * ldcc];
  __syncthreads();
  // own row split: the grid is not tied to the cooperative kernel's slices
  const int rpc = (((p.n + gridDim.x - 1) / gridDim.x) + 31) & ~31;
  int r0 = blockIdx.x * rpc, r1 = min(p.n, r0 + rpc);
  int cbase_in = p.kcap - nin_c;
  int cbase_out = p.kcap - nout_c;
  for (int row = r0 + threadIdx.x; row < r1; row += NT) {
    double au[KT], ac[KT];
#pragma unroll
    for (int q = 0; q < KT; ++q) {
      au[q] = 0.0;
      ac[q] = 0.0;
    }
    // input columns in batches of 8 loads (issued before the FMAs)
    constexpr int LB = KT >= 24 ? 4 : 8;
    if (nout_u > 0)
      for (int c0 = 0; c0 < nin_u; c0 += LB) {
        double v[LB];
#pragma unroll
        for (int u = 0; u < LB; ++u) v[u] = c0 + u < nin_u ? colU(p, c0 + u)[row] : 0.0;
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int c = min(c0 + u, nin_u - 1);
#pragma unroll
          for (int q = 0; q < KT; ++q)
            if (q < nout_u) au[q] += v[u] * s_cu[c + q * LDC];
        }
      }
    if (nout_c > 0)
      for (int c0 = 0; c0 < nin_c; c0 += LB) {
        double v[LB];
#pragma unroll
        for (int u = 0; u < LB; ++u)
          v[u] = c0 + u < nin_c ? colC(p, cbase_in + c0 + u)[row] : 0.0;
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int c = min(c0 + u, nin_c - 1);
#pragma unroll
          for (int q = 0; q < KT; ++q)
            if (q < nout_c) ac[q] += v[u] * s_cc[c + q * LDC];
        }
      }
    if (mode == CM_CYCLE && (nout_u > 0 || nout_c > 0)) {
      for (int v0 = 0; v0 <= nv; v0 += LB) {
        double x[LB];
#pragma unroll
        for (int u = 0; u < LB; ++u) x[u] = v0 + u <= nv ? colV(p, v0 + u)[row] : 0.0;
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int v = min(v0 + u, nv);
          if (v < nv)
#pragma unroll
            for (int q = 0; q < KT; ++q)
              if (q < nout_u) au[q] += x[u] * s_cu[nin_u + v + q * LDC];
#pragma unroll
          for (int q = 0; q < KT; ++q)
            if (q < nout_c) ac[q] += x[u] * s_cc[nin_c + v + q * LDC];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < KT; ++q) {
      if (q < nout_u) colU(p, q)[row] = au[q];
      if (q < nout_c) colC(p, cbase_out + q)[row] = ac[q];
    }
  }
  if (mode == CM_CYCLE && !st->done) {
    // partials for the next cycle start: C^T r (kc) and |U_c|^2 (kc)
    int kc = st->kc;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->comb_part = 1;
      st->comb_nblk = gridDim.x;
    }
    __syncthreads();
    for (int c = 0; c < kc; ++c) {
      const double* C = colC(p, p.kcap - kc + c);
      const double* U = colU(p, c);
      double s1 = 0.0, s2 = 0.0;
      for (int row = r0 + threadIdx.x; row < r1; row += NT) {
        s1 += C[row] * p.r[row];
        double u = U[row];
        s2 += u * u;
      }
      double t1 = block_sum(s1, s_red);
      double t2 = block_sum(s2, s_red);
      if (threadIdx.x == 0) {  // this CTA's slot of the COMB_PART0 rows
        p.part[(size_t)(COMB_PART0 + c) * GRID_MAX + blockIdx.x] = t1;
        p.part[(size_t)(COMB_PART0 + kc + c) * GRID_MAX + blockIdx.x] = t2;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// the persistent Arnoldi-cycle kernel
// ---------------------------------------------------------------------------
constexpr int PVC = KMAX + MMAX;  // basis columns, upper bound

struct CycleSmem {
  double red[PV_STEP];
  double a[KMAX + MMAX];     // reorthogonalisation coefficients of the pending vector
  double bb[KMAX + MMAX];    // first-pass coefficients of the new vector (scaled)
  double cs[MMAX], sn[MMAX], gv[MMAX + 1];
  double hp[MMAX + 1];       // first-pass H column of the pending vector
  double bp[KMAX];           // first-pass B column
  double dk[KMAX], cr[KMAX];
  double y[KMAX + MMAX];
  double hcol[MMAX + 2];     // column being finalised (Givens in place)
  double sc[16];             // scalars
  double bred[3 * NW];
  int flag;
  unsigned ep;  // neighbour-epoch target of the current step
};


// Warp reduce-scatter of NV values per lane (butterfly: NV - 1 + 5 - log2 NV
// shuffles). Returns the warp sum of v[(lane >> (5 - log2 NV)) & (NV - 1)];
// the 32 / NV lanes of a group hold the same value.
template <int NV>
__device__ __forceinline__ double bfly(double (&v)[NV], int lane) {
  const unsigned F = 0xffffffffu;
  int off = 16;
#pragma unroll
  for (int h = NV / 2; h >= 1; h /= 2, off /= 2) {
    const bool hi = lane & off;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      double send = hi ? v[k] : v[k + h], keep = hi ? v[k + h] : v[k];
      v[k] = keep + __shfl_xor_sync(F, send, off);
    }
  }
  double r = v[0];
#pragma unroll
  for (; off >= 1; off /= 2) r += __shfl_xor_sync(F, r, off);
  return r;
}
template <int NV>
__host__ __device__ constexpr int log2c() { return NV <= 1 ? 0 : 1 + log2c<NV / 2>(); }

// z_i = (A x)[row_i] for R rows per lane, every row summed sequentially in
// CSR order with round-to-nearest mul/add (bit-exact with scipy csr_matvec);
// the R rows' loads are interleaved for memory-level parallelism. LOCAL: the
// CTA's CSR slice is in shared memory (rp rebased to r0).
template <int R, bool LOCAL>
__device__ __forceinline__ void spmv_rows(const int* rp, const int* ci, const double* av,
                                          const double* xv, const int (&row)[R],
                                          const bool (&ok)[R], int r0, double (&z)[R]) {
  int a0[R], len[R];
  int lm = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int rr = LOCAL ? row[i] - r0 : row[i];
    const int b0 = LOCAL ? rp[rr] : __ldg(rp + rr);
    const int b1 = LOCAL ? rp[rr + 1] : __ldg(rp + rr + 1);
    a0[i] = b0;
    len[i] = ok[i] ? b1 - b0 : 0;
    lm = max(lm, len[i]);
    z[i] = 0.0;
  }
  for (int q = 0; q < lm; ++q) {
    double a[R], x[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (q < len[i]) {
        const int e = a0[i] + q;
        a[i] = LOCAL ? av[e] : __ldg(av + e);
        x[i] = xv[LOCAL ? ci[e] : __ldg(ci + e)];
      }
    }
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (q < len[i]) z[i] = __dadd_rn(z[i], __dmul_rn(a[i], x[i]));
  }
}

#define CPROF(idx)                                                \
  do {                                                            \
    if (blk == 0 && tid == 0) {                                   \
      long long _t = clock64();                                   \
      st->prof[16 + (idx)] += _t - cprof_t;                       \
      cprof_t = _t;                                               \
    }                                                             \
  } while (0)

#define CYCLE_SYNC()                                              \
  do {                                                            \
    if (!grid_sync(bc, abt, nblk, &S.flag, bar_seen)) {           \
      if (tid == 0) {                                             \
        st->done = 1;                                             \
        if (blk == 0) flag_host(st, cycle_id, 1);                 \
      }                                                           \
      return;                                                     \
    }                                                             \
  } while (0)

// |C^T r| / beta above which the cycle forms V_0 from r - C C^T r (cycle start)
constexpr double V0_PROJ_RTOL = 1e-12;

#ifndef SKR_SW1_PREFETCH
#define SKR_SW1_PREFETCH 0  // measured: the 16 extra live registers spill into sweep 2 (C3 -27%)
#endif
constexpr bool SW1_PREFETCH = SKR_SW1_PREFETCH != 0;  // sweep 1: first basis batch ahead of the SpMV
constexpr int GT_LD = 33;  // padded rows per staged Gram column (odd: conflict-free)
constexpr int FUSE_COMB_ROWS = 4096;  // rows per CTA from which k_cycle applies the update
constexpr int GM_MMAX = 40;  // Arnoldi length up to which the cycle end uses the DMMA Gram
constexpr int GM_LD = 36;  // the same for the DMMA Gram (== 4 mod 16: conflict-free fragments)

// k_cycle dynamic shared memory, sized by (m, kcap) (offsets in doubles):
// [ Gram tile (2 kcap + m + 1 cols x GT_LD; aliased by the sweep-1 partials)
//   | packed R (m (m+1)/2) | B (kcap x m) | optional CSR slice cache ]
struct CycleSmemLayout {
  size_t R, B, csr, cmb;
};
// leading dimension of the transposed recycle-update coefficients staged for
// the DMMA combine: >= m + 1 inputs rounded to the k-step, and == 4 or 12
// (mod 16) doubles so a half-warp's A fragments (4 outputs x 4 inputs) fall
// on distinct bank pairs
__host__ __device__ inline int comb_ld(int m) {
  const int need = (m + 4) & ~3;
  return need <= 44 ? 44 : need <= 52 ? 52 : need <= 60 ? 60 : 68;
}
inline CycleSmemLayout cycle_smem_layout(int m, int kcap) {
  CycleSmemLayout L;
  size_t gt = (size_t)(2 * kcap + m + 1) * GM_LD + NT;  // + the x-update scratch
  if (gt < (size_t)NW * 2 * PVC) gt = (size_t)NW * 2 * PVC;
  // the cycle-start recycle update stages (2 kcap + m + 2) columns and then
  // the two coefficient blocks; at that point the R and B areas are free, so
  // the combine may run into them
  const size_t kb = (size_t)((kcap + 7) / 8) * 8;
  L.cmb = (size_t)(2 * kcap + m + 2) * GM_LD;
  const size_t cmb_end = L.cmb + 2 * kb * (size_t)comb_ld(m);
  const size_t rb = (size_t)m * (m + 1) / 2 + (size_t)kcap * m;
  if (gt + rb < cmb_end) gt = cmb_end - rb;
  // the cycle-end DMMA pass (m <= GM_MMAX) streams its tiles through two
  // stages [0, gs) and [gs + NT, 2 gs + NT) around the x-update scratch; the
  // second stage may run into R and B (dead at the cycle end), so at C3 the
  // ring fits in the footprint the cycle-start update needs anyway (shared
  // memory, and with it L1 -- which sweep 2 depends on -- is unchanged)
  if (m <= GM_MMAX) {
    const size_t gs = (size_t)(kcap + m + 1) * GM_LD;
    if (gt + rb < 2 * gs + NT) gt = 2 * gs + NT - rb;
  }
  L.R = gt;
  L.B = L.R + (size_t)m * (m + 1) / 2;
  L.csr = (L.B + (size_t)kcap * m + 1) & ~(size_t)1;  // 16-byte aligned
  return L;
}
// dynamic smem per CTA that keeps 2 CTAs (+ ~7.6 KB static each) on an SM
#ifndef SKR_CYCLE_DSMEM_KB
#define SKR_CYCLE_DSMEM_KB 96
#endif
constexpr size_t CYCLE_DSMEM_BUDGET = SKR_CYCLE_DSMEM_KB * 1024;

// The recycle update of a finished cycle (gcrodr.py:444-467), in place, over this
// CTA's rows [blockIdx.x * rpb, ...): U <- [U | V_0..V_{j-1}] coefU, C <- [C | V_0..V_j]
// coefC (coefficients of the dense kernel's P_CYCLE), on the fp64 tensor cores:
// DMMA m8n8k4 with A = coef^T (outputs x inputs) and B = the staged 32-row tile
// (inputs x rows), so no output padding beyond 8 columns is wasted. With
// `partials`, the next cycle start's per-CTA sums C^T r and |U_c|^2 are formed from
// the new columns in the same pass. Called from k_cycle (fused) or k_update.
__device__ __forceinline__ void recycle_update_dmma(const Ptrs& p, double* cdyn, double* bred,
                                                    bool partials) {
  State* st = p.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, blk = blockIdx.x;
  const int kcap = p.kcap, m = st->m;
  const int r0 = blk * p.rpb, r1 = min(p.n, r0 + p.rpb);
  const int kcp = st->kc_prev, jj = st->j;
  const int nout = st->upd ? st->k_new : 0;
  double* part0 = p.part + (size_t)COMB_PART0 * GRID_MAX + blk;
  if (nout == 0) {  // no update: the next cycle's partials from U, C as they are
    if (!partials) return;
    for (int c = 0; c < kcp; ++c) {
      const double* Cc = colC(p, kcap - kcp + c);
      const double* Uc = colU(p, c);
      double s1 = 0.0, s2 = 0.0;
      for (int row = r0 + tid; row < r1; row += NT) {
        s1 += Cc[row] * p.r[row];
        const double u = Uc[row];
        s2 += u * u;
      }
      const double t1 = block_sum(s1, bred);
      const double t2 = block_sum(s2, bred);
      if (tid == 0) {
        part0[(size_t)c * GRID_MAX] = t1;
        part0[(size_t)(kcp + c) * GRID_MAX] = t2;
      }
    }
    return;
  }
  const int nin_u = kcp + jj, nin_c = kcp + jj + 1;
  const int ncs = 2 * kcp + jj + 1;  // staged [U (kcp) | C (kcp) | V_0..V_jj], then r
  const int cld = comb_ld(m);
  const int kbn = ((nout + 7) >> 3) * 8, nmb = kbn >> 3;  // padded outputs, <= 4 blocks
  double* stg = cdyn;
  double* cfs = cdyn + p.sm_cmb;
  for (int e = tid; e < 2 * kbn * cld; e += NT) {  // cfs[(h kbn + q) cld + i] = coef_h[i][q]
    const int i = e % cld, q = (e / cld) % kbn, h = e / (cld * kbn);
    cfs[e] = (q < nout && i < (h ? nin_c : nin_u)) ? (h ? st->coefC : st->coefU)[i + q * LDC]
                                                   : 0.0;
  }
  // warp: outputs of U (uc 0) or C (uc 1), rows 8 nbr .. 8 nbr + 7 of a tile
  const int uc = warp >> 2, nbr = warp & 3, ln = lane >> 2, lk = lane & 3;
  const int nin = uc ? nin_c : nin_u, nks = (nin + 3) >> 2;
  const double* cf = cfs + (size_t)(uc * kbn + ln) * cld + lk;  // A: coef^T[8 mb + ln][4 ks + lk]
  auto scol = [&](int i) -> int {  // staged column of input i (padding clamped)
    i = min(i, nin - 1);
    return i < kcp ? (uc ? kcp + i : i) : 2 * kcp + (i - kcp);
  };
  // staged column c lives at basis column c (U) or c + 2 (kcap - kcp) (the
  // right-aligned C block and V follow each other); column ncs is r
  auto src_col = [&](int c) -> const double* {
    return c >= ncs ? p.r : p.basis + (size_t)(c < kcp ? c : c + 2 * (kcap - kcp)) * p.ld;
  };
  // a thread stages row pairs (16-byte loads and shared stores) of the columns
  // (tid >> 4) + 16 k: pointers fixed for the whole pass, the next two
  // tiles' elements in flight in registers
  constexpr int GPF = 4;
  double2 pf[GPF], pf2[GPF];
  const int prr = 2 * (tid & 15), pc0 = tid >> 4;
  auto load_tile = [&](double2 (&dst)[GPF], int t0) {
    const int row = t0 + prr;
#pragma unroll
    for (int k = 0; k < GPF; ++k) {
      const int c = pc0 + 16 * k;
      if (c > ncs) continue;
      const double* q = src_col(c) + row;
      if (row + 1 < r1)
        dst[k] = *reinterpret_cast<const double2*>(q);
      else
        dst[k] = make_double2(row < r1 ? q[0] : 0.0, 0.0);
    }
  };
  double psq[4] = {0.0, 0.0, 0.0, 0.0};  // |U_q|^2 (uc 0) or C_q . r (uc 1), this lane's rows
  if (r0 < r1) load_tile(pf, r0);
  if (r0 + 32 < r1) load_tile(pf2, r0 + 32);
  for (int t0 = r0; t0 < r1; t0 += 32) {
    __syncthreads();  // the previous tile (and the coefficients) are in place / consumed
#pragma unroll
    for (int k = 0; k < GPF; ++k)
      if (pc0 + 16 * k <= ncs)
        *reinterpret_cast<double2*>(stg + (pc0 + 16 * k) * GM_LD + prr) = pf[k];
    for (int e = tid + 32 * 16 * GPF; e < 32 * (ncs + 1); e += NT) {  // columns past 64 (m > 40)
      const int row = t0 + (e & 31);
      stg[(e >> 5) * GM_LD + (e & 31)] = row < r1 ? src_col(e >> 5)[row] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < GPF; ++k) pf[k] = pf2[k];
    if (t0 + 64 < r1) load_tile(pf2, t0 + 64);
    double acc[4][2];
#pragma unroll
    for (int mb = 0; mb < 4; ++mb) acc[mb][0] = acc[mb][1] = 0.0;
    for (int ks = 0; ks < nks; ++ks) {
      const double bf = stg[scol(4 * ks + lk) * GM_LD + 8 * nbr + ln];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb)
        if (mb < nmb)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(acc[mb][0]), "+d"(acc[mb][1])
              : "d"(cf[(size_t)mb * 8 * cld + 4 * ks]), "d"(bf));
    }
    // D[output 8 mb + ln][row 8 nbr + 2 lk + e]
    const int rl = 8 * nbr + 2 * lk, row = t0 + rl;
#pragma unroll
    for (int mb = 0; mb < 4; ++mb) {
      const int q = 8 * mb + ln;
      if (mb < nmb && q < nout) {
        double* dst = uc ? colC(p, kcap - nout + q) : colU(p, q);
        if (row + 1 < r1)
          *reinterpret_cast<double2*>(dst + row) = make_double2(acc[mb][0], acc[mb][1]);
        else if (row < r1)
          dst[row] = acc[mb][0];
        if (partials) {
          if (uc)
            psq[mb] += acc[mb][0] * stg[ncs * GM_LD + rl] + acc[mb][1] * stg[ncs * GM_LD + rl + 1];
          else
            psq[mb] += acc[mb][0] * acc[mb][0] + acc[mb][1] * acc[mb][1];
        }
      }
    }
  }
  if (partials) {  // lanes of an output, then the 4 row-block warps, in a fixed order
#pragma unroll
    for (int mb = 0; mb < 4; ++mb) {
      psq[mb] += __shfl_xor_sync(0xffffffffu, psq[mb], 1);
      psq[mb] += __shfl_xor_sync(0xffffffffu, psq[mb], 2);
    }
    __syncthreads();
    double* red = stg;
    if (lk == 0)
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) red[(uc * 4 + nbr) * 32 + 8 * mb + ln] = psq[mb];
    __syncthreads();
    for (int e = tid; e < 2 * nout; e += NT) {
      const int h = e / nout, q = e % nout;  // h 1: C^T r, h 0: |U|^2
      const double* rq = red + h * 4 * 32 + q;
      part0[(size_t)(h ? q : nout + q) * GRID_MAX] = ((rq[0] + rq[32]) + rq[64]) + rq[96];
    }
  }
  __syncthreads();
}

// The update without the shared-memory tile (k_update): every warp loads its
// own B fragments straight from the basis (lane (ln, lk): input column
// 4 ks + lk, row 8 nbr + ln of the tile: four 64-byte pieces per load, every
// sector used), one tile ahead in registers, so the warps never meet at a
// block barrier and one warp's DMMAs overlap the others' loads. Rows are owned
// by a warp (block nbr of 8 rows, U or C outputs), the in-place update needs
// no ordering between warps. NKS: k-steps (4 inputs each) compiled in.
template <int NKS>
__device__ __forceinline__ void recycle_update_direct(const Ptrs& p, double* cdyn, double* bred,
                                                      bool partials) {
  State* st = p.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, blk = blockIdx.x;
  const int kcap = p.kcap, m = st->m;
  const int r0 = blk * p.rpb, r1 = min(p.n, r0 + p.rpb);
  const int kcp = st->kc_prev, jj = st->j;
  const int nout = st->upd ? st->k_new : 0;
  double* part0 = p.part + (size_t)COMB_PART0 * GRID_MAX + blk;
  const int nin_u = kcp + jj, nin_c = kcp + jj + 1;
  const int cld = comb_ld(m);
  const int kbn = ((nout + 7) >> 3) * 8, nmb = kbn >> 3;  // padded outputs, <= 4 blocks
  double* cfs = cdyn;
  for (int e = tid; e < 2 * kbn * cld; e += NT) {  // cfs[(h kbn + q) cld + i] = coef_h[i][q]
    const int i = e % cld, q = (e / cld) % kbn, h = e / (cld * kbn);
    cfs[e] = (q < nout && i < (h ? nin_c : nin_u)) ? (h ? st->coefC : st->coefU)[i + q * LDC]
                                                   : 0.0;
  }
  __syncthreads();
  const int uc = warp >> 2, nbr = warp & 3, ln = lane >> 2, lk = lane & 3;
  const int nin = uc ? nin_c : nin_u, nks = (nin + 3) >> 2;
  const double* cf = cfs + (size_t)(uc * kbn + ln) * cld + lk;  // A: coef^T[8 mb + ln][4 ks + lk]
  // input i of this warp's product: U column i (uc 0, i < kcp), else the
  // contiguous [C | V] range (basis column i + 2 kcap - kcp)
  const size_t ld = p.ld;
  auto in_col = [&](int i) -> const double* {
    i = min(i, nin - 1);
    return p.basis + (size_t)((uc == 0 && i < kcp) ? i : i + 2 * kcap - kcp) * ld;
  };
  const int rb = 8 * nbr + ln;  // B fragment row of the tile
  double bcur[NKS], bnext[NKS];
  auto load_b = [&](double (&dst)[NKS], int t0) {
    const int row = t0 + rb;
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks)
      if (ks < nks) dst[ks] = row < r1 ? in_col(4 * ks + lk)[row] : 0.0;
  };
  double psq[4] = {0.0, 0.0, 0.0, 0.0};  // |U_q|^2 (uc 0) or C_q . r (uc 1), this lane's rows
  if (r0 < r1) load_b(bnext, r0);
  for (int t0 = r0; t0 < r1; t0 += 32) {
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks) bcur[ks] = bnext[ks];
    if (t0 + 32 < r1) load_b(bnext, t0 + 32);
    const int rl = 8 * nbr + 2 * lk, row = t0 + rl;  // D fragment rows
    double2 rv = make_double2(0.0, 0.0);
    if (partials && uc) {
      if (row + 1 < r1)
        rv = *reinterpret_cast<const double2*>(p.r + row);
      else if (row < r1)
        rv.x = p.r[row];
    }
    double acc[4][2];
#pragma unroll
    for (int mb = 0; mb < 4; ++mb) acc[mb][0] = acc[mb][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks)
      if (ks < nks) {
#pragma unroll
        for (int mb = 0; mb < 4; ++mb)
          if (mb < nmb)
            asm volatile(
                "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc[mb][0]), "+d"(acc[mb][1])
                : "d"(cf[(size_t)mb * 8 * cld + 4 * ks]), "d"(bcur[ks]));
      }
    // D[output 8 mb + ln][row 8 nbr + 2 lk + e]
#pragma unroll
    for (int mb = 0; mb < 4; ++mb) {
      const int q = 8 * mb + ln;
      if (mb < nmb && q < nout) {
        double* dst = uc ? colC(p, kcap - nout + q) : colU(p, q);
        if (row + 1 < r1)
          *reinterpret_cast<double2*>(dst + row) = make_double2(acc[mb][0], acc[mb][1]);
        else if (row < r1)
          dst[row] = acc[mb][0];
        if (partials) {
          if (uc)
            psq[mb] += acc[mb][0] * rv.x + acc[mb][1] * rv.y;
          else
            psq[mb] += acc[mb][0] * acc[mb][0] + acc[mb][1] * acc[mb][1];
        }
      }
    }
  }
  if (partials) {  // lanes of an output, then the 4 row-block warps, in a fixed order
#pragma unroll
    for (int mb = 0; mb < 4; ++mb) {
      psq[mb] += __shfl_xor_sync(0xffffffffu, psq[mb], 1);
      psq[mb] += __shfl_xor_sync(0xffffffffu, psq[mb], 2);
    }
    __syncthreads();  // the coefficients are consumed
    double* red = cdyn;
    if (lk == 0)
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) red[(uc * 4 + nbr) * 32 + 8 * mb + ln] = psq[mb];
    __syncthreads();
    for (int e = tid; e < 2 * nout; e += NT) {
      const int h = e / nout, q = e % nout;  // h 1: C^T r, h 0: |U|^2
      const double* rq = red + h * 4 * 32 + q;
      part0[(size_t)(h ? q : nout + q) * GRID_MAX] = ((rq[0] + rq[32]) + rq[64]) + rq[96];
    }
  }
  (void)bred;
}

// The same update as its own launch (host: SKR_FUSE_COMB=2), nblk CTAs (the
// chain's share of the SMs) on the slices of the cycle kernel, with its own
// register allocation; partials in the k_combine protocol (comb_part = 1).
__global__ void __launch_bounds__(NT, 2) k_update(Ptrs p) {
  State* st = p.st;
  if (!st->ran) return;  // nothing ran since the last update (look-ahead launch)
  extern __shared__ double cdyn[];
  __shared__ double bred[3 * NW];
  const bool partials = !st->done;
  const int nout = st->upd ? st->k_new : 0;
  const int nks = (st->kc_prev + st->j + 1 + 3) >> 2;
  if (nout == 0 || p.upd_direct == 0)
    recycle_update_dmma(p, cdyn, bred, partials);  // (also: no update, partials only)
  else if (nks <= 8)
    recycle_update_direct<8>(p, cdyn, bred, partials);
  else if (nks <= 12)
    recycle_update_direct<12>(p, cdyn, bred, partials);
  else
    recycle_update_direct<16>(p, cdyn, bred, partials);
  if (partials && blockIdx.x == 0 && threadIdx.x == 0) {
    st->comb_part = 1;
    st->comb_nblk = gridDim.x;
  }
}

// R = rows per lane in the Arnoldi sweeps: warp-owned tiles of 32 R consecutive
// rows; every lane keeps its rows' w = V_t and z = op(V_t) in registers.
#ifndef SKR_CYCLE_MINB
#define SKR_CYCLE_MINB 2  // CTAs per SM the register allocation must allow
#endif
// GPC: a general preconditioner (p.pch) instead of none / Jacobi: 1 = the
// triangular kinds (SOR, ILU(0), IC(0)), 2 = block Jacobi.
template <int R, int GPC>
__global__ void __launch_bounds__(NT, SKR_CYCLE_MINB) k_cycle(Ptrs p, int cycle_id, int csr_cap) {
  State* st = p.st;
  __shared__ CycleSmem S;
  __shared__ PcView s_pc;
  if (GPC) {
    if (threadIdx.x == 0) s_pc = p.pch->v;
    __syncthreads();
  }
  extern __shared__ double cdyn[];
  // offsets from the host (cycle_smem_layout): kernel parameters, not registers
  double* gtile = cdyn;          // Gram tile, column-major, ld GT_LD
  double* sacc = cdyn;           // aliases gtile (sweep 1 only): per-warp partials [a | bb]
  double* Rsm = cdyn + p.sm_R;   // packed R (Givens-rotated H)
  double* Bsm = cdyn + p.sm_B;   // B, ld kcap
  int* csr_rp = reinterpret_cast<int*>(cdyn + p.sm_csr);  // cached CSR slice (optional)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int blk = blockIdx.x, nblk = p.nblk;
  const int n = p.n;
  const int m = st->m;
  const int kcap = p.kcap;
  const int r0 = blk * p.rpb, r1 = min(n, r0 + p.rpb);
  unsigned long long* bc = &st->bar_count;
  int* abt = &st->abort_flag;
  // completed grid barriers of this solve (no barrier is in flight at launch)
  unsigned long long bar_seen = tid == 0 ? ld_relaxed_gpu64(bc) / (unsigned long long)nblk : 0ull;
  auto cycle_sync = [&]() -> bool { return grid_sync(bc, abt, nblk, &S.flag, bar_seen); };
  auto cycle_abort = [&]() {
    if (tid == 0) {
      st->done = 1;
      if (blk == 0) flag_host(st, cycle_id, 1);
    }
  };

#ifdef SKR_NO_FUSED_UPDATE  // build without the in-kernel update (k_update only): A/B of the register allocation
  auto apply_update = [&](bool) {};
#else
  auto apply_update = [&](bool partials) { recycle_update_dmma(p, cdyn, S.bred, partials); };
#endif
  if (st->done) {
    // the look-ahead launch after the final cycle applies that cycle's update
    // (the next solve's refresh reads U), then leaves
    if (p.fuse_comb && st->comb_pending) {
      apply_update(false);
      if (!grid_sync(bc, abt, nblk, &S.flag, bar_seen)) return;
      if (blk == 0 && tid == 0) st->comb_pending = 0;
    }
    if (blk == 0 && tid == 0) st->ran = 0;
    return;
  }
  const int kc = st->kc;
  const bool defl = kc > 0;
  int budget = st->max_iter - st->iters;
  int s = defl ? max(1, m - kc) : m;
  s = min(s, budget);
  const double abs_tol = st->abs_tol;
  const double beta = st->rnorm;
  double* Qb = colC(p, kcap - kc);  // [C | V_0 ...] contiguous
  constexpr int TR = 32 * R;
  constexpr int CB = R >= 4 ? 4 : 8;         // sweep-1 basis columns per butterfly batch
  constexpr int SW2_COLS = R >= 4 ? 4 : 8;   // sweep-2 basis columns per load batch
  const int ntile = r1 > r0 ? (r1 - r0 + TR - 1) / TR : 0;
  // ---- cache this CTA's CSR slice in shared memory when it fits ---------------
  const bool sten = sten_ok(p.sv);
  bool csr_local = false;
  int* lci = nullptr;
  double* lav = nullptr;
  if (!sten && csr_cap > 0 && r1 > r0) {
    const int e0 = __ldg(p.rp + r0), e1 = __ldg(p.rp + r1);
    const int rows = r1 - r0, nz = e1 - e0;
    const size_t off_ci = (size_t)(rows + 1);
    const size_t off_av = ((off_ci + nz) * sizeof(int) + 7) / 8;  // in doubles
    if ((off_av + nz) * sizeof(double) <= (size_t)csr_cap) {
      csr_local = true;
      lci = csr_rp + off_ci;
      lav = reinterpret_cast<double*>(csr_rp) + off_av;
      for (int q = tid; q <= rows; q += NT) csr_rp[q] = __ldg(p.rp + r0 + q) - e0;
      for (int q = tid; q < nz; q += NT) {
        lci[q] = __ldg(p.ci + e0 + q);
        lav[q] = __ldg(p.av + e0 + q);
      }
    }
    __syncthreads();
  }
  // ---- or its slice of the 2-D stencil form: D, W (+1), S (+sx) ------------
  bool sten_local = false;
  const double *lD = nullptr, *lW = nullptr, *lS = nullptr;
  if (sten && !p.sv.sxy && csr_cap > 0 && r1 > r0) {
    const int rows = r1 - r0, sx = p.sv.sx;
    if ((size_t)(3 * rows + 1 + sx) * sizeof(double) <= (size_t)csr_cap) {
      double* c0 = reinterpret_cast<double*>(csr_rp);
      for (int q = tid; q < rows; q += NT) c0[q] = __ldg(p.sv.D + r0 + q);
      for (int q = tid; q <= rows; q += NT) c0[rows + q] = __ldg(p.sv.W + r0 + q);
      for (int q = tid; q < rows + sx; q += NT) c0[2 * rows + 1 + q] = __ldg(p.sv.S + r0 + q);
      lD = c0;
      lW = c0 + rows;
      lS = c0 + 2 * rows + 1;
      sten_local = true;
    }
    __syncthreads();
  }
  auto row_dot = [&](const double* xv, int row) -> double {
    if (sten_local)
      return sten_row_at<false>(lD, lW, lS, nullptr, p.sv.sx, 0, n, xv, row, row - r0);
    if (csr_local) {
      int a0 = csr_rp[row - r0], a1 = csr_rp[row - r0 + 1];
      double acc = 0.0;
      for (int q = a0; q < a1; ++q) acc = __dadd_rn(acc, __dmul_rn(lav[q], xv[lci[q]]));
      return acc;
    }
    return op_row(p, sten, xv, row);
  };
  const size_t ld = p.ld;
  // Through the stencil form the next SpMV reads only rows within
  // max(sx, sxy) of this CTA's own: after sweep 2 a CTA waits for the `halo`
  // neighbour CTAs on each side instead of the whole grid.
  unsigned* nbe = st->nb_epoch;
  unsigned my_ep = tid == 0 ? ld_relaxed_gpu(nbe + blk * 16) : 0u;
  const int halo = sten ? (max(p.sv.sx, p.sv.sxy) + p.rpb - 1) / p.rpb : -1;
  const bool nbsync = halo >= 0 && 2 * halo + 1 < nblk && 2 * halo + 1 <= NT;
  // ---- cycle start --------------------------------------------------------
  const bool pend = p.fuse_comb && st->comb_pending != 0;
  long long cprof_t = clock64();
  if (pend) {
    apply_update(defl);
    CYCLE_SYNC();  // every CTA has read comb_pending and written its partials
    if (blk == 0 && tid == 0) st->comb_pending = 0;
  }
  CPROF(12);
  // partials: this launch's update (pend), k_project after a refresh
  // (comb_part 0), or a k_combine (comb_part 1)
  const bool comb_part = pend || st->comb_part != 0;
  if (defl) {
    reduce_partials(p.part + (comb_part ? (size_t)COMB_PART0 * GRID_MAX : 0), GRID_MAX,
                    pend ? nblk : comb_part ? st->comb_nblk : nblk, 0, 2 * kc, S.red);
    if (tid < kc) {
      double u2 = S.red[kc + tid];
      double un = sqrt(u2);
      S.dk[tid] = un == 0.0 ? 1.0 : 1.0 / un;
      S.cr[tid] = S.red[tid];
    }
  }
  // V_0. The reference takes r / beta as it is (gcrodr.py:412). In exact
  // arithmetic C^T r = 0 at every cycle start (the refresh projection and the
  // deflated LS both leave r orthogonal to C). The reference's sequential
  // CGS(C) + MGS(V) keeps |C^T r| / beta at 1e-10..1e-7 (measured with the
  // oracle on C3 system 5); the one-reduction DCGS2 treats [C | V] as
  // orthonormal and lets the component ride along with the lagged vector, so
  // it grew x2-4 per cycle (to 0.4 on C3 system 5, whose residual then stalled
  // at |C^T r| until the Pythagorean norm reported a spurious breakdown) and
  // C lost orthonormality (||C^T C - I|| 1e-14 -> 1e-7 over 9 cycles). When
  // |c_r| > V0_PROJ_RTOL beta (rounding level), V_0 is therefore formed from
  // r - C c_r with its measured norm beta0 (r = C c_r + beta0 V_0 exactly,
  // [C | V] orthonormal again); the LS keeps the reference's form
  // [c_r; beta0; 0]. Equal in exact arithmetic (c_r = 0).
  double beta0 = beta;
  bool v0proj = false;
  if (defl) {
    __syncthreads();
    double c2 = 0.0;
    for (int q = 0; q < kc; ++q) c2 = fma(S.cr[q], S.cr[q], c2);  // same order in every CTA
    v0proj = c2 > (p.v0_rtol * beta) * (p.v0_rtol * beta);
  }
  {
    double* V0 = colV(p, 0);
    if (v0proj) {
      double ss = 0.0;
      for (int row = r0 + tid; row < r1; row += NT) {
        double v = p.r[row];
        for (int c = 0; c < kc; ++c) v = fma(-colC(p, kcap - kc + c)[row], S.cr[c], v);
        V0[row] = v;
        ss = fma(v, v, ss);
      }
      const double t_ss = block_sum(ss, S.bred);
      if (tid == 0) p.part[(size_t)GRAM_PART0 * GRID_MAX + blk] = t_ss;
      CYCLE_SYNC();
      reduce_partials(p.part + (size_t)GRAM_PART0 * GRID_MAX, GRID_MAX, nblk, 0, 1, S.red);
      beta0 = sqrt(S.red[0]);
      for (int row = r0 + tid; row < r1; row += NT) V0[row] = V0[row] / beta0;
      if (blk == 0 && tid == 0) st->v0proj += 1;
    } else {
      for (int row = r0 + tid; row < r1; row += NT) V0[row] = p.r[row] / beta;
    }
  }
  if (tid == 0) S.gv[0] = beta0;
  if (blk == 0 && tid < kc) {
    st->dk[tid] = S.dk[tid];
    st->cr[tid] = S.cr[tid];
  }
#ifdef SKR_DIAG
  __syncthreads();
  if (blk == 0 && tid == 0) {
    double c2 = 0.0;
    for (int q = 0; q < kc; ++q) c2 += S.cr[q] * S.cr[q];
    printf("DIAG start st=%p cyc=%d kc=%d iters=%d beta=%.3e abstol=%.3e cr/beta=%.3e\n", (void*)st,
           st->cycles, kc, st->iters, beta, abs_tol, sqrt(c2) / beta);
  }
#endif
  int red_idx = 0;
  CYCLE_SYNC();
  CPROF(13);

  int j = 0;
  bool brk = false;
  double wn0_pending = 0.0;  // ||w - C C^T w|| / eta of the pending vector's step
  double hres = beta0;
  for (int t = 0; t <= s; ++t) {
    const bool do_spmv = (t < s);
    const int pb = kc + t;  // final basis columns [C | v_0..v_{t-1}]
    double* Vt = colV(p, t);
    // ---- sweep 1: z = op(V_t); dots of V_t and z against the final basis --
    // no block barrier inside: each warp streams its own tiles, the basis
    // columns in batches of CB (CB R independent loads per lane in flight), and
    // reduce-scatters the 2 CB partial dots of a batch with one butterfly.
    if (GPC && do_spmv) {
      // z = M^-1 (A V_t): the SpMV over this CTA's rows, then the grid-wide sweeps
      for (int row = r0 + tid; row < r1; row += NT) p.z[row] = row_dot(Vt, row);
      CYCLE_SYNC();
      if (!pc_apply_grid<GPC>(s_pc, p.z, 1, 0, cycle_sync)) {
        cycle_abort();
        return;
      }
    }
    double* sw = sacc + warp * 2 * PVC;
    for (int c = lane; c < 2 * PVC; c += 32) sw[c] = 0.0;
    __syncwarp();
    double nu = 0.0, mu = 0.0, ze = 0.0;
    for (int tile = warp; tile < ntile; tile += NW) {
      const int base = r0 + tile * TR + lane;
      int row[R];
      bool ok[R];
      double w[R], z[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int rr = base + 32 * i;
        ok[i] = rr < r1;
        row[i] = ok[i] ? rr : r1 - 1;
        w[i] = Vt[row[i]];
      }
      double dgv[R];  // Jacobi pivots, loaded ahead of the SpMV's dependent chain
#pragma unroll
      for (int i = 0; i < R; ++i) dgv[i] = p.dg ? __ldg(p.dg + row[i]) : 1.0;
      // all CB x R loads of a batch first (no branch: columns past pb re-read
      // column pb - 1 and their sums are dropped), then the FMAs. The first
      // batch is issued here, ahead of the SpMV: its round trip then overlaps
      // the SpMV's instead of following it (the compiler cannot hoist the loads
      // over the store of z)
      double qv[CB][R];
      auto load_batch = [&](int c0) {
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) {
          const double* Qc = Qb + (size_t)min(c0 + cc, pb - 1) * ld + base;
#pragma unroll
          for (int i = 0; i < R; ++i) qv[cc][i] = ok[i] ? Qc[32 * i] : 0.0;
        }
      };
      if (SW1_PREFETCH && pb > 0) load_batch(0);
      if (do_spmv && GPC) {
#pragma unroll
        for (int i = 0; i < R; ++i) z[i] = p.z[row[i]];  // M^-1 A V_t of the phase above
      } else if (do_spmv) {
        if (sten_local) {
#pragma unroll
          for (int i = 0; i < R; ++i)
            z[i] = sten_row_at<false>(lD, lW, lS, nullptr, p.sv.sx, 0, n, Vt, row[i], row[i] - r0);
        } else if (sten) {
#pragma unroll
          for (int i = 0; i < R; ++i) z[i] = sten_row(p.sv, Vt, row[i]);
        } else if (csr_local)
          spmv_rows<R, true>(csr_rp, lci, lav, Vt, row, ok, r0, z);
        else
          spmv_rows<R, false>(p.rp, p.ci, p.av, Vt, row, ok, r0, z);
#pragma unroll
        for (int i = 0; i < R; ++i) {
          if (p.dg) z[i] = __ddiv_rn(z[i], dgv[i]);
          if (ok[i]) p.z[row[i]] = z[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < R; ++i) z[i] = 0.0;
      }
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if (!ok[i]) w[i] = z[i] = 0.0;
        nu += w[i] * w[i];
        mu += w[i] * z[i];
        ze += z[i] * z[i];
      }
      for (int c0 = 0; c0 < pb; c0 += CB) {
        if (!SW1_PREFETCH || c0 > 0) load_batch(c0);
        double v[2 * CB];
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) {
          double dw = 0.0, dz = 0.0;
#pragma unroll
          for (int i = 0; i < R; ++i) {
            dw = fma(qv[cc][i], w[i], dw);
            dz = fma(qv[cc][i], z[i], dz);
          }
          v[cc] = dw;
          v[CB + cc] = dz;
        }
        const double tot = bfly<2 * CB>(v, lane);
        constexpr int SH = 5 - log2c<2 * CB>();
        const int idx = (lane >> SH) & (2 * CB - 1), col = c0 + (idx % CB);
        if (!(lane & ((1 << SH) - 1)) && col < pb) sw[(idx / CB) * PVC + col] += tot;
      }
    }

    // warp partials of |w|^2, w.z, |z|^2 next to the column partials
    for (int o = 16; o > 0; o >>= 1) {
      nu += __shfl_xor_sync(0xffffffffu, nu, o);
      mu += __shfl_xor_sync(0xffffffffu, mu, o);
      ze += __shfl_xor_sync(0xffffffffu, ze, o);
    }
    if (lane == 0) {
      S.bred[3 * warp] = nu;
      S.bred[3 * warp + 1] = mu;
      S.bred[3 * warp + 2] = ze;
    }
    __syncthreads();
    // cross-CTA sums, deterministic: every CTA stores its partials (layout: 0
    // nu, 1 mu, 2 ze, 3.. a (pb), 3+pb.. bb (pb)) to its own slot of a
    // double-buffered array; after the grid barrier every CTA sums all slots
    // in one fixed order, so all CTAs hold bit-identical totals and a solve
    // is reproducible run to run. Buffer r % 2 is rewritten at step r + 2, after
    // barrier r + 1, which every reader of step r has passed.
    const int nv = 3 + 2 * pb;
    double* sbuf = p.sred + (size_t)(red_idx & 1) * GRID_MAX * PV_STEP;
    {
      double* mine = sbuf + (size_t)blk * PV_STEP;
      for (int e = tid; e < nv; e += NT) {
        double sum = 0.0;
        if (e < 3) {
#pragma unroll
          for (int q = 0; q < NW; ++q) sum += S.bred[3 * q + e];
        } else {
          const int which = e - 3 >= pb, col = which ? e - 3 - pb : e - 3;
#pragma unroll
          for (int q = 0; q < NW; ++q) sum += sacc[q * 2 * PVC + which * PVC + col];
        }
        mine[e] = sum;
      }
    }
    CPROF(0);
    CYCLE_SYNC();
    CPROF(1);
    {
      // ng thread groups per value: group g sums slots g, g + ng, ... in
      // chunks of RL loads issued together (one L2 round trip per chunk; at
      // 64 CTAs per chain that is a single chunk), each chunk added as a
      // fixed tree; the groups are combined in order below
      constexpr int RL = 16;
      const int ng = max(1, NT / nv);
      double* gsum = sacc;  // sweep-1 partials are consumed: reuse the area
      if (tid < ng * nv) {
        const int v = tid % nv, g = tid / nv;
        double acc = 0.0;
        for (int b0 = g; b0 < nblk; b0 += RL * ng) {
          double q[RL];
#pragma unroll
          for (int u = 0; u < RL; ++u) {
            const int b = b0 + u * ng;
            q[u] = b < nblk ? sbuf[(size_t)b * PV_STEP + v] : 0.0;
          }
#pragma unroll
          for (int w = RL / 2; w >= 1; w /= 2)
#pragma unroll
            for (int u = 0; u < w; ++u) q[u] += q[u + w];
          acc += q[0];
        }
        gsum[g * nv + v] = acc;
      }
      __syncthreads();
      for (int v = tid; v < nv; v += NT) {
        double t = gsum[v];
        for (int g = 1; g < ng; ++g) t += gsum[g * nv + v];
        S.red[v] = t;
      }
    }
    ++red_idx;
    __syncthreads();
    // ---- LS / control (identical in every CTA) ------------------------------
    // warp 0: eta, the final column t-1, its Givens update and the first-pass
    // column t; warps 1..: copy the sweep-2 coefficients (a, and b unscaled:
    // sweep 2 divides by eta). One block barrier.
    static_assert(NW >= 2, "the LS phase splits warp 0 from the others");
    const double* A_ = S.red + 3;
    const double* BB = S.red + 3 + pb;
    if (warp == 0) {
      double aa = 0.0, ab = 0.0, cc = 0.0, ag = 0.0;
      for (int c = lane; c < pb; c += 32) {
        double av = (t >= 1) ? A_[c] : 0.0, bv = BB[c];
        aa += av * av;
        ab += av * bv;
        if (c < kc) {
          cc += bv * bv;
          ag += av * S.cr[c];  // a_C . (C^T r)
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        aa += __shfl_xor_sync(0xffffffffu, aa, o);
        ab += __shfl_xor_sync(0xffffffffu, ab, o);
        cc += __shfl_xor_sync(0xffffffffu, cc, o);
        ag += __shfl_xor_sync(0xffffffffu, ag, o);
      }
      // ||w - Q a||^2 = ||w||^2 - |a|^2 + a^T (Q^T Q - I) a. Every basis
      // vector is projected against C except V_0 = r / beta (reference
      // semantics), whose Gram block with C is C^T r / beta (the cycle-start
      // c_r): near convergence r's direction is rounding noise, V_0 is far
      // from orthogonal to C, and without this term the Pythagorean eta falls
      // to 0 (a spurious breakdown; the reference measures ||w|| directly).
      const double gcorr = (t >= 1 && kc > 0 && !v0proj) ? 2.0 * A_[kc] * ag / beta : 0.0;
      const double eta0 = (t >= 1) ? sqrt(fmax(S.red[0] - aa + gcorr, 0.0)) : 1.0;
      const bool brk0 =
          t >= 1 && eta0 < 1e-14 * fmax(wn0_pending, 2.2250738585072014e-308);
#ifdef SKR_DIAG
      if (blk == 0 && lane == 0 && t >= 1 && (brk0 || S.red[0] - aa + gcorr < 0.5 * S.red[0]))
        printf("DIAG bessel st=%p cyc=%d t=%d nu=%.3e aa=%.3e gcorr=%.3e eta0=%.3e wn0=%.3e brk=%d\n",
               (void*)st, st->cycles, t, S.red[0], aa, gcorr, eta0, wn0_pending, (int)brk0);
#endif
      if (t >= 1) {
        // final column i = t-1: first pass + reorthogonalisation coefficients
        const int i = t - 1;
        for (int q = lane; q <= i + 1; q += 32) S.hcol[q] = (q <= i) ? S.hp[q] + A_[kc + q] : eta0;
        for (int c = lane; c < kc; c += 32) {
          double v = S.bp[c] + A_[c];
          Bsm[c + i * kcap] = v;
          if (blk == 0) st->B[c + i * LDB] = v;
        }
        if (blk == 0)
          for (int q = lane; q < LDH; q += 32)
            st->H[q + i * LDH] = (q <= i) ? S.hp[q] + A_[kc + q] : (q == i + 1 ? eta0 : 0.0);
      }
      __syncwarp();
      if (lane == 0) {
        bool stop0 = false;
        if (t >= 1) {
          // Givens update of column i; the running entry stays in a register
          const int i = t - 1;
          double* hcol = S.hcol;
          double run = hcol[0];
#pragma unroll 4
          for (int q = 0; q < i; ++q) {
            const double cq = S.cs[q], sq = S.sn[q], nx = hcol[q + 1];
            hcol[q] = fma(cq, run, sq * nx);
            run = fma(-sq, run, cq * nx);
          }
          hcol[i] = run;
          const double hn = hcol[i + 1];
          const double d2 = fma(run, run, hn * hn);
          double den, cs_, sn_;
          if (d2 == 0.0 || !(d2 < 1e300) || d2 < 1e-300) {  // rare: the overflow-safe path
            den = hypot(run, hn);
            cs_ = den == 0.0 ? 1.0 : run / den;
            sn_ = den == 0.0 ? 0.0 : hn / den;
          } else {
            const double rd = rsqrt(d2);
            den = d2 * rd;
            cs_ = run * rd;
            sn_ = hn * rd;
          }
          S.cs[i] = cs_;
          S.sn[i] = sn_;
          hcol[i] = den;
          S.gv[i + 1] = -sn_ * S.gv[i];
          S.gv[i] = cs_ * S.gv[i];
          hres = fabs(S.gv[i + 1]);
          if (blk == 0) p.hist[st->hist_len + i] = hres;
          stop0 = brk0 || hres <= abs_tol || t == s;
        }
        S.sc[0] = eta0;
        S.sc[1] = stop0 ? 1.0 : 0.0;
        S.sc[2] = brk0 ? 1.0 : 0.0;
        if (!stop0) {
          const double ie = 1.0 / eta0;
          S.sc[3] = (S.red[1] - ab) * ie * ie;  // h_tt = (mu - a.bb) / eta^2
          wn0_pending = sqrt(fmax(S.red[2] - cc, 0.0)) * ie;
        }
      }
      __syncwarp();
      const bool stop0 = S.sc[1] != 0.0;
      if (t >= 1) {
        const int i = t - 1;
        const int base = i * (i + 1) / 2;  // packed upper-triangular R
        for (int q = lane; q <= i; q += 32) Rsm[base + q] = S.hcol[q];
      }
      if (!stop0) {  // first-pass column t (scaled), finalised at the next step
        const double ie = 1.0 / eta0;
        for (int c = lane; c < kc; c += 32) S.bp[c] = BB[c] * ie;
        for (int q = lane; q < t; q += 32) S.hp[q] = BB[kc + q] * ie;
        if (lane == 0) S.hp[t] = S.sc[3];
      }
    } else {
      for (int c = tid - 32; c < pb; c += NT - 32) {
        S.a[c] = (t >= 1) ? A_[c] : 0.0;
        S.bb[c] = BB[c];
      }
    }
    __syncthreads();
    const double eta = S.sc[0];
    brk = S.sc[2] != 0.0;
    const bool stop = S.sc[1] != 0.0;
    CPROF(2);
    // ---- sweep 2: finish V_t, project the new vector into V_{t+1} ----------
    {
      const double htt = S.sc[3];
      const double ieta = 1.0 / eta;  // one reciprocal per step, not two divides per row
      double* Vn = colV(p, t + 1);
      const bool need = (t >= 1 || !stop);
      // tiles in the reverse order of sweep 1 (and of the next sweep 1): the
      // rows streamed last are still in L2 when this sweep starts on them
      for (int rt = warp; rt < ntile; rt += NW) {
        const int tile = ntile - 1 - rt;
        const int base = r0 + tile * TR + lane;
        bool ok[R];
        double ta[R], tb[R], wv[R], zv[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          ok[i] = base + 32 * i < r1;
          ta[i] = 0.0;
          tb[i] = 0.0;
          // this row's pending vector and z, in flight during the batches
          const int rr = ok[i] ? base + 32 * i : r1 - 1;
          wv[i] = Vt[rr];
          zv[i] = p.z[rr];
        }
        if (need) {
          for (int c0 = 0; c0 < pb; c0 += SW2_COLS) {
            // SW2_COLS x R loads first; columns past pb get zero coefficients
            double qv[SW2_COLS][R];
#pragma unroll
            for (int cc = 0; cc < SW2_COLS; ++cc) {
              const double* Qc = Qb + (size_t)min(c0 + cc, pb - 1) * ld + base;
#pragma unroll
              for (int i = 0; i < R; ++i) qv[cc][i] = ok[i] ? Qc[32 * i] : 0.0;
            }
#pragma unroll
            for (int cc = 0; cc < SW2_COLS; ++cc) {
              const bool in = c0 + cc < pb;
              const double ca = in ? S.a[c0 + cc] : 0.0, cb = in ? S.bb[c0 + cc] : 0.0;
#pragma unroll
              for (int i = 0; i < R; ++i) {
                ta[i] = fma(qv[cc][i], ca, ta[i]);
                tb[i] = fma(qv[cc][i], cb, tb[i]);
              }
            }
          }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
          if (!ok[i]) continue;
          const int rr = base + 32 * i;
          double vt = wv[i];
          if (t >= 1) {
            vt = brk ? 0.0 : (wv[i] - ta[i]) * ieta;
            Vt[rr] = vt;
          }
          if (!stop) Vn[rr] = (zv[i] - tb[i]) * ieta - vt * htt;  // tb: unscaled b
        }
      }

    }
    if (stop) {
      j = t;
      // every CTA: y2 = R^-1 g (warp 0, packed R in smem), y1 = (cr - B y2) / dk
      if (warp == 0) {
        for (int q = lane; q < j; q += 32) S.y[kc + q] = S.gv[q];
        __syncwarp();
        for (int kk = j - 1; kk >= 0; --kk) {
          const int bk = kk * (kk + 1) / 2;
          double yk = S.y[kc + kk] / Rsm[bk + kk];
          __syncwarp();
          for (int q = lane; q < kk; q += 32) S.y[kc + q] -= Rsm[bk + q] * yk;
          if (lane == 0) S.y[kc + kk] = yk;
          __syncwarp();
        }
        for (int c = lane; c < kc; c += 32) {
          double sacc = S.cr[c];
          for (int q = 0; q < j; ++q) sacc -= Bsm[c + q * kcap] * S.y[kc + q];
          S.y[c] = sacc / S.dk[c];
        }
        __syncwarp();
        if (blk == 0)
          for (int q = lane; q < kc + j; q += 32) st->y[q] = S.y[q];
      }
      if (blk == 0 && tid == 0) {
        st->j = j;
        st->brk = brk ? 1 : 0;
        st->g[0] = hres;
      }
      __syncthreads();
      CPROF(7);
      break;
    }
    CPROF(3);
    if (nbsync) {
      // publish this CTA's sweep, then wait for the halo neighbours' (release /
      // acquire at gpu scope, as grid_sync; a timeout aborts instead of hanging)
      __syncthreads();
      if (tid == 0) {
        fence_acq_rel_gpu();
        ++my_ep;
        atomicExch(nbe + blk * 16, my_ep);
        S.ep = my_ep;
        S.flag = 0;
      }
      __syncthreads();
      const int nb = blk - halo + tid;
      if (tid <= 2 * halo && nb >= 0 && nb < nblk && nb != blk) {
        const unsigned target = S.ep;
        unsigned long long t0 = gtimer();
        unsigned polls = 0;
        while (ld_acquire_gpu(nbe + nb * 16) < target) {
          if ((++polls & 255) == 0 &&
              (gtimer() - t0 > BARRIER_TIMEOUT_NS ||
               ld_relaxed_gpu(reinterpret_cast<unsigned*>(abt)))) {
            atomicExch(abt, 1);
            S.flag = 1;
            break;
          }
        }
        fence_acq_rel_gpu();
      }
      __syncthreads();
      if (S.flag) {
        if (tid == 0) {
          st->done = 1;
          if (blk == 0) flag_host(st, cycle_id, 1);
        }
        return;
      }
    } else {
      CYCLE_SYNC();
    }
    CPROF(4);
  }

  // ---- cycle end: x update, explicit residual, cross-Gram partials ---------
  for (int q = tid; q < kc; q += NT) S.y[q] *= S.dk[q];
  __syncthreads();
  const int mm = kc + j;
  // cross-Gram What[:, :mm]^T Vhat (mm x mm, What = [C | V_0..V_{j-1}], Vhat
  // = [U | V_0..V_{j-1}]) over this CTA's rows. For mm <= 40 (every BASELINE
  // config but C2) on the fp64 tensor cores (DMMA m8n8k4, rows = the k
  // dimension), in the same pass over the staged 32-row tiles as the x update
  // x += U (dk y1) + V y2, whose U and V columns are staged anyway; otherwise
  // the register-tiled CUDA-core Gram after the residual (below).
  const bool gmma = defl && m <= GM_MMAX;
  auto tile_col = [&](int c) -> const double* {  // staged columns [U (kc) | C (kc) | V (j)]
    // basis column c (U) or c + 2 (kcap - kc): the right-aligned C block and V are adjacent
    return p.basis + (size_t)(c < kc ? c : c + 2 * (kcap - kc)) * ld;
  };
  if (gmma) {
    constexpr int GL = GM_LD;  // == 4 (mod 16) doubles: conflict-free fragment loads
    const int ncs = 2 * kc + j;
    const int nb = (mm + 7) >> 3;  // 8 x 8 blocks per side, <= 5
    // Vhat block columns the tensor cores compute: all of them, or (gram_half)
    // only those holding U columns -- What^T V = [0; I] is then taken from the
    // orthonormality DCGS2 maintains (see the cross reduction below)
    const int nby = p.gram_half ? (kc + 7) >> 3 : nb;
    // warp w: block rows bi in [3 h, 3 h + 3) (h = w & 1), k-steps 2 (w >> 1)
    // and 2 (w >> 1) + 1 of every tile (rows 4 ks .. 4 ks + 3); lane l holds
    // A[m = l/4][k = l%4] = What(row, 8 bi + m), B[k][n = l/4] = Vhat(row, 8 bj + n)
    const int h = warp & 1, ks0 = 2 * (warp >> 1);
    const int ln = lane >> 2, lk = lane & 3;
    int wa[3], vb[5];
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const int a = min(8 * (3 * h + x) + ln, mm - 1);
      wa[x] = ((a < kc) ? kc + a : 2 * kc + (a - kc)) * GL + lk;
    }
#pragma unroll
    for (int y = 0; y < 5; ++y) {
      const int b = min(8 * y + ln, mm - 1);
      vb[y] = ((b < kc) ? b : 2 * kc + (b - kc)) * GL + lk;
    }
    double acc[3][5][2];
#pragma unroll
    for (int x = 0; x < 3; ++x)
#pragma unroll
      for (int y = 0; y < 5; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    // tiles through a two-stage shared-memory ring filled by 16-byte cp.async
    // copies (no registers: the pass's DMMA accumulators need them), one
    // tile in flight while the other is consumed; rows past r1 zero-filled
    const int gs = (kcap + m + 1) * GL;  // doubles per stage (ncs <= kcap + m + 1)
    double* xpart = cdyn + gs;           // x-update scratch between the stages
    double* stage1 = cdyn + gs + NT;
    const int ntl = (r1 - r0 + 31) >> 5;
    auto issue_tile = [&](int i) {
      if (i < ntl) {
        const int t0 = r0 + 32 * i;
        double* dst = (i & 1) ? stage1 : gtile;
        for (int e = tid; e < 16 * ncs; e += NT) {
          const int c = e >> 4, rr = 2 * (e & 15), row = t0 + rr;
          const int nbytes = row < r1 ? (row + 1 < r1 ? 16 : 8) : 0;
          const double* src = tile_col(c) + (nbytes ? row : r0);
          const unsigned d = (unsigned)__cvta_generic_to_shared(dst + c * GL + rr);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
                       "r"(nbytes) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue_tile(0);
    for (int it = 0; it < ntl; ++it) {
      const int t0 = r0 + 32 * it;
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();  // tile `it` landed for every thread; the other stage is consumed
      issue_tile(it + 1);
      const double* gtl = (it & 1) ? stage1 : gtile;
      // warp 0 fetches this tile's x now: its latency hides behind the DMMAs
      const double xold = (tid < 32 && t0 + tid < r1) ? p.x[t0 + tid] : 0.0;
      {  // x update partials: warp w sums the [U | V] columns c == w (mod NW)
        double xs = 0.0;
        for (int c = warp; c < kc + j; c += NW) {
          const int sc = c < kc ? c : 2 * kc + (c - kc);
          xs = fma(gtl[sc * GL + lane], S.y[c], xs);
        }
        xpart[warp * 32 + lane] = xs;
      }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int roff = 4 * (ks0 + kk);
        double af[3], bf[5];
#pragma unroll
        for (int x = 0; x < 3; ++x) af[x] = gtl[wa[x] + roff];
#pragma unroll
        for (int y = 0; y < 5; ++y)
          if (y < nby) bf[y] = gtl[vb[y] + roff];
#pragma unroll
        for (int x = 0; x < 3; ++x)
          if (3 * h + x < nb)
#pragma unroll
            for (int y = 0; y < 5; ++y)
              if (y < nby)
                asm volatile(
                    "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(acc[x][y][0]), "+d"(acc[x][y][1])
                    : "d"(af[x]), "d"(bf[y]));
      }
      __syncthreads();
      if (tid < 32 && t0 + tid < r1) {  // warps' partials added in order
        double xs = xpart[tid];
#pragma unroll
        for (int w = 1; w < NW; ++w) xs += xpart[w * 32 + tid];
        p.x[t0 + tid] = xold + xs;
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // the four k-step pairs of each half are added in warp order (fixed)
    double* gb = gtile;
    for (int q = 0; q < NW; ++q) {
      if (warp == q) {
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int y = 0; y < 5; ++y) {
            const int bi = 3 * h + x;
            if (bi < nb && y < nby) {
              const int idx = (bi * nb + y) * 64 + ln * 8 + 2 * lk;
              if (q < 2) {
                gb[idx] = acc[x][y][0];
                gb[idx + 1] = acc[x][y][1];
              } else {
                gb[idx] += acc[x][y][0];
                gb[idx + 1] += acc[x][y][1];
              }
            }
          }
      }
      __syncthreads();
    }
    for (int e = tid; e < mm * (p.gram_half ? kc : mm); e += NT) {
      const int a = e % mm, b = e / mm;
      p.part[(size_t)(GRAM_PART0 + e) * GRID_MAX + blk] =
          gb[((a >> 3) * nb + (b >> 3)) * 64 + (a & 7) * 8 + (b & 7)];
    }
  } else {
    for (int row = r0 + tid; row < r1; row += NT) {
      double su = 0.0, sv = 0.0;
      for (int c = 0; c < kc; ++c) su += colU(p, c)[row] * S.y[c];
      for (int v = 0; v < j; ++v) sv += colV(p, v)[row] * S.y[kc + v];
      p.x[row] = p.x[row] + (su + sv);
    }
  }
  CPROF(8);
  CYCLE_SYNC();
  CPROF(9);

  // ---- explicit residual (needs the neighbours' updated x) --------------------
  double rr = 0.0;
  for (int row = r0 + tid; row < r1; row += NT) {
    double rv = __dsub_rn(__ldg(p.b + row), row_dot(p.x, row));
    if (p.dg) rv = __ddiv_rn(rv, __ldg(p.dg + row));
    p.r[row] = rv;
    rr += rv * rv;
  }
  if (GPC) {
    CYCLE_SYNC();
    if (!pc_apply_grid<GPC>(s_pc, p.r, 1, 0, cycle_sync)) {
      cycle_abort();
      return;
    }
    rr = 0.0;
    for (int row = r0 + tid; row < r1; row += NT) rr = fma(p.r[row], p.r[row], rr);
  }
  if (defl && !gmma) {
    // cross-Gram What[:, :mm]^T Vhat over this CTA's rows, register-tiled: a
    // thread owns the 4 x 4 entries (ai + x*na4, bi + y*na4), so consecutive
    // lanes read consecutive columns of a 32-row tile staged column-major with
    // an odd leading dimension (conflict-free); 8 shared loads feed 16 FMAs.
    // Per-CTA sums go to p.part[(GRAM_PART0 + entry) * GRID_MAX + blk]; after
    // the barrier every entry is summed over the CTAs in a fixed order
    // (deterministic). staged columns: [U (kc) | C (kc) | V_0..V_{j-1}]
    const int ncs = 2 * kc + j;
    const int na4 = (mm + 3) / 4;
    const int nblkt = na4 * na4;  // thread blocks of entries (<= 256 for mm <= 64)
    // G groups of threads split each tile's 32 rows (idle threads otherwise);
    // their sums are added in group order through the staging area at the end
    int ngr = NT / nblkt;
    ngr = ngr > 4 ? 4 : ngr;
    while (ngr > 1 && (size_t)(ngr - 1) * nblkt * 16 > (size_t)p.sm_R) --ngr;
    const int gblk = tid % nblkt, grp = tid / nblkt;
    const int rows_g = 32 / ngr, rlo = grp * rows_g, rhi = grp == ngr - 1 ? 32 : rlo + rows_g;
    double gacc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) gacc[q] = 0.0;
    int ca[4], cb[4];
    {
      const int ai = gblk % na4, bi = gblk / na4;
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        int a = min(ai + x * na4, mm - 1);
        ca[x] = ((a < kc) ? kc + a : 2 * kc + (a - kc)) * GT_LD;  // What col: C or V
        int b = min(bi + x * na4, mm - 1);
        cb[x] = ((b < kc) ? b : 2 * kc + (b - kc)) * GT_LD;  // Vhat col: U or V
      }
    }
    // the next 32-row tile is loaded into registers while this one is reduced
    // (the first GPF elements per thread: all of them when ncs <= 64)
    constexpr int GPF = 8;
    auto tile_src = [&](int e, int t0) -> double {
      const int rrw = e & 31, c = e >> 5, row = t0 + rrw;
      const double* col = (c < kc) ? colU(p, c)
                          : (c < 2 * kc) ? colC(p, kcap - kc + (c - kc))
                                         : colV(p, c - 2 * kc);
      return row < r1 ? col[row] : 0.0;
    };
    double pf[GPF];
    auto load_tile = [&](int t0) {
#pragma unroll
      for (int k = 0; k < GPF; ++k) {
        const int e = tid + k * NT;
        if (e < 32 * ncs) pf[k] = tile_src(e, t0);
      }
    };
    if (r0 < r1) load_tile(r0);
    for (int t0 = r0; t0 < r1; t0 += 32) {
#pragma unroll
      for (int k = 0; k < GPF; ++k) {
        const int e = tid + k * NT;
        if (e < 32 * ncs) gtile[(e >> 5) * GT_LD + (e & 31)] = pf[k];
      }
      for (int e = tid + GPF * NT; e < 32 * ncs; e += NT)
        gtile[(e >> 5) * GT_LD + (e & 31)] = tile_src(e, t0);
      __syncthreads();
      if (t0 + 32 < r1) load_tile(t0 + 32);
      __syncthreads();
      if (grp < ngr) {
#pragma unroll 4
        for (int rrw = rlo; rrw < rhi; ++rrw) {
          double wa[4], vb[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) wa[x] = gtile[ca[x] + rrw];
#pragma unroll
          for (int y = 0; y < 4; ++y) vb[y] = gtile[cb[y] + rrw];
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) gacc[x * 4 + y] = fma(wa[x], vb[y], gacc[x * 4 + y]);
        }
      }
      __syncthreads();
    }
    if (ngr > 1) {  // groups 1.. hand their sums to group 0 (fixed order)
      if (grp >= 1 && grp < ngr)
#pragma unroll
        for (int q = 0; q < 16; ++q) gtile[((size_t)(grp - 1) * nblkt + gblk) * 16 + q] = gacc[q];
      __syncthreads();
      if (grp == 0)
        for (int g = 1; g < ngr; ++g)
#pragma unroll
          for (int q = 0; q < 16; ++q) gacc[q] += gtile[((size_t)(g - 1) * nblkt + gblk) * 16 + q];
    }
    if (grp == 0) {
      const int ai = gblk % na4, bi = gblk / na4;
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int a = ai + x * na4, b = bi + y * na4;
          if (a < mm && b < mm)
            p.part[(size_t)(GRAM_PART0 + a + b * mm) * GRID_MAX + blk] = gacc[x * 4 + y];
        }
    }
  }
  {
    double t_rr = block_sum(rr, S.bred);
    if (tid == 0) p.part[blk] = t_rr;
  }
  CPROF(10);
  CYCLE_SYNC();
  CPROF(11);
  if (defl) {
    // one warp per cross entry: sum the CTAs' partials (lane-strided, then a
    // butterfly: a fixed order), scale Vhat's U columns by dk (Vhat =
    // [U diag(dk), V]) into st->cross
    const bool half = gmma && p.gram_half;
    for (int e = blk * NW + warp; e < mm * mm; e += nblk * NW) {
      const int a = e % mm, b = e / mm;
      if (half && b >= kc) {
        // What^T V_{b - kc}: [C | V] is orthonormal (DCGS2 + the V_0 projection
        // keep ||Q^T Q - I|| at 1e-13), so the column is e_b
        if (lane == 0) st->cross[a + b * LDX] = a == b ? 1.0 : 0.0;
        continue;
      }
      const double* q = p.part + (size_t)(GRAM_PART0 + e) * GRID_MAX;
      double v = 0.0;
      for (int c = lane; c < nblk; c += 32) v += q[c];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) st->cross[a + b * LDX] = (b < kc) ? v * st->dk[b] : v;
    }
  }
  if (blk == 0) {
    reduce_partials(p.part, GRID_MAX, nblk, 0, 1, S.red);
    if (tid == 0) {
      double rnorm = sqrt(S.red[0]);
      st->rnorm = rnorm;
      st->converged = rnorm <= abs_tol ? 1 : 0;
#ifdef SKR_DIAG
      printf("DIAG end st=%p cyc=%d j=%d brk=%d lsres=%.3e rnorm=%.3e conv=%d\n", (void*)st, st->cycles,
             j, st->brk, st->g[0], rnorm, st->converged);
#endif
      p.checks[2 * st->nchecks] = st->g[0];
      p.checks[2 * st->nchecks + 1] = rnorm;
      st->nchecks += 1;
      st->hist_len += j;
      st->iters += j;
      st->steps += j;
      if (defl) st->defl_steps += j;
      st->cycles += 1;
      st->ran = 1;
      st->prof[21] += clock64() - cprof_t;  // tail: distributed Gram reduce + r norm
      st->prof[22] += j + 1;                // sweep iterations
      // SURVEY 8(d) algorithmic bytes: per step B_spmv + 8N(2p+6), p = basis width
      double N = (double)n;
      // (stencil form: D, W, S (, B) instead of the CSR arrays)
      double bsp = sten ? (p.sv.sxy ? 32.0 : 24.0) * N + 16.0 * N
                        : 12.0 * (double)(__ldg(p.rp + n)) + 4.0 * (N + 1) + 16.0 * N;
      double acc = 0.0;
      for (int q = 0; q < j; ++q) {
        int pw = kc + q + 1;
        acc += bsp + 8.0 * N * (2.0 * pw + 6.0);
      }
      st->step_bytes += acc;
    }
  }
  (void)cycle_id;
}

// ---------------------------------------------------------------------------
// diagnostics (collect_diagnostics, gcrodr.py:116-123, :372-376, :461-467):
// ||op U - C||_F and ||C^T C - I||_F of the current pair, after the refresh
// (stage 0) and after every deflated cycle's recycle update (stage 1)
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool diag_skip(const State* st, int stage) {
  if (st->zero_rhs) return true;
  return stage == 1 && (!st->ran || st->kc_prev == 0);  // GMRES cycles log nothing
}
// per-CTA partials (rows DIAG_PART0..): [0] sum (op U_q - C_q)^2, [1 + a kc + b] (C^T C)_ab
__global__ void __launch_bounds__(NT) k_diag(Ptrs p, int stage) {
  State* st = p.st;
  if (diag_skip(st, stage)) return;
  const int kc = st->kc;
  __shared__ double tile[32][KMAX + 1];
  __shared__ double s_red[NW];
  const int r0 = blockIdx.x * p.rpb, r1 = min(p.n, r0 + p.rpb);
  const bool sten = sten_ok(p.sv);
  double res = 0.0;
  for (int row = r0 + threadIdx.x; row < r1; row += NT) {
    const double d = p.dg ? __ldg(p.dg + row) : 1.0;
    for (int q = 0; q < kc; ++q) {
      // general preconditioner: op(U_q) was formed in the V block (k_pc_cols target 2)
      double v = p.pch ? colV(p, q)[row] : op_row(p, sten, colU(p, q), row);
      if (p.dg) v = __ddiv_rn(v, d);
      v -= colC(p, p.kcap - kc + q)[row];
      res += v * v;
    }
  }
  const double tres = block_sum(res, s_red);
  double acc[2] = {0.0, 0.0};  // kc^2 <= 441 < 2 NT entries
  for (int t0 = r0; t0 < r1; t0 += 32) {
    for (int e = threadIdx.x; e < 32 * kc; e += NT) {
      const int rr = e & 31, c = e >> 5, row = t0 + rr;
      tile[rr][c] = row < r1 ? colC(p, p.kcap - kc + c)[row] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = threadIdx.x + h * NT;
      if (e < kc * kc) {
        const int a = e / kc, b = e % kc;
        double g = 0.0;
        for (int rr = 0; rr < 32; ++rr) g += tile[rr][a] * tile[rr][b];
        acc[h] += g;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) p.part[(size_t)DIAG_PART0 * GRID_MAX + blockIdx.x] = tres;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int e = threadIdx.x + h * NT;
    if (e < kc * kc) p.part[(size_t)(DIAG_PART0 + 1 + e) * GRID_MAX + blockIdx.x] = acc[h];
  }
}
// one CTA: fixed-order sums of the partials, one record appended to the log
__global__ void __launch_bounds__(NT) k_diag_fin(Ptrs p, int stage) {
  State* st = p.st;
  if (diag_skip(st, stage)) return;
  const int kc = st->kc;
  __shared__ double red[1 + KMAX * KMAX];
  reduce_partials(p.part + (size_t)DIAG_PART0 * GRID_MAX, GRID_MAX, p.nblk, 0, 1 + kc * kc, red);
  if (threadIdx.x == 0) {
    double o = 0.0;
    for (int a = 0; a < kc; ++a)
      for (int b = 0; b < kc; ++b) {
        const double g = red[1 + a * kc + b] - (a == b ? 1.0 : 0.0);
        o += g * g;
      }
    double* rec = p.dlog + 4 * (size_t)st->ndiag;
    rec[0] = stage;
    rec[1] = kc;
    rec[2] = kc > 0 ? sqrt(red[0]) : 0.0;
    rec[3] = kc > 0 ? sqrt(o) : 0.0;
    st->ndiag += 1;
  }
}

// ---------------------------------------------------------------------------
// the single-CTA dense kernel (programs)
// ---------------------------------------------------------------------------
__device__ void set_done(State* st, int cycle) {
  st->done = 1;
  flag_host(st, cycle, 1);
}

__global__ void __launch_bounds__(NT) k_dense(Ptrs p, int prog, int arg, int cycle_id) {
  State* st = p.st;
  extern __shared__ double dsm[];
  __shared__ int s_iw[8 * skrd::LDD];
  __shared__ int s_kept[KMAX];
  skrd::Ctx c = skrd::ctx();
  skrd::Arena ar = skrd::make_arena(dsm, s_iw, c.nw, skrd::arena_ld(st->m));
  const int tid = threadIdx.x;
  switch (prog) {
    case P_INIT: {
      reduce_partials(p.part, GRID_MAX, p.nblk, 0, 3, ar.red);
      if (tid == 0) {
        double bn = sqrt(ar.red[0]);
        st->bnorm = bn;
        if (bn == 0.0) {
          st->zero_rhs = 1;
          st->converged = 1;
          st->rnorm = 0.0;
          p.hist[0] = 0.0;
          st->hist_len = 1;
          set_done(st, -1);
        } else {
          double bp = sqrt(ar.red[1]);
          st->bprec = bp;
          st->abs_tol = st->tol * bp;
          double rn = sqrt(ar.red[2]);
          st->rnorm = rn;
          p.hist[0] = rn;
          st->hist_len = 1;
          st->kc = 0;
          st->ncol_a = st->k_in;
          if (st->k_in > 0) st->iters += st->k_in;  // gcrodr.py:363
          st->converged = rn <= st->abs_tol ? 1 : 0;
          if (st->k_in == 0 && (st->converged || st->iters >= st->max_iter)) set_done(st, -1);
        }
      }
      break;
    }
    case P_CHOL1: {
      if (st->done) break;
      int nc = arg == 0 ? st->ncol_a : st->ncol_b;
      if (nc <= 0) break;
      // gram -> T1 (coefU or coefC block), R1
      double* T = arg == 0 ? st->coefU : st->coefC;
      int r = skrd::cholqr_pass1(c, ar, st->gram, LDK, nc, T, LDC, st->R1, LDK);
      if (tid == 0) {
        st->r_tmp = r;
        st->cm_mode = arg == 0 ? CM_U_ONLY : CM_C_ONLY;
        st->cm_nin_u = arg == 0 ? nc : 0;
        st->cm_nout_u = arg == 0 ? r : 0;
        st->cm_nin_c = arg == 0 ? 0 : nc;
        st->cm_nout_c = arg == 0 ? 0 : r;
        if (r < nc) st->warn |= (arg == 0 ? skrd::W_RANK_DROP : skrd::W_REFRESH_RANK);
        if (arg == 0)
          st->ncol_a = r;
        else
          st->ncol_b = r;
        st->ncol_orig = nc;  // original width for pass 2
      }
      break;
    }
    case P_CHOL2: {
      if (st->done) break;
      int r = arg == 0 ? st->ncol_a : st->ncol_b;
      int korig = st->ncol_orig;
      if (r <= 0) {
        if (tid == 0) {
          st->kc = 0;
          st->ncol_a = 0;
          st->ncol_b = 0;
          st->cm_mode = CM_U_ONLY;
          st->cm_nin_u = 0;
          st->cm_nout_u = 0;
          st->cm_nin_c = 0;
          st->cm_nout_c = 0;
          if (st->converged || st->iters >= st->max_iter) set_done(st, -1);
        }
        break;
      }
      double* T2 = arg == 0 ? st->coefU : st->coefC;
      double* Rinv = ar.M4;
      // pass 2 on the materialised X1 (its Gram reduced into st->gram)
      int r2 = skrd::cholqr_pass2(c, ar, st->gram, LDK, r, st->R1, LDK, korig, T2, LDC, s_kept,
                                  Rinv, ar.ld);
      if (arg == 1 && r2 > 0) {
        // U = Yo[:, kept] R'^-1 : coefU (ncol_a x r2), rows = Yo columns
        int ry = st->ncol_a;
        for (int e = tid; e < ry * r2; e += NT) {
          int i = e % ry, q = e / ry;
          double sacc = 0.0;
          for (int t = 0; t <= q; ++t)
            if (s_kept[t] == i) sacc += Rinv[t + q * ar.ld];
          st->coefU[i + q * LDC] = sacc;
        }
      }
      __syncthreads();
      if (tid == 0) {
        if (r2 < korig) st->warn |= (arg == 0 ? skrd::W_RANK_DROP : skrd::W_REFRESH_RANK);
        if (arg == 0) {
          st->ncol_a = r2;
          st->ncol_b = r2;
          st->cm_mode = CM_U_ONLY;
          st->cm_nin_u = r;
          st->cm_nout_u = r2;
          st->cm_nin_c = 0;
          st->cm_nout_c = 0;
          if (r2 == 0) {
            st->kc = 0;
            if (st->converged || st->iters >= st->max_iter) set_done(st, -1);
          }
        } else {
          st->cm_mode = CM_REFRESH;
          st->cm_nin_c = r;
          st->cm_nout_c = r2;
          st->cm_nin_u = st->ncol_a;
          st->cm_nout_u = r2;
          st->kc = r2;
          if (r2 == 0) {
            st->ncol_a = 0;
            if (st->converged || st->iters >= st->max_iter) set_done(st, -1);
          }
        }
      }
      break;
    }
    case P_PROJ_FIN: {
      if (st->done || st->kc == 0) break;
      int kc = st->kc;
      reduce_partials(p.part, GRID_MAX, p.nblk, 2 * kc, 1, ar.red);
      if (tid == 0) {
        double rn = sqrt(ar.red[0]);
        st->rnorm = rn;
        p.hist[st->hist_len] = rn;
        st->hist_len += 1;
        st->converged = rn <= st->abs_tol ? 1 : 0;
        if (st->converged || st->iters >= st->max_iter) set_done(st, -1);
      }
      break;
    }
    case P_CYCLE: {
      if (!st->ran) break;
      ar.prof = st->prof;
      int kc = st->kc, j = st->j;
      int warn = 0;
      int r;
      if (st->k == 0) {
        r = 0;  // k == 0: plain restarted GMRES, no recycle space (gcrodr.py:326-330)
      } else if (kc == 0) {
        r = skrd::recycle_first(c, ar, st->H, LDH, j, st->k, st->coefU, LDC, st->coefC, LDC, &warn);
      } else {
        r = skrd::recycle_next(c, ar, st->H, LDH, st->B, LDB, st->dk, kc, j, st->cross, LDX, st->k,
                               st->coefU, LDC, st->coefC, LDC, &warn);
      }
      if (tid == 0) {
        st->warn |= warn;
        if (r < 0) st->status |= (1 << (-r));
        st->kc_prev = kc;
        st->comb_pending = 1;
        if (r > 0) {
          st->upd = 1;
          st->k_new = r;
          st->kc = r;
        } else {
          st->upd = 0;
          st->k_new = kc;  // unchanged (None stays None)
        }
        bool done = st->converged || (st->brk && !st->converged) || st->iters >= st->max_iter;
        if (done) {
          set_done(st, cycle_id);
        } else {
          flag_host(st, cycle_id, 0);
        }
      }
      break;
    }
    case P_FINAL: {
      reduce_partials(p.part, GRID_MAX, p.nblk, 0, 1, ar.red);
      if (tid == 0) {
        st->true_rel = st->bnorm > 0.0 ? sqrt(ar.red[0]) / st->bnorm : 0.0;
        if (st->kc == 0) st->fallback = 1;
      }
      break;
    }
  }
}

// single-CTA test entry points for the harmonic Ritz programs
__global__ void __launch_bounds__(NT) k_dense_hr(const double* H, int ldh, int m, int k,
                                                 const double* G, int ldg, const double* cross,
                                                 int ldx, double* P, int ldp, int* out) {
  extern __shared__ double dsm[];
  __shared__ int s_iw[8 * skrd::LDD];
  skrd::Ctx c = skrd::ctx();
  skrd::Arena ar = skrd::make_arena(dsm, s_iw, c.nw, skrd::LDD);
  int warn = 0;
  int r;
  if (H) {
    r = skrd::hr_first(c, ar, H, ldh, m, k, &warn);
  } else {
    for (int e = threadIdx.x; e < (m + 1) * m; e += NT)
      ar.G[(e % (m + 1)) + (e / (m + 1)) * skrd::LDD] = G[(e % (m + 1)) + (e / (m + 1)) * ldg];
    __syncthreads();
    r = skrd::hr_next(c, ar, m, cross, ldx, k, &warn);
  }
  int rows = m;
  if (r > 0)
    for (int e = threadIdx.x; e < rows * r; e += NT)
      P[(e % rows) + (e / rows) * ldp] = ar.M2[(e % rows) + (e / rows) * skrd::LDD];
  if (threadIdx.x == 0) {
    out[0] = r;
    out[1] = warn;
  }
}

// standalone SpMV / residual kernels (K1)
__global__ void __launch_bounds__(NT) k_spmv(int n, const int32_t* rp, const int32_t* ci,
                                              const double* av, const double* dg, StenView sv,
                                              const double* x, double* y) {
  const bool sten = sten_ok(sv);
  for (int row = blockIdx.x * NT + threadIdx.x; row < n; row += gridDim.x * NT) {
    double v = sten ? sten_row(sv, x, row) : csr_row(rp, ci, av, x, row);
    if (dg) v = __ddiv_rn(v, __ldg(dg + row));
    y[row] = v;
  }
}
__global__ void __launch_bounds__(NT) k_resid(int n, const int32_t* rp, const int32_t* ci,
                                               const double* av, const double* dg, StenView sv,
                                               const double* b, const double* x, double* r) {
  const bool sten = sten_ok(sv);
  for (int row = blockIdx.x * NT + threadIdx.x; row < n; row += gridDim.x * NT) {
    double v = __dsub_rn(__ldg(b + row), sten ? sten_row(sv, x, row) : csr_row(rp, ci, av, x, row));
    if (dg) v = __ddiv_rn(v, __ldg(dg + row));
    r[row] = v;
  }
}

// stencil form (skr_stencil_build): lower entries + diagonal of every row,
// then the upper entries checked bitwise against their mirrors
__global__ void __launch_bounds__(NT) k_sten_lower(int n, const int32_t* rp, const int32_t* ci,
                                                   const double* av, StenView sv) {
  int* hdr = const_cast<int*>(sv.hdr);
  double* D = const_cast<double*>(sv.D);
  double* W = const_cast<double*>(sv.W);
  double* S = const_cast<double*>(sv.S);
  double* B = const_cast<double*>(sv.B);
  for (int i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
    bool bad = false, hasd = false;
    for (int q = __ldg(rp + i), e = __ldg(rp + i + 1); q < e; ++q) {
      const int d = __ldg(ci + q) - i;
      const double v = __ldg(av + q);
      if (d == 0) {
        D[i] = v;
        hasd = true;
      } else if (d == 1 || d == sv.sx || (sv.sxy && d == sv.sxy)) {
        // upper: k_sten_upper
      } else if (v == 0.0) {
        bad = true;  // explicit zero off the diagonal: CSR would add 0 x
      } else if (d == -1) {
        W[i] = v;
      } else if (d == -sv.sx) {
        S[i] = v;
      } else if (sv.sxy && d == -sv.sxy) {
        B[i] = v;
      } else {
        bad = true;  // off the seven diagonals
      }
    }
    if (bad || !hasd) atomicOr(hdr + 1, 1);
  }
}
__global__ void __launch_bounds__(NT) k_sten_upper(int n, const int32_t* rp, const int32_t* ci,
                                                   const double* av, StenView sv) {
  int* hdr = const_cast<int*>(sv.hdr);
  for (int i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
    bool bad = false;
    int nup = 0;
    for (int q = __ldg(rp + i), e = __ldg(rp + i + 1); q < e; ++q) {
      const int d = __ldg(ci + q) - i;
      if (d <= 0) continue;
      const double v = __ldg(av + q);
      // only the three upper diagonals have a mirror array (B only in 3-D);
      // any other positive offset disqualifies the row without a load
      if (d != 1 && d != sv.sx && !(sv.sxy && d == sv.sxy)) {
        bad = true;
        continue;
      }
      const double m = d == 1 ? sv.W[i + 1] : d == sv.sx ? sv.S[i + sv.sx] : sv.B[i + sv.sxy];
      if (v == 0.0 || __double_as_longlong(v) != __double_as_longlong(m)) bad = true;
      ++nup;
    }
    // every lower entry of a later row must have this row's upper mirror
    int nmir = (sv.W[i + 1] != 0.0) + (sv.S[i + sv.sx] != 0.0) +
               (sv.sxy ? (sv.B[i + sv.sxy] != 0.0) : 0);
    if (bad || nup != nmir) atomicOr(hdr + 1, 1);
  }
}
__global__ void k_sten_final(int* hdr) { hdr[0] = hdr[1] == 0 ? 1 : 0; }

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// k_dense dynamic smem for Arnoldi length m (the arena's ld follows m, so at
// m = 40 it is ~80 KB and the kernel fits next to a cycle CTA on an SM)
static size_t dense_smem_bytes(int m = skrd::DMAX - 1) {
  return skrd::arena_doubles(NW, skrd::arena_ld(m)) * sizeof(double);
}


struct DevInfo {
  int sms = 0;
  int cycle_blocks_per_sm = 0;
  long long l2 = 0;
  bool ok = false;
};
static DevInfo g_dev[16];
static std::mutex g_mu;

// k_cycle instantiation for R rows per lane (1, 2 or 4)
static const void* cycle_kernel(int R) {
  switch (R) {
    case 1: return (const void*)k_cycle<1, 0>;
    case 2: return (const void*)k_cycle<2, 0>;
    case 4: return (const void*)k_cycle<4, 0>;
    case 8: return (const void*)k_cycle<2, 1>;   // general preconditioner, triangular kinds
    default: return (const void*)k_cycle<2, 2>;  // block Jacobi
  }
}

// rows per lane: 1 for slices of at most NT rows, else 2 (larger slices loop
// over tiles; R = 4 measured slower at N = 1M)
static int cycle_rows_per_lane(int rpb) {
  int R = rpb <= NT ? 1 : 2;
  if (const char* e = getenv("SKR_CYCLE_R")) R = std::max(1, std::min(4, atoi(e)));
  return R == 3 ? 4 : R;
}

static int ensure_dev(DevInfo** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return SKR_ERR_CUDA;
  if (dev < 0 || dev >= 16) return SKR_ERR_UNSUPPORTED;
  std::lock_guard<std::mutex> lk(g_mu);
  DevInfo& d = g_dev[dev];
  if (!d.ok) {
    if (cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return SKR_ERR_CUDA;
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    d.l2 = l2;
    if (cudaFuncSetAttribute(k_dense, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dense_smem_bytes()) != cudaSuccess)
      return SKR_ERR_CUDA;
    if (cudaFuncSetAttribute(k_dense_hr, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dense_smem_bytes()) != cudaSuccess)
      return SKR_ERR_CUDA;
    int nb = 1 << 30;
    for (int v = 0; v < 5; ++v) {
      const void* f = cycle_kernel(1 << v);
      if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)CYCLE_DSMEM_BUDGET) != cudaSuccess)
        return SKR_ERR_CUDA;
      int nbv = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbv, f, NT,
                                                        CYCLE_DSMEM_BUDGET) != cudaSuccess)
        return SKR_ERR_CUDA;
      nb = std::min(nb, nbv);
    }
    d.cycle_blocks_per_sm = nb;
    cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)CYCLE_DSMEM_BUDGET);
    const int combine_smem = 2 * LDC * KMAX * (int)sizeof(double);
    cudaFuncSetAttribute(k_combine<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, combine_smem);
    cudaFuncSetAttribute(k_combine<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, combine_smem);
    cudaFuncSetAttribute(k_combine<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, combine_smem);
    cudaFuncSetAttribute(k_combine<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, combine_smem);
    d.ok = true;
  }
  *out = &d;
  return SKR_OK;
}

// mapped host flags for the cycle look-ahead
static int* g_flags_host = nullptr;
static int* g_flags_dev = nullptr;
static std::atomic<unsigned long long> g_slot_mask{0};

static int acquire_slot(int** hptr, int** dptr) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_flags_host) {
      if (cudaHostAlloc((void**)&g_flags_host, 64 * 2 * sizeof(int), cudaHostAllocMapped) !=
          cudaSuccess)
        return -1;
      if (cudaHostGetDevicePointer((void**)&g_flags_dev, g_flags_host, 0) != cudaSuccess)
        return -1;
    }
  }
  for (int i = 0; i < 64; ++i) {
    unsigned long long bit = 1ull << i;
    unsigned long long old = g_slot_mask.fetch_or(bit);
    if (!(old & bit)) {
      *hptr = g_flags_host + 2 * i;
      *dptr = g_flags_dev + 2 * i;
      return i;
    }
  }
  return -1;
}
static void release_slot(int i) {
  if (i >= 0) g_slot_mask.fetch_and(~(1ull << i));
}

// per-thread pool of timing events (cycle kernel / dense kernel brackets)
struct EventPool {
  std::mutex mu;  // several host threads may share a stream's pool
  std::vector<cudaEvent_t> ev;
  cudaEvent_t get(size_t i) {
    std::lock_guard<std::mutex> lk(mu);
    while (ev.size() <= i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    return ev[i];
  }
};
// per-cycle timing events: a ring of EV_RING (cycle, dense) bracket triples;
// a slot's times are collected before the slot is reused
constexpr int EV_RING = 16;
// timing events per stream (reused across solves and host threads: creating
// CUDA objects in a fresh host thread while other chains' kernels run can
// stall for a long time)
static std::mutex g_pool_mu;
static std::vector<std::pair<cudaStream_t, EventPool*>> g_pools;
static EventPool& event_pool(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (auto& e : g_pools)
    if (e.first == s) return *e.second;
  g_pools.emplace_back(s, new EventPool());
  return *g_pools.back().second;
}
// the native chain driver's streams, created once and reused
static std::vector<cudaStream_t> g_chain_streams[16];
static int chain_streams(int dev, int n, std::vector<cudaStream_t>& out) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto& v = g_chain_streams[dev];
  while ((int)v.size() < n) {
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return SKR_ERR_CUDA;
    v.push_back(s);
  }
  out.assign(v.begin(), v.begin() + n);
  return SKR_OK;
}

// CTAs of the row-partitioned kernels: enough for >= SKR_ROWS_MIN (256) rows
// each, at most what is co-resident on the GPU; `grid_ctas` > 0 (skr_config)
// caps it so several concurrent chains share the SMs.
static int cfg_nblk(const DevInfo& d, int n, int grid_ctas) {
  const int maxb = std::min(GRID_MAX, d.sms * std::max(1, d.cycle_blocks_per_sm));
  int rows_min = 256;
  if (const char* e = getenv("SKR_ROWS_MIN")) rows_min = std::max(32, atoi(e));
  int want = (n + rows_min - 1) / rows_min;
  if (grid_ctas > 0) want = std::min(want, grid_ctas);
  return std::max(1, std::min(maxb, want));
}

static int launch_combine(int kt, Ptrs p, int nblk, int cycle_mode, cudaStream_t s) {
  const int smem = 2 * LDC * KMAX * (int)sizeof(double);
  if (kt <= 8)
    k_combine<8><<<nblk, NT, smem, s>>>(p, cycle_mode);
  else if (kt <= 16)
    k_combine<16><<<nblk, NT, smem, s>>>(p, cycle_mode);
  else if (kt <= 24)
    k_combine<24><<<nblk, NT, smem, s>>>(p, cycle_mode);
  else
    k_combine<32><<<nblk, NT, smem, s>>>(p, cycle_mode);
  return cudaGetLastError() == cudaSuccess ? SKR_OK : SKR_ERR_CUDA;
}

}  // namespace skr

using namespace skr;

static StenView stencil_of(const skr_csr* A) {
  if (A->stencil) return sten_view(A->stencil, A->n, A->sx, A->sxy);
  StenView v{};
  v.hdr = nullptr;
  return v;
}

extern "C" {

int skr_version(void) { return 101; }

size_t skr_stencil_bytes(int32_t n, int32_t sx, int32_t sxy) {
  if (n < 1 || sx < 2 || (sxy != 0 && sxy <= sx)) return 0;
  return sten_doubles(n, sx, sxy) * sizeof(double);
}

int skr_stencil_build(const skr_csr* A, int32_t sx, int32_t sxy, void* buf, size_t bytes,
                      void* stream) {
  if (!A || !buf || A->n < 1 || !A->row_ptr || !A->col_idx || !A->values) return SKR_ERR_ARG;
  size_t need = skr_stencil_bytes(A->n, sx, sxy);
  if (need == 0) return SKR_ERR_ARG;
  if (bytes < need) return SKR_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(buf, 0, need, s) != cudaSuccess) return SKR_ERR_CUDA;
  StenView v = sten_view(buf, A->n, sx, sxy);
  int grid = std::min(148 * 8, (A->n + NT - 1) / NT);
  k_sten_lower<<<grid, NT, 0, s>>>(A->n, A->row_ptr, A->col_idx, A->values, v);
  k_sten_upper<<<grid, NT, 0, s>>>(A->n, A->row_ptr, A->col_idx, A->values, v);
  k_sten_final<<<1, 1, 0, s>>>(const_cast<int*>(v.hdr));
  return cudaGetLastError() == cudaSuccess ? SKR_OK : SKR_ERR_CUDA;
}

const char* skr_status_string(int s) {
  switch (s) {
    case SKR_OK: return "ok";
    case SKR_ERR_ARG: return "invalid argument";
    case SKR_ERR_WORKSPACE: return "workspace too small";
    case SKR_ERR_CUDA: return "CUDA error";
    case SKR_ERR_TIMEOUT: return "timeout";
    case SKR_ERR_UNSUPPORTED: return "unsupported configuration";
  }
  return "unknown";
}

int skr_device_info(int* sm_count, long long* l2_bytes) {
  DevInfo* d;
  int rc = ensure_dev(&d);
  if (rc) return rc;
  if (sm_count) *sm_count = d->sms;
  if (l2_bytes) *l2_bytes = d->l2;
  return SKR_OK;
}

int skr_spmv(const skr_csr* A, const double* x, double* y, int apply_prec, void* stream) {
  if (!A || A->n < 0 || (A->n > 0 && (!x || !y || !A->row_ptr))) return SKR_ERR_ARG;
  if (A->n == 0) return SKR_OK;
  int grid = std::min(148 * 8, (A->n + NT - 1) / NT);
  const bool gpc = apply_prec && A->precond;
  k_spmv<<<grid, NT, 0, (cudaStream_t)stream>>>(A->n, A->row_ptr, A->col_idx, A->values,
                                                 apply_prec && !gpc ? A->diag : nullptr,
                                                 stencil_of(A), x, y);
  if (cudaGetLastError() != cudaSuccess) return SKR_ERR_CUDA;
  return gpc ? skr_precond_apply(A->precond, y, y, 1, A->n, A->n, stream) : SKR_OK;
}

int skr_residual(const skr_csr* A, const double* b, const double* x, double* r, int apply_prec,
                 void* stream) {
  if (!A || A->n < 0) return SKR_ERR_ARG;
  if (A->n == 0) return SKR_OK;
  int grid = std::min(148 * 8, (A->n + NT - 1) / NT);
  const bool gpc = apply_prec && A->precond;
  k_resid<<<grid, NT, 0, (cudaStream_t)stream>>>(A->n, A->row_ptr, A->col_idx, A->values,
                                                  apply_prec && !gpc ? A->diag : nullptr,
                                                  stencil_of(A), b, x, r);
  if (cudaGetLastError() != cudaSuccess) return SKR_ERR_CUDA;
  return gpc ? skr_precond_apply(A->precond, r, r, 1, A->n, A->n, stream) : SKR_OK;
}

size_t skr_gcrodr_workspace_bytes(int32_t n, int32_t m, int32_t k, int32_t max_iter) {
  if (n < 0 || m < 2 || k < 0 || k >= m || m + 1 > MMAX || k + 1 > KMAX || max_iter < 1) return 0;
  return make_layout(n, m, k, max_iter).total;
}

int skr_gcrodr_recycle_view(void* ws, size_t ws_bytes, int32_t n, int32_t m, int32_t k, double** U,
                            double** C, int32_t* k_out, int32_t* ld) {
  if (!ws) return SKR_ERR_ARG;
  Layout L = make_layout(n, m, k, 1);
  (void)ws_bytes;
  char* base = (char*)ws;
  State* st = (State*)(base + L.state);
  int kc = 0;
  if (cudaMemcpy(&kc, &st->kc, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
    return SKR_ERR_CUDA;
  double* basis = (double*)(base + L.basis);
  if (U) *U = basis;
  if (C) *C = basis + (size_t)(L.kcap + L.kcap - kc) * L.ld;
  if (k_out) *k_out = kc;
  if (ld) *ld = L.ld;
  return SKR_OK;
}

int skr_gcrodr_solve(const skr_csr* A, const double* b, const double* x0, double* x,
                     const skr_config* cfg, const double* U_in, int32_t ldu, int32_t k_in,
                     void* ws, size_t ws_bytes, skr_report* rep, double* hist, int32_t hist_cap,
                     double* checks, int32_t checks_cap, void* stream_) {
  if (!A || !b || !x || !cfg || !ws || !rep) return SKR_ERR_ARG;
  const int n = A->n;
  if (n <= 0 || cfg->m < 2 || cfg->k < 0 || cfg->k >= cfg->m || !(cfg->tol > 0) ||
      cfg->max_iter < 1 || cfg->grid_ctas < 0)
    return SKR_ERR_ARG;
  if (cfg->m + 1 > MMAX || cfg->k + 1 > KMAX) return SKR_ERR_UNSUPPORTED;
  if (k_in < 0 || k_in > cfg->k + 1 || (k_in > 0 && (!U_in || ldu < n))) return SKR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream_;
  DevInfo* d;
  int rc = ensure_dev(&d);
  if (rc) return rc;
  Layout L = make_layout(n, cfg->m, cfg->k, cfg->max_iter);
  if (ws_bytes < L.total) return SKR_ERR_WORKSPACE;
  char* base = (char*)ws;
  Ptrs p;
  p.st = (State*)(base + L.state);
  p.rp = A->row_ptr;
  p.ci = A->col_idx;
  p.av = A->values;
  p.pch = (PcHeader*)A->precond;
  p.dg = p.pch ? nullptr : A->diag;  // a general preconditioner replaces the Jacobi diagonal
  p.sv = stencil_of(A);
  p.b = b;
  p.x = x;
  p.r = (double*)(base + L.r);
  p.z = (double*)(base + L.z);
  p.basis = (double*)(base + L.basis);
  p.part = (double*)(base + L.part);
  p.sred = (double*)(base + L.sred);
  p.hist = (double*)(base + L.hist);
  p.checks = (double*)(base + L.checks);
  p.dlog = (double*)(base + L.dlog);
  p.n = n;
  p.ld = L.ld;
  p.kcap = L.kcap;
  const int nblk = cfg_nblk(*d, n, cfg->grid_ctas);
  int launches_pc = 0;
  p.nblk = nblk;
  p.rpb = (int)align_up((size_t)((n + nblk - 1) / nblk), 32);
  // the in-kernel (tensor-core) recycle update pays off when the row slices
  // are long; with short ones (C1 at 64 CTAs: 1,024 rows) a separate
  // k_combine on every SM has the lower latency (measured: C1 -5% fused)
  p.fuse_comb = p.rpb >= FUSE_COMB_ROWS ? 1 : 0;
  p.upd_direct = 1;
  if (const char* e = getenv("SKR_UPD_DIRECT")) p.upd_direct = atoi(e) ? 1 : 0;
  bool kupd = false;  // the DMMA update as its own launch (k_update) instead of inside k_cycle
  if (const char* e = getenv("SKR_FUSE_COMB")) {
    p.fuse_comb = atoi(e) == 1 ? 1 : 0;
    kupd = atoi(e) == 2;
  }
#ifdef SKR_NO_FUSED_UPDATE
  if (p.fuse_comb) {
    p.fuse_comb = 0;
    kupd = true;
  }
#endif
  p.v0_rtol = V0_PROJ_RTOL;
  if (const char* e = getenv("SKR_V0_RTOL")) p.v0_rtol = atof(e);
  p.gram_half = 0;
  if (const char* e = getenv("SKR_GRAM_HALF")) p.gram_half = atoi(e) ? 1 : 0;
  const bool diag = (cfg->flags & SKR_COLLECT_DIAGNOSTICS) != 0;
  if (diag) p.fuse_comb = 0;  // the update is applied before each record
  const int kt = L.kcap;
  const int k_eff = cfg->k == 0 ? 0 : k_in;
  // CSR slice cache: sized from the mean row length with headroom; CTAs whose
  // slice does not fit read the matrix from global memory instead.
  const CycleSmemLayout SL = cycle_smem_layout(cfg->m, L.kcap);
  p.sm_R = (int)SL.R;
  p.sm_B = (int)SL.B;
  p.sm_csr = (int)SL.csr;
  p.sm_cmb = (int)SL.cmb;
  const size_t cycle_fixed = SL.csr * sizeof(double);
  size_t csr_cap = 0;
  {
    double per_row = (double)A->nnz / std::max(1, n);
    size_t want = (size_t)((p.rpb + 1) * 4 + (per_row * p.rpb * 1.06 + 64) * 12 + 64);
    want = (want + 255) / 256 * 256;
    if (cycle_fixed + want <= CYCLE_DSMEM_BUDGET && !getenv("SKR_NO_CSR_CACHE")) csr_cap = want;
  }
  size_t cycle_dsmem = cycle_fixed + csr_cap;
  const size_t upd_smem =
      (SL.cmb + 2 * (size_t)((L.kcap + 7) / 8 * 8) * comb_ld(cfg->m)) * sizeof(double);
  int csr_cap_i = (int)csr_cap;
  int pc_family = 0;  // 1 triangular, 2 block Jacobi
  if (p.pch) {
    pc_family = A->precond_kind == SKR_PC_BJACOBI ? 2 : A->precond_kind > 0 ? 1 : 0;
    if (!pc_family) {  // kind not given: read it from the buffer's header
      int hk = 0;
      if (cudaMemcpyAsync(&hk, &p.pch->v.kind, sizeof(int), cudaMemcpyDeviceToHost, s) !=
              cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess)
        return SKR_ERR_CUDA;
      pc_family = hk == PC_BJACOBI ? 2 : 1;
    }
  }
  const void* cycle_fn =
      cycle_kernel(pc_family ? 8 * pc_family : cycle_rows_per_lane(p.rpb));
  int pc_target = 0, pc_stage = 0;
  void* pcargs[3] = {&p, &pc_target, &pc_stage};
  auto launch_pc = [&](int target, int stage) {
    pc_target = target;
    pc_stage = stage;
    ++launches_pc;
    return cudaLaunchCooperativeKernel((const void*)k_pc_cols, dim3(nblk), dim3(NT), pcargs, 0, s);
  };
  // k_combine is latency-bound per row: run it on >= 2 CTAs per SM (its
  // next-cycle partials are folded into nblk slots, so the grid is free)
  const int ncomb = std::max(1, std::min(std::min(GRID_MAX, std::max(nblk, 2 * d->sms)),
                                         (n + 31) / 32));

  int* hflag = nullptr;
  int* dflag = nullptr;
  int slot = acquire_slot(&hflag, &dflag);
  if (slot < 0) return SKR_ERR_CUDA;
  hflag[0] = -1;
  hflag[1] = 0;

  EventPool& t_events = event_pool(s);
  cudaEvent_t ev0 = t_events.get(0), ev1 = t_events.get(1);
  int launches = 0;
  cudaEventRecord(ev0, s);
  k_setup<<<1, NT, 0, s>>>(p.st, n, L.ld, cfg->m, cfg->k, cfg->max_iter, cfg->tol,
                           A->diag ? 1 : 0, nblk, p.rpb, k_eff, x0 ? 1 : 0, dflag);
  if (k_eff > 0 && U_in != p.basis) {
    cudaMemcpy2DAsync(p.basis, (size_t)L.ld * sizeof(double), U_in, (size_t)ldu * sizeof(double),
                      (size_t)n * sizeof(double), k_eff, cudaMemcpyDeviceToDevice, s);
  }
  k_init<<<nblk, NT, 0, s>>>(p, x0);
  if (p.pch) launch_pc(0, 0);
  const size_t dsm = dense_smem_bytes(cfg->m);
  k_dense<<<1, NT, dsm, s>>>(p, P_INIT, 0, -1);
  launches += 3;
  static const bool gram_simple = getenv("SKR_GRAM_SIMPLE") != nullptr;
  auto gram = [&](int which, int from_state) {
    if (gram_simple)
      k_gram<<<nblk, NT, 0, s>>>(p, which, from_state);
    else
      k_gram_dmma<<<nblk, NT, 0, s>>>(p, which, from_state);
  };
  if (k_eff > 0) {
    // orth(U_in): CholQR pass 1 + pass 2 with QRCP(R)
    gram(0, 0);
    k_reduce<<<8, NT, 0, s>>>(p, 0, 0);
    k_dense<<<1, NT, dsm, s>>>(p, P_CHOL1, 0, -1);
    launch_combine(kt, p, ncomb, 0, s);
    gram(0, 0);
    k_reduce<<<8, NT, 0, s>>>(p, 0, 0);
    k_dense<<<1, NT, dsm, s>>>(p, P_CHOL2, 0, -1);
    launch_combine(kt, p, ncomb, 0, s);
    // W = op(Yo) into the C block; QRCP(W) -> C, U
    k_spmm<<<nblk, NT, 0, s>>>(p);
    if (p.pch) launch_pc(1, 0);
    gram(1, 1);
    k_reduce<<<8, NT, 0, s>>>(p, 1, 0);
    k_dense<<<1, NT, dsm, s>>>(p, P_CHOL1, 1, -1);
    launch_combine(kt, p, ncomb, 0, s);
    gram(1, 1);
    k_reduce<<<8, NT, 0, s>>>(p, 1, 0);
    k_dense<<<1, NT, dsm, s>>>(p, P_CHOL2, 1, -1);
    launch_combine(kt, p, ncomb, 0, s);
    // projection alpha = C^T r ; x += U alpha ; r -= C alpha
    k_ctr<<<nblk, NT, 0, s>>>(p);
    k_reduce<<<8, NT, 0, s>>>(p, 2, 0);
    k_project<<<nblk, NT, 0, s>>>(p);
    k_dense<<<1, NT, dsm, s>>>(p, P_PROJ_FIN, 0, -1);
    launches += 21;
    if (diag) {
      if (p.pch) launch_pc(2, 0);
      k_diag<<<nblk, NT, 0, s>>>(p, 0);
      k_diag_fin<<<1, NT, 0, s>>>(p, 0);
      launches += 2;
    }
  }
  if (cudaGetLastError() != cudaSuccess) {
    release_slot(slot);
    return SKR_ERR_CUDA;
  }
  double cyc_ms = 0.0, den_ms = 0.0;
  auto collect = [&](int c2) {  // cycle c2's kernel times (its events are recorded)
    const size_t sl = 3 * (size_t)(c2 % EV_RING);
    cudaEventSynchronize(t_events.get(4 + sl));
    float a = 0.f, b2 = 0.f;
    cudaEventElapsedTime(&a, t_events.get(2 + sl), t_events.get(3 + sl));
    cudaEventElapsedTime(&b2, t_events.get(3 + sl), t_events.get(4 + sl));
    cyc_ms += a;
    den_ms += b2;
  };
  // cycles with look-ahead
  const int LOOK = 2;
  int enq = 0, seen = 0;
  int result = SKR_OK;
  void* cargs[3];
  int cyc = 0;
  cargs[0] = &p;
  cargs[1] = &cyc;
  cargs[2] = &csr_cap_i;
  auto t_last = std::chrono::steady_clock::now();
  while (true) {
    volatile int* vf = hflag;
    if (vf[1]) break;
    while (enq < seen + LOOK) {
      cyc = enq;
      if (enq >= EV_RING) collect(enq - EV_RING);
      const size_t slot3 = 3 * (size_t)(enq % EV_RING);
      cudaEventRecord(t_events.get(2 + slot3), s);
      cudaError_t e =
          cudaLaunchCooperativeKernel(cycle_fn, dim3(nblk), dim3(NT), cargs, cycle_dsmem, s);
      if (e != cudaSuccess) {
        result = SKR_ERR_CUDA;
        break;
      }
      cudaEventRecord(t_events.get(3 + slot3), s);
      k_dense<<<1, NT, dsm, s>>>(p, P_CYCLE, 0, enq);
      cudaEventRecord(t_events.get(4 + slot3), s);
      launches += 2;
      // fused: the update is applied at the start of the next k_cycle
      if (!p.fuse_comb) {
        if (kupd)
          k_update<<<nblk, NT, upd_smem, s>>>(p);
        else
          launch_combine(kt, p, ncomb, 1, s);
        ++launches;
      }
      if (diag) {
        if (p.pch) launch_pc(2, 1);
        k_diag<<<nblk, NT, 0, s>>>(p, 1);
        k_diag_fin<<<1, NT, 0, s>>>(p, 1);
        launches += 2;
      }
      ++enq;
    }
    if (result) break;
    // wait for cycle `seen` to be processed (or done). The mapped flag is
    // polled with a short sleep; the driver (cudaStreamQuery) is asked only
    // every ~64 polls -- several chains' threads spinning on it contend for
    // the driver lock that their kernel launches also need. The look-ahead
    // keeps LOOK cycles queued, so the poll latency does not idle the GPU.
    unsigned polls = 0;
    while (true) {
      if (vf[1]) break;
      if (vf[0] >= seen) break;
      if ((++polls & 63) != 0) {
        std::this_thread::sleep_for(std::chrono::microseconds(5));
        continue;
      }
      cudaError_t q = cudaStreamQuery(s);
      if (q == cudaSuccess) {
        // stream drained: either done (flag) or stalled; re-check
        if (vf[1] || vf[0] >= seen) break;
        // nothing pending and no progress flag: the state says done
        int hdone = 0;
        cudaMemcpyAsync(&hdone, &p.st->done, sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (hdone) {
          vf[1] = 1;
          break;
        }
        if (vf[0] < seen) {
          // the cycle ran without flagging: count it as processed
          break;
        }
      } else if (q != cudaErrorNotReady) {
        result = SKR_ERR_CUDA;
        break;
      }
      auto now = std::chrono::steady_clock::now();
      if (std::chrono::duration_cast<std::chrono::seconds>(now - t_last).count() > 120) {
        result = SKR_ERR_TIMEOUT;
        break;
      }
    }
    if (result) break;
    t_last = std::chrono::steady_clock::now();
    if (vf[1]) break;
    ++seen;
  }
  // the last cycle's update if no look-ahead k_cycle launch applied it
  if (p.fuse_comb) launch_combine(kt, p, ncomb, 1, s);
  k_final_resid<<<nblk, NT, 0, s>>>(p);
  k_dense<<<1, NT, dsm, s>>>(p, P_FINAL, 0, -1);
  launches += 3 + p.fuse_comb;  // incl. k_setup
  cudaEventRecord(ev1, s);
  if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess)
    result = SKR_ERR_CUDA;
  release_slot(slot);
  if (result) return result;
  std::vector<char> hbuf(offsetof(State, kept));
  // stream-ordered reads (never the legacy default stream: other chains run
  // concurrently on their own streams)
  cudaMemcpyAsync(hbuf.data(), p.st, offsetof(State, kept), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  const State& hs = *reinterpret_cast<const State*>(hbuf.data());
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  for (int c2 = std::max(0, enq - EV_RING); c2 < enq; ++c2) collect(c2);
  if (hs.abort_flag) return SKR_ERR_TIMEOUT;
  memset(rep, 0, sizeof(*rep));
  rep->iterations = hs.iters;
  rep->converged = hs.converged;
  rep->k_out = hs.kc;
  rep->hist_len = hs.hist_len;
  rep->n_checks = hs.nchecks;
  rep->deflated_steps = hs.defl_steps;
  rep->warn_bits = hs.warn;
  rep->status_bits = hs.status;
  rep->zero_rhs = hs.zero_rhs;
  rep->gmres_fallback = hs.kc == 0 ? 1 : 0;
  rep->cycles = hs.cycles;
  rep->v0_projections = hs.v0proj;
  rep->true_relative_residual = hs.true_rel;
  rep->rnorm = hs.rnorm;
  rep->abs_tol = hs.abs_tol;
  rep->bnorm = hs.bnorm;
  rep->device_ms = ms;
  rep->spmv_ortho_bytes = hs.step_bytes;
  rep->cycle_kernel_ms = cyc_ms;
  rep->dense_kernel_ms = den_ms;
  rep->launches = launches + launches_pc;
  rep->arnoldi_steps = hs.steps;
  if (hist && hist_cap > 0)
    cudaMemcpyAsync(hist, p.hist, sizeof(double) * std::min(hist_cap, hs.hist_len),
                    cudaMemcpyDeviceToHost, s);
  if (checks && checks_cap > 0)
    cudaMemcpyAsync(checks, p.checks, sizeof(double) * 2 * std::min(checks_cap, hs.nchecks),
                    cudaMemcpyDeviceToHost, s);
  if ((hist && hist_cap > 0) || (checks && checks_cap > 0)) cudaStreamSynchronize(s);
  return SKR_OK;
}

int skr_gcrodr_solve_chains(const skr_system* systems, const int32_t* chain_first,
                            int32_t n_chains, const skr_config* cfg, void* const* workspaces,
                            size_t ws_bytes, const double* const* U_first,
                            const int32_t* ldu_first, const int32_t* k_first,
                            skr_report* reports) {
  if (!systems || !chain_first || n_chains < 1 || !cfg || !workspaces || !reports)
    return SKR_ERR_ARG;
  for (int c = 0; c < n_chains; ++c)
    if (chain_first[c + 1] < chain_first[c] || !workspaces[c]) return SKR_ERR_ARG;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return SKR_ERR_CUDA;
  if (dev < 0 || dev >= 16) return SKR_ERR_UNSUPPORTED;
  DevInfo* dinfo;
  if (int rc0 = ensure_dev(&dinfo)) return rc0;
  std::vector<cudaStream_t> streams;
  if (int rc0 = chain_streams(dev, n_chains, streams)) return rc0;
  for (int c = 0; c < n_chains; ++c) {  // event pools up front, on this thread
    EventPool& ep = event_pool(streams[c]);
    ep.get(2 + 3 * EV_RING);
  }
  std::vector<int> status(n_chains, SKR_OK);
  auto run_chain = [&](int c) {
    if (cudaSetDevice(dev) != cudaSuccess) {
      status[c] = SKR_ERR_CUDA;
      return;
    }
    cudaStream_t s = streams[c];
    if (getenv("SKR_TRACE"))
      fprintf(stderr, "trace chain %d start_us %lld\n", c,
              (long long)std::chrono::duration_cast<std::chrono::microseconds>(
                  std::chrono::steady_clock::now().time_since_epoch())
                  .count());
    const double* U = U_first ? U_first[c] : nullptr;
    int ldu = ldu_first ? ldu_first[c] : 0;
    int k = k_first ? k_first[c] : 0;
    if (!U) k = 0;
    static const bool trace = getenv("SKR_TRACE") != nullptr;
    for (int i = chain_first[c]; i < chain_first[c + 1]; ++i) {
      const skr_system& sy = systems[i];
      const auto h0 = std::chrono::steady_clock::now();
      int rc = skr_gcrodr_solve(&sy.A, sy.b, nullptr, sy.x, cfg, k > 0 ? U : nullptr, ldu, k,
                                workspaces[c], ws_bytes, &reports[i], nullptr, 0, nullptr, 0, s);
      if (trace) {
        const auto h1 = std::chrono::steady_clock::now();
        auto us = [](std::chrono::steady_clock::time_point t) {
          return (long long)std::chrono::duration_cast<std::chrono::microseconds>(
                     t.time_since_epoch()).count();
        };
        fprintf(stderr, "trace chain %d sys %d host_us %lld %lld device_ms %.3f its %d\n", c, i,
                us(h0), us(h1), reports[i].device_ms, reports[i].iterations);
      }
      if (rc != SKR_OK) {
        status[c] = rc;
        break;
      }
      // the next system refreshes from the U this solve left in the workspace
      if (cfg->k > 0 && !reports[i].zero_rhs) {
        double* Uw = nullptr;
        int32_t kw = 0, ldw = 0;
        Layout L = make_layout(sy.A.n, cfg->m, cfg->k, cfg->max_iter);
        Uw = (double*)((char*)workspaces[c] + L.basis);
        kw = reports[i].k_out;
        ldw = L.ld;
        U = Uw;
        ldu = ldw;
        k = kw;
      }
    }
    cudaStreamSynchronize(s);
  };
  std::vector<std::thread> th;
  th.reserve(n_chains);
  for (int c = 0; c < n_chains; ++c) th.emplace_back(run_chain, c);
  for (auto& t : th) t.join();
  for (int c = 0; c < n_chains; ++c)
    if (status[c] != SKR_OK) return status[c];
  return SKR_OK;
}

int skr_gcrodr_diagnostics(void* ws, size_t ws_bytes, int32_t n, int32_t m, int32_t k,
                           int32_t max_iter, double* out, int32_t cap) {
  if (!ws || (!out && cap > 0) || max_iter < 1) return -SKR_ERR_ARG;
  Layout L = make_layout(n, m, k, max_iter);
  if (ws_bytes < L.total) return -SKR_ERR_WORKSPACE;
  const State* st = (const State*)((char*)ws + L.state);
  int nd = 0;
  if (cudaMemcpy(&nd, &st->ndiag, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -SKR_ERR_CUDA;
  const int ncopy = std::min(nd, cap);
  if (ncopy > 0 &&
      cudaMemcpy(out, (char*)ws + L.dlog, sizeof(double) * 4 * ncopy, cudaMemcpyDeviceToHost) !=
          cudaSuccess)
    return -SKR_ERR_CUDA;
  return nd;
}

int skr_gcrodr_profile(void* ws, size_t ws_bytes, int32_t n, int32_t m, int32_t k,
                       long long* out32) {
  if (!ws || !out32) return SKR_ERR_ARG;
  (void)ws_bytes;
  Layout L = make_layout(n, m, k, 1);
  State* st = (State*)((char*)ws + L.state);
  if (cudaMemcpy(out32, st->prof, 32 * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return SKR_ERR_CUDA;
  return SKR_OK;
}

int skr_dense_hr_first(const double* H, int32_t ldh, int32_t m, int32_t k, double* P, int32_t ldp,
                       int32_t* ncols, void* stream) {
  if (!H || !P || !ncols || m < 1 || m > skrd::DMAX || ldh < m + 1 || ldp < m) return SKR_ERR_ARG;
  DevInfo* d;
  int rc = ensure_dev(&d);
  if (rc) return rc;
  int* dout;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMallocAsync((void**)&dout, 2 * sizeof(int), s) != cudaSuccess) return SKR_ERR_CUDA;
  k_dense_hr<<<1, NT, dense_smem_bytes(), s>>>(H, ldh, m, k, nullptr, 0, nullptr, 0, P, ldp, dout);
  int hout[2] = {0, 0};
  cudaMemcpyAsync(hout, dout, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(dout, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return SKR_ERR_CUDA;
  ncols[0] = hout[0];
  ncols[1] = hout[1];
  return SKR_OK;
}

int skr_dense_hr_next(const double* G, int32_t ldg, const double* cross, int32_t ldx, int32_t mm,
                      int32_t k, double* P, int32_t ldp, int32_t* ncols, void* stream) {
  if (!G || !cross || !P || !ncols || mm < 1 || mm + 1 > skrd::LDD || ldg < mm + 1 || ldx < mm ||
      ldp < mm)
    return SKR_ERR_ARG;
  DevInfo* d;
  int rc = ensure_dev(&d);
  if (rc) return rc;
  int* dout;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMallocAsync((void**)&dout, 2 * sizeof(int), s) != cudaSuccess) return SKR_ERR_CUDA;
  k_dense_hr<<<1, NT, dense_smem_bytes(), s>>>(nullptr, 0, mm, k, G, ldg, cross, ldx, P, ldp,
                                                dout);
  int hout[2] = {0, 0};
  cudaMemcpyAsync(hout, dout, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(dout, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return SKR_ERR_CUDA;
  ncols[0] = hout[0];
  ncols[1] = hout[1];
  return SKR_OK;
}

}  // extern "C"
