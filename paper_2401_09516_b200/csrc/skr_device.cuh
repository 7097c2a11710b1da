// Shared device helpers: CSR row kernel (bit-exact with scipy csr_matvec),
// grid barrier with timeout for cooperative persistent kernels, block/warp
// reductions over per-CTA partial sums.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/skr.h"

namespace skr {

constexpr int NT = 256;              // threads per CTA (streaming kernels)
constexpr int NW = NT / 32;          // warps per CTA
constexpr int KMAX = 32;             // max recycle columns incl. pair widening (k+1)
constexpr int MMAX = 64;             // max Arnoldi columns (m + 1)
constexpr int GRID_MAX = 1184;       // max persistent CTAs (148 SMs x 8)
constexpr int PV_STEP = 2 * (KMAX + MMAX) + 8;      // reduction values per Arnoldi step
constexpr int PV_MAX = MMAX * MMAX;  // largest reduction (cross-Gram mm x mm)
constexpr unsigned long long BARRIER_TIMEOUT_NS = 8000000000ull;  // 8 s

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// y_i = sum_k a_ik x_k, sequential in column order from 0.0, separate multiply
// and add (scipy sparsetools csr_matvec). x may be written by the
// running kernel, so it is read through the coherent path.
__device__ __forceinline__ double csr_row(const int32_t* __restrict__ rp,
                                          const int32_t* __restrict__ ci,
                                          const double* __restrict__ av, const double* x, int r) {
  int s = __ldg(rp + r), e = __ldg(rp + r + 1);
  double acc = 0.0;
  for (int q = s; q < e; ++q) acc = __dadd_rn(acc, __dmul_rn(__ldg(av + q), x[__ldg(ci + q)]));
  return acc;
}

// Symmetric 7-diagonal ("stencil") form of a CSR matrix whose entries lie on
// the diagonals {0, +-1, +-sx, +-sxy} (5-/7-point finite-difference operators
// in natural ordering), with A(i, i+d) == A(i+d, i) bitwise, nonzero
// off-diagonal entries and a diagonal entry in every row. Stored as the
// diagonal D and the lower entries W (d = -1), S (-sx), B (-sxy), each
// zero-padded past n so the upper entries W[i+1], S[i+sx], B[i+sxy] need no
// bounds test; a zero coefficient marks an absent entry. Built and verified
// on the device by skr_stencil_build; hdr[0] == 1 when the matrix qualified.
// 24 (2-D) or 32 (3-D) bytes per row instead of CSR's 64 / 88.
struct StenView {
  const int* hdr;  // nullptr: no stencil form
  const double* D;
  const double* W;
  const double* S;
  const double* B;  // nullptr in 2-D (sxy == 0)
  int n, sx, sxy;
};
constexpr int STEN_HDR_DOUBLES = 8;  // 64-byte header: int ok, int fail, ...

__host__ __device__ inline size_t sten_doubles(int n, int sx, int sxy) {
  return (size_t)STEN_HDR_DOUBLES + (size_t)n + (size_t)(n + 1) + (size_t)(n + sx) +
         (sxy ? (size_t)(n + sxy) : 0);
}
__host__ __device__ inline StenView sten_view(const void* buf, int n, int sx, int sxy) {
  StenView v;
  const double* d = (const double*)buf;
  v.hdr = (const int*)buf;
  v.D = d + STEN_HDR_DOUBLES;
  v.W = v.D + n;
  v.S = v.W + (n + 1);
  v.B = sxy ? v.S + (n + sx) : nullptr;
  v.n = n;
  v.sx = sx;
  v.sxy = sxy;
  return v;
}
__device__ __forceinline__ bool sten_ok(const StenView& v) {
  return v.hdr != nullptr && *(const volatile int*)v.hdr == 1;
}

// Row i of A x in CSR column order (i - sxy, i - sx, i - 1, i, i + 1, i + sx,
// i + sxy) with the same separate round-to-nearest multiply and add as
// csr_row and absent entries skipped: bit-identical to csr_row on the CSR the
// form was built from. x loads are clamped in range and issued up front.
// Coefficients are read at index c (c = i for the global arrays, i - r0 for a
// CTA's shared-memory slice whose S part starts at row r0 as well).
template <bool GLOBAL>
__device__ __forceinline__ double sten_row_at(const double* D, const double* W, const double* S,
                                              const double* B, int sx, int sxy, int n,
                                              const double* x, int i, int c) {
  const int n1 = n - 1;
  auto ld = [](const double* q) { return GLOBAL ? __ldg(q) : *q; };
  double cb = 0.0, ct = 0.0, xb = 0.0, xt = 0.0;
  if (sxy) {
    cb = ld(B + c);
    ct = ld(B + c + sxy);
    xb = x[max(i - sxy, 0)];
    xt = x[min(i + sxy, n1)];
  }
  const double cs = ld(S + c), cn = ld(S + c + sx);
  const double cw = ld(W + c), ce = ld(W + c + 1), cd = ld(D + c);
  const double xs = x[max(i - sx, 0)], xn = x[min(i + sx, n1)];
  const double xw = x[max(i - 1, 0)], xe = x[min(i + 1, n1)], xd = x[i];
  double acc = 0.0;
  if (cb != 0.0) acc = __dadd_rn(acc, __dmul_rn(cb, xb));
  if (cs != 0.0) acc = __dadd_rn(acc, __dmul_rn(cs, xs));
  if (cw != 0.0) acc = __dadd_rn(acc, __dmul_rn(cw, xw));
  acc = __dadd_rn(acc, __dmul_rn(cd, xd));
  if (ce != 0.0) acc = __dadd_rn(acc, __dmul_rn(ce, xe));
  if (cn != 0.0) acc = __dadd_rn(acc, __dmul_rn(cn, xn));
  if (ct != 0.0) acc = __dadd_rn(acc, __dmul_rn(ct, xt));
  return acc;
}
__device__ __forceinline__ double sten_row(const StenView& v, const double* x, int i) {
  return sten_row_at<true>(v.D, v.W, v.S, v.B, v.sx, v.sxy, v.n, x, i, i);
}

__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Grid-wide barrier for a cooperatively launched kernel. Thread 0 of each CTA
// arrives on a 64-bit counter that is never reset within a solve: barrier b
// (counted from the start of the solve) is complete when the counter reaches
// nblk * (b + 1), which every CTA polls for directly (no separate generation
// word, so the last arriver does no extra round trip; a fire-and-forget
// red.release arrival measured slower than fence + atomicAdd). `seen` is thread 0's
// count of completed barriers (counter / nblk, read once per launch with
// ld_relaxed_gpu64 while no barrier is in flight). A spin longer than
// BARRIER_TIMEOUT_NS sets *abort and returns false (uniform across the CTA)
// instead of hanging the GPU.
__device__ __forceinline__ unsigned long long ld_relaxed_gpu64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ bool grid_sync(unsigned long long* count, int* abort_flag, unsigned nblk,
                                          int* s_flag, unsigned long long& seen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int aborted = 0;
    const unsigned long long target = (seen + 1ull) * nblk;
    fence_acq_rel_gpu();  // release this CTA's writes (block-scope ordered by bar.sync)
    const unsigned long long arrived = atomicAdd(count, 1ull) + 1ull;
    if (arrived < target) {
      unsigned long long t0 = gtimer();
      unsigned polls = 0;
      while (ld_relaxed_gpu64(count) < target) {
        __nanosleep(polls < 64 ? 20 : 100);
        if ((++polls & 255) == 0) {
          if (gtimer() - t0 > BARRIER_TIMEOUT_NS) {
            atomicExch(abort_flag, 1);
            aborted = 1;
            break;
          }
          if (ld_relaxed_gpu(reinterpret_cast<unsigned*>(abort_flag))) {
            aborted = 1;
            break;
          }
        }
      }
    }
    seen += 1ull;
    fence_acq_rel_gpu();  // acquire the other CTAs' writes
    *s_flag = aborted;
  }
  __syncthreads();
  return *s_flag == 0;
}

// Sum over CTAs of partial values part[v * pstride + b], b < nblk, for
// v in [v0, v0 + nv), into out[v - v0]. Deterministic: every CTA (and every
// call) sums in the same order. Block-cooperative; ends with __syncthreads.
__device__ __forceinline__ void reduce_partials(const double* part, int pstride, int nblk, int v0,
                                                int nv, double* out) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int v = v0 + warp; v < v0 + nv; v += NW) {
    const double* p = part + (size_t)v * pstride;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += p[b];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    s = __shfl_sync(0xffffffffu, s, 0);
    if (lane == 0) out[v - v0] = s;
  }
  __syncthreads();
}

// Block sums of three values per thread (results valid in every thread).
__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* s_red) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  __syncthreads();
  if (lane == 0) {
    s_red[3 * warp] = a;
    s_red[3 * warp + 1] = b;
    s_red[3 * warp + 2] = c;
  }
  __syncthreads();
  a = b = c = 0.0;
  for (int w = 0; w < NW; ++w) {
    a += s_red[3 * w];
    b += s_red[3 * w + 1];
    c += s_red[3 * w + 2];
  }
}

// Block sum of one value per thread (result valid in every thread).
__device__ __forceinline__ double block_sum(double v, double* s_red) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < NW; ++w) t += s_red[w];
  return t;
}

}  // namespace skr
