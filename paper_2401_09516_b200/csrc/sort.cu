// Greedy nearest-neighbour ordering of the system batch on the GPU
// (kryrec/sorting.py:55-80, Alg. 1 of the paper).
//
// 1. squared distances D2[i][j] = sum_p (a_ip - a_jp)^2:
//    * binary batches (every parameter in {v0, v1}, (v1-v0)^2 integral): bit-pack
//      and D2 = (v1-v0)^2 * popcount(xor) -- exact, hence bit-identical to the
//      reference's pairwise-summed distances;
//    * otherwise an fp64 64x64-tiled difference kernel (sub + FMA, chunked sums).
// 2. the greedy chain: one CTA, visited bitmap in shared memory, per step a
//    masked arg-min of sqrt(D2[last, :]) with the lowest-index tie-break. For
//    non-exact D2 the arg-min is CERTIFIED: when any other candidate lies
//    within a 1e-10 relative window of the best, every candidate in the window
//    is re-evaluated in the reference's exact arithmetic (numpy pairwise
//    summation of fl(fl(a-b)^2), zero start, correctly rounded sqrt) and the
//    first minimum wins, exactly as np.argmin over np.linalg.norm(axis=1).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/skr.h"

namespace skrsort {

constexpr int TS = 64;     // distance tile
constexpr int TK = 16;     // k-chunk
constexpr int CHAIN_NT = 1024;
constexpr double CERT_RTOL = 1e-10;

// ---------------------------------------------------------------------------
// binary detection
// ---------------------------------------------------------------------------
__global__ void k_minmax(const double* __restrict__ a, int64_t total, double* part) {
  double mn = INFINITY, mx = -INFINITY;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = __ldg(a + i);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  __shared__ double smn[32], smx[32];
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    mn = fmin(mn, smn[0]);
    mx = fmax(mx, smx[0]);
    part[2 * blockIdx.x] = mn;
    part[2 * blockIdx.x + 1] = mx;
  }
}

__global__ void k_minmax_final(double* part, int nb, double* out) {
  if (threadIdx.x == 0) {
    double mn = INFINITY, mx = -INFINITY;
    for (int b = 0; b < nb; ++b) {
      mn = fmin(mn, part[2 * b]);
      mx = fmax(mx, part[2 * b + 1]);
    }
    out[0] = mn;
    out[1] = mx;
  }
}

__global__ void k_two_valued(const double* __restrict__ a, int64_t total, const double* mm,
                             int* bad) {
  double v0 = mm[0], v1 = mm[1];
  int local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = __ldg(a + i);
    if (v != v0 && v != v1) local = 1;
  }
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(bad, 1);
}

__global__ void k_pack(const double* __restrict__ a, int n_sys, int64_t P, int64_t W, double v1,
                       unsigned long long* bits) {
  int64_t total = (int64_t)n_sys * W;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / W, w = e % W;
    const double* row = a + i * P + w * 64;
    int64_t lim = min((int64_t)64, P - w * 64);
    unsigned long long word = 0;
    for (int64_t b = 0; b < lim; ++b)
      if (__ldg(row + b) == v1) word |= (1ull << b);
    bits[e] = word;
  }
}

// D2 tile of Hamming distances x delta2 ; rows [row0,row1), cols all
__global__ void __launch_bounds__(256) k_hamming(const unsigned long long* __restrict__ bits,
                                                 int n_sys, int64_t W, int row0, int row1,
                                                 double delta2, double* D2) {
  __shared__ unsigned long long sa[32][33], sb[32][33];
  int ti = threadIdx.x / 32, tj = threadIdx.x % 32;  // 8 x 32 threads, 4 rows each
  int i0 = row0 + blockIdx.y * 32, j0 = blockIdx.x * 32;
  if (i0 >= row1) return;
  unsigned long long cnt[4] = {0, 0, 0, 0};
  for (int64_t w0 = 0; w0 < W; w0 += 32) {
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      int r = e / 32, c = e % 32;
      int64_t w = w0 + c;
      int gi = i0 + r, gj = j0 + r;
      sa[r][c] = (gi < row1 && w < W) ? bits[(int64_t)gi * W + w] : 0ull;
      sb[r][c] = (gj < n_sys && w < W) ? bits[(int64_t)gj * W + w] : 0ull;
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
      unsigned long long bj = sb[tj][c];
#pragma unroll
      for (int q = 0; q < 4; ++q) cnt[q] += __popcll(sa[ti * 4 + q][c] ^ bj);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int gi = i0 + ti * 4 + q, gj = j0 + tj;
    if (gi < row1 && gj < n_sys) D2[(int64_t)(gi - row0) * n_sys + gj] = (double)cnt[q] * delta2;
  }
}

// fp64 difference tiles: D2[i][j] = sum (a_i - a_j)^2, rows [row0,row1).
// symmetric mode (row0 == 0, row1 == n): only tiles bj >= bi, mirrored.
__global__ void __launch_bounds__(256) k_dist2(const double* __restrict__ a, int n_sys, int64_t P,
                                               int row0, int row1, int symmetric, double* D2) {
  int bi = blockIdx.y, bj = blockIdx.x;
  if (symmetric && bj < bi) return;
  int i0 = row0 + bi * TS, j0 = bj * TS;
  if (i0 >= row1) return;
  __shared__ double sa[TK][TS + 1], sb[TK][TS + 1];
  int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 16 x 16 threads, 4 x 4 outputs each
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  for (int64_t k0 = 0; k0 < P; k0 += TK) {
    for (int e = threadIdx.x; e < TS * TK; e += 256) {
      int r = e / TK, kk = e % TK;
      int64_t k = k0 + kk;
      int gi = i0 + r, gj = j0 + r;
      sa[kk][r] = (gi < row1 && k < P) ? __ldg(a + (int64_t)gi * P + k) : 0.0;
      sb[kk][r] = (gj < n_sys && k < P) ? __ldg(a + (int64_t)gj * P + k) : 0.0;
    }
    __syncthreads();
    double part[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) part[u][v] = 0.0;
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = sa[kk][ty * 4 + u];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = sb[kk][tx * 4 + v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          double d = av[u] - bv[v];
          part[u][v] = fma(d, d, part[u][v]);
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] += part[u][v];
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      int gi = i0 + ty * 4 + u, gj = j0 + tx * 4 + v;
      if (gi < row1 && gj < n_sys) {
        D2[(int64_t)(gi - row0) * n_sys + gj] = acc[u][v];
        if (symmetric && bj > bi) D2[(int64_t)gj * n_sys + gi] = acc[u][v];
      }
    }
}

// numpy pairwise_sum_DOUBLE over t_k = fl(fl(p_k - q_k)^2), k in [off, off+n)
__device__ double pw_leaf(const double* p, const double* q, int64_t off, int64_t n) {
  auto term = [&](int64_t k) {
    double d = __dsub_rn(p[off + k], q[off + k]);
    return __dmul_rn(d, d);
  };
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, term(i));
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = term(j);
  int64_t i = 8, stop = n - (n % 8);
  for (; i < stop; i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], term(i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, term(i));
  return res;
}

__device__ double reference_distance(const double* p, const double* q, int64_t P) {
  struct Fr {
    int64_t off, n;
    int state;
    double left;
  };
  Fr st[48];
  int sp = 0;
  st[0] = {0, P, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Fr& f = st[sp];
    if (f.n <= 128) {
      ret = pw_leaf(p, q, f.off, f.n);
      --sp;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp + 1] = {f.off, n2, 0, 0.0};
      ++sp;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.off + n2, f.n - n2, 0, 0.0};
      ++sp;
    } else {
      ret = __dadd_rn(f.left, ret);
      --sp;
    }
  }
  return __dsqrt_rn(__dadd_rn(0.0, ret));
}

__device__ __forceinline__ bool better(double d, int j, double bd, int bj) {
  return d < bd || (d == bd && j < bj);
}

// Single-CTA greedy chain.
__global__ void __launch_bounds__(CHAIN_NT) k_chain(const double* __restrict__ D2,
                                                    const double* __restrict__ params, int n_sys,
                                                    int64_t P, int exact, int* order,
                                                    int* n_cert) {
  extern __shared__ unsigned int visited[];  // bitmap
  __shared__ double s_bd[32], s_sd[32];
  __shared__ int s_bj[32];
  __shared__ int s_pick, s_need;
  __shared__ double s_win;
  __shared__ double s_xd[CHAIN_NT];
  __shared__ int s_xj[CHAIN_NT];
  int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  int words = (n_sys + 31) / 32;
  for (int w = tid; w < words; w += blockDim.x) visited[w] = 0u;
  __syncthreads();
  if (tid == 0) {
    visited[0] |= 1u;
    order[0] = 0;
    *n_cert = 0;
  }
  __syncthreads();
  int last = 0;
  for (int step = 1; step < n_sys; ++step) {
    const double* row = D2 + (int64_t)last * n_sys;
    double bd = INFINITY, sd = INFINITY;
    int bj = 0x7fffffff;
    for (int j = tid; j < n_sys; j += blockDim.x) {
      if (visited[j >> 5] & (1u << (j & 31))) continue;
      double d = __dsqrt_rn(row[j]);
      if (better(d, j, bd, bj)) {
        sd = bd;
        bd = d;
        bj = j;
      } else if (d < sd) {
        sd = d;
      }
    }
    // warp reduce (best, index) and second best value
    for (int o = 16; o > 0; o >>= 1) {
      double obd = __shfl_xor_sync(0xffffffffu, bd, o);
      int obj = __shfl_xor_sync(0xffffffffu, bj, o);
      double osd = __shfl_xor_sync(0xffffffffu, sd, o);
      if (better(obd, obj, bd, bj)) {
        sd = fmin(bd, osd);
        bd = obd;
        bj = obj;
      } else {
        sd = fmin(sd, obd);
        sd = fmin(sd, osd);
      }
    }
    if (lane == 0) {
      s_bd[warp] = bd;
      s_bj[warp] = bj;
      s_sd[warp] = sd;
    }
    __syncthreads();
    if (tid == 0) {
      double B = s_bd[0], Sd = s_sd[0];
      int Bj = s_bj[0];
      for (int w = 1; w < nw; ++w) {
        if (better(s_bd[w], s_bj[w], B, Bj)) {
          Sd = fmin(B, Sd);
          B = s_bd[w];
          Bj = s_bj[w];
        } else {
          Sd = fmin(Sd, s_bd[w]);
        }
        Sd = fmin(Sd, s_sd[w]);
      }
      s_pick = Bj;
      s_win = B * (1.0 + CERT_RTOL) + 1e-300;
      s_need = (!exact && Sd <= s_win) ? 1 : 0;
    }
    __syncthreads();
    if (s_need) {
      // exact re-evaluation of every candidate inside the window
      double win = s_win;
      double xb = INFINITY;
      int xj = 0x7fffffff;
      const double* pl = params + (int64_t)last * P;
      for (int j = tid; j < n_sys; j += blockDim.x) {
        if (visited[j >> 5] & (1u << (j & 31))) continue;
        double d = __dsqrt_rn(row[j]);
        if (d <= win) {
          double e = reference_distance(params + (int64_t)j * P, pl, P);
          if (better(e, j, xb, xj)) {
            xb = e;
            xj = j;
          }
        }
      }
      s_xd[tid] = xb;
      s_xj[tid] = xj;
      __syncthreads();
      if (tid == 0) {
        double B = s_xd[0];
        int Bj = s_xj[0];
        for (int t = 1; t < (int)blockDim.x; ++t)
          if (better(s_xd[t], s_xj[t], B, Bj)) {
            B = s_xd[t];
            Bj = s_xj[t];
          }
        s_pick = Bj;
        *n_cert += 1;
      }
      __syncthreads();
    }
    int pick = s_pick;
    if (tid == 0) {
      order[step] = pick;
      visited[pick >> 5] |= (1u << (pick & 31));
    }
    last = pick;
    __syncthreads();
  }
}

struct SortLayout {
  size_t part, mm, bad, bits, d2, total;
};
static SortLayout sort_layout(int n_sys, int64_t P) {
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  SortLayout L;
  size_t off = 0;
  L.part = off;
  off = al(off + 2 * 1184 * sizeof(double));
  L.mm = off;
  off = al(off + 2 * sizeof(double));
  L.bad = off;
  off = al(off + sizeof(int) * 4);
  L.bits = off;
  int64_t W = (P + 63) / 64;
  off = al(off + (size_t)n_sys * W * sizeof(unsigned long long));
  L.d2 = off;
  off = al(off + (size_t)n_sys * n_sys * sizeof(double));
  L.total = off;
  return L;
}


// ---------------------------------------------------------------------------
// grouped_sort's first principal coordinate (sorting.py:96-105) without the
// SVD of the centered batch: the Gram matrix of the centered rows is the
// double-centered distance matrix, G = -1/2 J D2 J (J = I - 11^T / n), and the
// reference's key = centered @ vt[0] is sqrt(lambda_1) u_1 for G's dominant
// eigenpair. u_1 comes from PCA_SQUARINGS trace-normalised squarings of G
// (G^(2^s) -> u u^T; own fp64 GEMM tiles) and PCA_REFINE power steps on G
// itself; the sign follows the reference's rule on vt[0] = flat^T u / |.|
// (largest-magnitude component positive, first index on ties).
// ---------------------------------------------------------------------------
constexpr int PCA_SQUARINGS = 24;
constexpr int PCA_REFINE = 6;
constexpr int PT = 64;  // GEMM tile

__global__ void __launch_bounds__(256) k_pca_rowmean(const double* __restrict__ D2, int n,
                                                     double* rm) {
  // rm[i] = mean_j D2[i][j]; one warp per row, fixed order
  const int lane = threadIdx.x & 31, w = (blockIdx.x * 256 + threadIdx.x) >> 5;
  const int nw = (gridDim.x * 256) >> 5;
  for (int i = w; i < n; i += nw) {
    double sacc = 0.0;
    for (int j = lane; j < n; j += 32) sacc += D2[(size_t)i * n + j];
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (lane == 0) rm[i] = sacc / n;
  }
}
__global__ void __launch_bounds__(1024) k_pca_mean(const double* rm, int n, double* mu) {
  __shared__ double sh[1024];
  double sacc = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) sacc += rm[i];
  sh[threadIdx.x] = sacc;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    mu[0] = sh[0] / n;
    mu[1] = 1.0;  // scale of the first squaring
  }
}
__global__ void __launch_bounds__(256) k_pca_center(const double* __restrict__ D2, int n,
                                                    const double* rm, const double* mu,
                                                    double* G) {
  const size_t tot = (size_t)n * n;
  for (size_t e = (size_t)blockIdx.x * 256 + threadIdx.x; e < tot; e += (size_t)gridDim.x * 256) {
    const int i = (int)(e / n), j = (int)(e % n);
    // symmetric by construction: the two row means enter in a fixed order
    const double a = i <= j ? rm[i] : rm[j], b = i <= j ? rm[j] : rm[i];
    const double d = i <= j ? D2[e] : D2[(size_t)j * n + i];
    G[e] = -0.5 * (((d - a) - b) + mu[0]);
  }
}
// C = (B^T B) / t^2 for symmetric B (row-major n x n), t = *scale (the trace
// of B as the previous squaring left it unnormalised); 64 x 64 tiles, 4 x 4 per thread
__global__ void __launch_bounds__(256) k_pca_square(const double* __restrict__ B, int n,
                                                    const double* scale, double* C) {
  __shared__ double sa[16][PT + 1], sb[16][PT + 1];
  const int i0 = blockIdx.y * PT, j0 = blockIdx.x * PT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < n; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * PT; e += 256) {
      const int kk = e / PT, c = e % PT, k = k0 + kk;
      sa[kk][c] = (k < n && i0 + c < n) ? B[(size_t)k * n + i0 + c] : 0.0;
      sb[kk][c] = (k < n && j0 + c < n) ? B[(size_t)k * n + j0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = sa[kk][ty + 16 * x];
#pragma unroll
      for (int y = 0; y < 4; ++y) b[y] = sb[kk][tx + 16 * y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
  }
  const double t = *scale, inv = 1.0 / (t * t);
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int i = i0 + ty + 16 * x, j = j0 + tx + 16 * y;
      if (i < n && j < n) C[(size_t)i * n + j] = acc[x][y] * inv;
    }
}
__global__ void __launch_bounds__(1024) k_pca_trace(const double* C, int n, double* scale) {
  __shared__ double sh[1024];
  double sacc = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) sacc += C[(size_t)i * n + i];
  sh[threadIdx.x] = sacc;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) scale[0] = sh[0] > 0.0 ? sh[0] : 1.0;
}
// one CTA: u = normalised row argmax diag(C) of C ~ u u^T, then power steps on G
__global__ void __launch_bounds__(1024) k_pca_finish(const double* C, const double* G, int n,
                                                     double* u, double* w, double* lam) {
  __shared__ double sh[1024];
  __shared__ int si[1024];
  const int tid = threadIdx.x;
  double best = -1.0;
  int bi = n;
  for (int i = tid; i < n; i += 1024) {
    const double d = C[(size_t)i * n + i];
    if (d > best) {
      best = d;
      bi = i;
    }
  }
  sh[tid] = best;
  si[tid] = bi;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (tid < o && (sh[tid + o] > sh[tid] || (sh[tid + o] == sh[tid] && si[tid + o] < si[tid]))) {
      sh[tid] = sh[tid + o];
      si[tid] = si[tid + o];
    }
    __syncthreads();
  }
  const int js = si[0] < n ? si[0] : 0;
  __syncthreads();
  auto normalise = [&](const double* src, double* dst) -> double {  // returns |src|
    double q = 0.0;
    for (int i = tid; i < n; i += 1024) q += src[i] * src[i];
    sh[tid] = q;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
      if (tid < o) sh[tid] += sh[tid + o];
      __syncthreads();
    }
    const double nrm = sqrt(sh[0]);
    __syncthreads();
    for (int i = tid; i < n; i += 1024) dst[i] = nrm > 0.0 ? src[i] / nrm : src[i];
    __syncthreads();
    return nrm;
  };
  normalise(C + (size_t)js * n, u);
  double l = 0.0;
  for (int it = 0; it < PCA_REFINE; ++it) {
    // w = G u through G's columns (G symmetric): coalesced over i
    for (int i = tid; i < n; i += 1024) {
      double q = 0.0;
      for (int j = 0; j < n; ++j) q = fma(G[(size_t)j * n + i], u[j], q);
      w[i] = q;
    }
    __syncthreads();
    l = normalise(w, u);  // |G u| -> lambda_1 for a unit u
  }
  if (tid == 0) lam[0] = l;
}
// d_j = sum_i u_i flat[i][j] (= (centered^T u)_j: sum_i u_i = 0); per-CTA
// arg max |d_j| (first index on ties) -> part[3 b .. 3 b + 2] = |d|, j, d
__global__ void __launch_bounds__(256) k_pca_dir(const double* __restrict__ flat, int n, int64_t P,
                                                 const double* __restrict__ u, double* part) {
  __shared__ double sv[256], sd[256];
  __shared__ long long sj[256];
  double best = -1.0, bd = 0.0;
  long long bj = P;
  for (int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x; j < P; j += (int64_t)gridDim.x * 256) {
    double d = 0.0;
    for (int i = 0; i < n; ++i) d = fma(__ldg(u + i), flat[(size_t)i * P + j], d);
    if (fabs(d) > best) {
      best = fabs(d);
      bj = j;
      bd = d;
    }
  }
  sv[threadIdx.x] = best;
  sj[threadIdx.x] = bj;
  sd[threadIdx.x] = bd;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    const int t = threadIdx.x;
    if (t < o && (sv[t + o] > sv[t] || (sv[t + o] == sv[t] && sj[t + o] < sj[t]))) {
      sv[t] = sv[t + o];
      sj[t] = sj[t + o];
      sd[t] = sd[t + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = sv[0];
    part[3 * blockIdx.x + 1] = (double)sj[0];
    part[3 * blockIdx.x + 2] = sd[0];
  }
}
__global__ void __launch_bounds__(256) k_pca_keys(const double* part, int nb, const double* u,
                                                  const double* lam, int n, double* keys) {
  __shared__ double s_sign;
  if (threadIdx.x == 0) {
    double best = -1.0, bj = 0.0, bd = 1.0;
    for (int b = 0; b < nb; ++b)
      if (part[3 * b] > best || (part[3 * b] == best && part[3 * b + 1] < bj)) {
        best = part[3 * b];
        bj = part[3 * b + 1];
        bd = part[3 * b + 2];
      }
    s_sign = bd < 0.0 ? -1.0 : 1.0;
  }
  __syncthreads();
  const double sc = s_sign * sqrt(fmax(lam[0], 0.0));
  for (int i = threadIdx.x; i < n; i += 256) keys[i] = sc * u[i];
}

struct PcaLayout {
  size_t G, B0, B1, rm, mu, u, w, lam, part, total;
};
static PcaLayout pca_layout(int n) {
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  PcaLayout L;
  size_t off = 0;
  const size_t nn = (size_t)n * n * sizeof(double);
  L.G = off;
  off = al(off + nn);
  L.B0 = off;
  off = al(off + nn);
  L.B1 = off;
  off = al(off + nn);
  L.rm = off;
  off = al(off + (size_t)n * sizeof(double));
  L.mu = off;
  off = al(off + 4 * sizeof(double));
  L.u = off;
  off = al(off + (size_t)n * sizeof(double));
  L.w = off;
  off = al(off + (size_t)n * sizeof(double));
  L.lam = off;
  off = al(off + 2 * sizeof(double));
  L.part = off;
  off = al(off + 3 * 1184 * sizeof(double));
  L.total = off;
  return L;
}

}  // namespace skrsort

using namespace skrsort;

extern "C" {

size_t skr_sort_workspace_bytes(int32_t n_sys, int64_t P) {
  if (n_sys <= 0 || P <= 0) return 0;
  return sort_layout(n_sys, P).total;
}

int skr_sort_binary_check(const double* params, int32_t n_sys, int64_t P, double* v0v1,
                          int32_t* is_binary, void* ws, size_t ws_bytes, void* stream) {
  if (!params || n_sys <= 0 || P <= 0 || !v0v1 || !is_binary || !ws) return SKR_ERR_ARG;
  SortLayout L = sort_layout(n_sys, P);
  if (ws_bytes < L.bits) return SKR_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  char* base = (char*)ws;
  double* part = (double*)(base + L.part);
  double* mm = (double*)(base + L.mm);
  int* bad = (int*)(base + L.bad);
  int64_t total = (int64_t)n_sys * P;
  int nb = (int)std::min<int64_t>(1184, (total + 255) / 256);
  k_minmax<<<nb, 256, 0, s>>>(params, total, part);
  k_minmax_final<<<1, 32, 0, s>>>(part, nb, mm);
  cudaMemsetAsync(bad, 0, sizeof(int), s);
  k_two_valued<<<nb, 256, 0, s>>>(params, total, mm, bad);
  int hbad = 1;
  cudaMemcpyAsync(v0v1, mm, 2 * sizeof(double), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return SKR_ERR_CUDA;
  // exact only if (v1-v0)^2 is an integer and P (v1-v0)^2 < 2^53
  double dl = v0v1[1] - v0v1[0];
  double d2 = dl * dl;
  bool integral = d2 == std::floor(d2) && d2 * (double)P < 9007199254740992.0;
  *is_binary = (!hbad && integral) ? 1 : 0;
  return SKR_OK;
}

int skr_sort_dist2(const double* params, int32_t n_sys, int64_t P, int32_t row0, int32_t row1,
                   int32_t binary, double v0, double v1, double* D2, void* ws, size_t ws_bytes,
                   void* stream) {
  if (!params || !D2 || n_sys <= 0 || P <= 0 || row0 < 0 || row1 > n_sys || row0 >= row1)
    return SKR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (binary) {
    SortLayout L = sort_layout(n_sys, P);
    if (!ws || ws_bytes < L.d2) return SKR_ERR_WORKSPACE;
    unsigned long long* bits = (unsigned long long*)((char*)ws + L.bits);
    int64_t W = (P + 63) / 64;
    int64_t tot = (int64_t)n_sys * W;
    int nb = (int)std::min<int64_t>(1184 * 4, (tot + 255) / 256);
    k_pack<<<nb, 256, 0, s>>>(params, n_sys, P, W, v1, bits);
    double dl = v1 - v0;
    dim3 grid((n_sys + 31) / 32, (row1 - row0 + 31) / 32);
    k_hamming<<<grid, 256, 0, s>>>(bits, n_sys, W, row0, row1, dl * dl, D2);
  } else {
    int sym = (row0 == 0 && row1 == n_sys) ? 1 : 0;
    dim3 grid((n_sys + TS - 1) / TS, (row1 - row0 + TS - 1) / TS);
    k_dist2<<<grid, 256, 0, s>>>(params, n_sys, P, row0, row1, sym, D2);
  }
  return cudaGetLastError() == cudaSuccess ? SKR_OK : SKR_ERR_CUDA;
}

int skr_sort_chain(const double* D2, const double* params, int32_t n_sys, int64_t P,
                   int32_t exact_d2, int32_t* order, int32_t* n_certified, void* stream) {
  if (!D2 || !order || !n_certified || n_sys <= 0 || (!exact_d2 && !params)) return SKR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  size_t smem = (size_t)((n_sys + 31) / 32) * sizeof(unsigned int);
  if (smem > 200 * 1024) return SKR_ERR_UNSUPPORTED;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_chain<<<1, CHAIN_NT, smem, s>>>(D2, params, n_sys, P, exact_d2, order, n_certified);
  return cudaGetLastError() == cudaSuccess ? SKR_OK : SKR_ERR_CUDA;
}


size_t skr_sort_pca_workspace_bytes(int32_t n_sys) {
  if (n_sys <= 0) return 0;
  return pca_layout(n_sys).total;
}

int skr_sort_pca_keys(const double* D2, const double* params, int32_t n_sys, int64_t P,
                      double* keys, void* ws, size_t ws_bytes, void* stream) {
  if (!D2 || !params || !keys || !ws || n_sys < 2 || P <= 0) return SKR_ERR_ARG;
  const PcaLayout L = pca_layout(n_sys);
  if (ws_bytes < L.total) return SKR_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  char* base = (char*)ws;
  double* G = (double*)(base + L.G);
  double* Bb[2] = {(double*)(base + L.B0), (double*)(base + L.B1)};
  double* rm = (double*)(base + L.rm);
  double* mu = (double*)(base + L.mu);  // [0] mean of D2, [1] scale of the next squaring
  double* u = (double*)(base + L.u);
  double* w = (double*)(base + L.w);
  double* lam = (double*)(base + L.lam);
  double* part = (double*)(base + L.part);
  const int n = n_sys;
  const int g1 = std::min(1184, (n + 7) / 8);
  k_pca_rowmean<<<g1, 256, 0, s>>>(D2, n, rm);
  k_pca_mean<<<1, 1024, 0, s>>>(rm, n, mu);
  const int g2 = (int)std::min<size_t>(1184 * 4, ((size_t)n * n + 255) / 256);
  k_pca_center<<<g2, 256, 0, s>>>(D2, n, rm, mu, G);
  dim3 gg((n + PT - 1) / PT, (n + PT - 1) / PT);
  const double* src = G;
  for (int q = 0; q < PCA_SQUARINGS; ++q) {
    double* dst = Bb[q & 1];
    k_pca_square<<<gg, 256, 0, s>>>(src, n, mu + 1, dst);
    k_pca_trace<<<1, 1024, 0, s>>>(dst, n, mu + 1);
    src = dst;
  }
  k_pca_finish<<<1, 1024, 0, s>>>(src, G, n, u, w, lam);
  const int nb = (int)std::min<int64_t>(1184, (P + 255) / 256);
  k_pca_dir<<<nb, 256, 0, s>>>(params, n, P, u, part);
  k_pca_keys<<<1, 256, 0, s>>>(part, nb, u, lam, n, keys);
  return cudaGetLastError() == cudaSuccess ? SKR_OK : SKR_ERR_CUDA;
}

int skr_greedy_sort(const double* params, int32_t n_sys, int64_t P, int32_t* order_host, void* ws,
                    size_t ws_bytes, void* stream) {
  if (!params || n_sys <= 0 || P <= 0 || !order_host || !ws) return SKR_ERR_ARG;
  SortLayout L = sort_layout(n_sys, P);
  if (ws_bytes < L.total) return SKR_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  double v[2];
  int32_t bin = 0;
  int rc = skr_sort_binary_check(params, n_sys, P, v, &bin, ws, ws_bytes, stream);
  if (rc) return rc;
  double* D2 = (double*)((char*)ws + L.d2);
  rc = skr_sort_dist2(params, n_sys, P, 0, n_sys, bin, v[0], v[1], D2, ws, ws_bytes, stream);
  if (rc) return rc;
  int* d_order = (int*)((char*)ws + L.bad) + 1;  // reuse: need n_sys ints -> use bits region
  d_order = (int*)((char*)ws + L.bits);
  int* d_cert = (int*)((char*)ws + L.bad) + 2;
  rc = skr_sort_chain(D2, params, n_sys, P, bin, d_order, d_cert, stream);
  if (rc) return rc;
  cudaMemcpyAsync(order_host, d_order, sizeof(int) * n_sys, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return SKR_ERR_CUDA;
  return SKR_OK;
}

}  // extern "C"
