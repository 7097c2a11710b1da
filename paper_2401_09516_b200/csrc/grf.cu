// Device sampling of the benchmark configs' coefficient fields (SURVEY 8(f)
// row 1: the config generators; replaces the host sampler problems.grf /
// system_params, which stand in for the reference's KL/SE samplers
// kryrec/problems.py:97-162 and the batch seeding of :488).
//
// The device generator is its own seeded definition ("philox" inputs,
// DESIGN.md §5): white noise from a counter-based Philox4x32-10 stream
// (Salmon et al., SC'11) mapped to N(0,1) by Box-Muller, one Philox block per
// pair of cells, so every cell's noise is a pure function of (seed, config,
// system, cell) and the sampling is embarrassingly parallel. The field is
//   g = DCT-III_ortho^{(dim)}( xi * coef ) / norm,
//   coef = 1 / (pi^2 |kappa|^2 + tau^2), coef_0 = 0,
// with the n x n DCT-III matrix applied along every axis as a batched fp64
// GEMM (2 dim n N flops per field: C3 1.6 GFLOP), the spectral multiply fused
// into the noise kernel and the pointwise coefficient law (threshold {3, 12},
// exp(s g), k0 (1 + 0.3 tanh g)) into the last pass's epilogue. The CPU
// restatement that checks it is oracle/grf_oracle.py.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/skr.h"

namespace skrgrf {

// ---- Philox4x32-10 -------------------------------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// 53-bit uniforms from two 32-bit words: [0, 1) and (0, 1]
__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double u53_open0(uint32_t a, uint32_t b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6) + 1.0) *
         (1.0 / 9007199254740992.0);
}

// the two normals of Philox block `pair` of (system, stream)
__device__ __forceinline__ void normal_pair(uint64_t pair, uint32_t sys, uint32_t stream,
                                            uint32_t k0, uint32_t k1, double& z0, double& z1) {
  const U4 r = philox4x32_10(U4{(uint32_t)pair, (uint32_t)(pair >> 32), sys, stream}, k0, k1);
  const double u1 = u53_open0(r.x, r.y), u2 = u53(r.z, r.w);
  const double rad = sqrt(-2.0 * log(u1));
  const double ang = 6.283185307179586 * u2;  // the same product as numpy's 2 * pi * u2
  double s, c;
  sincos(ang, &s, &c);
  z0 = rad * c;
  z1 = rad * s;
}

// xi_i * coef_i for every cell (C order, x fastest); count = n^dim
__global__ void k_noise_spectral(int dim, int n, long long count, double tau2, uint32_t sys,
                                 uint32_t k0, uint32_t k1, double* out) {
  const double pi = 3.141592653589793;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; 2 * p < count;
       p += (long long)gridDim.x * blockDim.x) {
    double z[2];
    normal_pair((uint64_t)p, sys, 0u, k0, k1, z[0], z[1]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long i = 2 * p + h;
      if (i >= count) break;
      // lam = sum over axes (slowest first, as problems._spectrum) of (pi k)^2
      long long rest = i;
      int kk[3];
      for (int ax = dim - 1; ax >= 0; --ax) {
        kk[ax] = (int)(rest % n);
        rest /= n;
      }
      double lam = 0.0;
      for (int ax = 0; ax < dim; ++ax) {
        const double pk = __dmul_rn(pi, (double)kk[ax]);
        lam = __dadd_rn(lam, __dmul_rn(pk, pk));
      }
      const double coef = i == 0 ? 0.0 : __ddiv_rn(1.0, __dadd_rn(lam, tau2));
      out[i] = __dmul_rn(z[h], coef);
    }
  }
}

// plain normals / uniforms of one (system, stream): the rhs noise of C1 and
// the per-system scalars of C2 (k0, bump centre)
__global__ void k_normals(long long count, uint32_t sys, uint32_t stream, uint32_t k0,
                          uint32_t k1, double scale, double* out) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; 2 * p < count;
       p += (long long)gridDim.x * blockDim.x) {
    double z0, z1;
    normal_pair((uint64_t)p, sys, stream, k0, k1, z0, z1);
    out[2 * p] = scale * z0;
    if (2 * p + 1 < count) out[2 * p + 1] = scale * z1;
  }
}

__global__ void k_uniforms(int count, uint32_t sys, uint32_t stream, uint32_t k0, uint32_t k1,
                           double* out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * p >= count) return;
  const U4 r = philox4x32_10(U4{(uint32_t)p, 0u, sys, stream}, k0, k1);
  out[2 * p] = u53(r.x, r.y);
  if (2 * p + 1 < count) out[2 * p + 1] = u53(r.z, r.w);
}

// ---- batched row-major fp64 GEMM  C[b] = A[b] (M x K) * B[b] (K x N) -------
// 64 x 64 output tiles, K in chunks of 16 staged in shared memory, 256
// threads with 4 x 4 register tiles. Epilogue 0 stores C; epilogue 1 is the
// field's last pass: g = acc / norm, then the coefficient law.
constexpr int TM = 64, TN = 64, TK = 16, GT = 256;

struct Epi {
  int mode;  // 0 store, 1 field
  int kind;  // 0 binary {3, 12}, 1 exp(param g), 2 param (1 + 0.3 tanh g)
  double norm, param;
  double* field;  // same indexing as C
  double* g;      // optional raw g (same indexing), may alias C
};

__global__ void __launch_bounds__(GT) k_gemm(int M, int N, int K, const double* __restrict__ A,
                                             long long lda, long long sA,
                                             const double* __restrict__ B, long long ldb,
                                             long long sB, double* C, long long ldc, long long sC,
                                             Epi epi) {
  __shared__ double As[TK][TM + 1];
  __shared__ double Bs[TK][TN];
  const int b = blockIdx.z;
  A += b * sA;
  B += b * sB;
  const long long coff = b * sC;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int e = threadIdx.x; e < TM * TK; e += GT) {  // A tile, k fastest (rows contiguous)
      const int kk = e % TK, mm = e / TK;
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[gm * lda + gk] : 0.0;
    }
    for (int e = threadIdx.x; e < TK * TN; e += GT) {  // B tile, n fastest
      const int nn = e % TN, kk = e / TN;
      const int gk = k0 + kk, gn = n0 + nn;
      Bs[kk][nn] = (gk < K && gn < N) ? B[gk * ldb + gn] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn >= N) continue;
      const long long o = coff + gm * ldc + gn;
      if (epi.mode == 0) {
        C[o] = acc[i][j];
      } else {
        const double g = acc[i][j] / epi.norm;
        double f;
        if (epi.kind == 0) f = g > 0.0 ? 12.0 : 3.0;
        else if (epi.kind == 1) f = exp(epi.param * g);
        else f = epi.param * (1.0 + 0.3 * tanh(g));
        epi.field[o] = f;
        if (epi.g) epi.g[o] = g;
      }
    }
  }
}

inline int blocks_for(long long work, int per) {
  long long b = (work + per - 1) / per;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace skrgrf

using namespace skrgrf;

extern "C" size_t skr_grf_workspace_bytes(int32_t dim, int32_t n) {
  if ((dim != 2 && dim != 3) || n < 2) return 0;
  const size_t N = dim == 3 ? (size_t)n * n * n : (size_t)n * n;
  return 2 * N * sizeof(double);
}

extern "C" int skr_grf_sample(int32_t dim, int32_t n, int32_t kind, double tau, double param,
                              double norm, const double* dct, uint64_t seed, uint32_t cid,
                              uint32_t idx, double* field, double* g_out, void* work,
                              size_t work_bytes, void* stream) {
  if ((dim != 2 && dim != 3) || n < 2 || kind < 0 || kind > 2 || !(norm > 0.0) || !dct || !field || !work)
    return SKR_ERR_ARG;
  if (work_bytes < skr_grf_workspace_bytes(dim, n)) return SKR_ERR_WORKSPACE;
  const long long N = dim == 3 ? (long long)n * n * n : (long long)n * n;
  if (N >= (1ll << 31)) return SKR_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  double* w0 = (double*)work;
  double* w1 = w0 + N;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32) ^ cid;
  k_noise_spectral<<<blocks_for(N / 2 + 1, 256), 256, 0, s>>>(dim, n, N, tau * tau, idx, k0, k1,
                                                            w0);
  const long long nn = n;
  const long long inner2 = dim == 3 ? nn * nn : nn;  // the slowest axis' row length
  Epi plain{0, 0, 0.0, 0.0, nullptr, nullptr};
  Epi last{1, kind, norm, param, field, g_out};
  // x (fastest) axis: rows of length n times DCT^T -- dct is passed as
  // [T | T^T] (2 n^2 doubles), T^T at dct + n^2
  {
    const long long rows = N / n;
    dim3 grid((n + TN - 1) / TN, (unsigned)((rows + TM - 1) / TM), 1);
    k_gemm<<<grid, GT, 0, s>>>((int)rows, n, n, w0, nn, 0, dct + nn * nn, nn, 0, w1, nn, 0,
                               plain);
  }
  if (dim == 3) {  // y axis: per z slab, T (n x n) times the slab (n x n)
    dim3 grid((n + TN - 1) / TN, (n + TM - 1) / TM, n);
    k_gemm<<<grid, GT, 0, s>>>(n, n, n, dct, nn, 0, w1, nn, nn * nn, w0, nn, nn * nn, plain);
  }
  // slowest axis: T (n x n) times the (n x inner2) array, field epilogue
  {
    const double* src = dim == 3 ? w0 : w1;
    dim3 grid((unsigned)((inner2 + TN - 1) / TN), (n + TM - 1) / TM, 1);
    k_gemm<<<grid, GT, 0, s>>>(n, (int)inner2, n, dct, nn, 0, src, inner2, 0, field, inner2, 0,
                               last);
  }
  return cudaGetLastError() == cudaSuccess ? SKR_OK : SKR_ERR_CUDA;
}

extern "C" int skr_philox_normals(int64_t count, uint64_t seed, uint32_t cid, uint32_t idx,
                                  uint32_t stream_id, double scale, double* out, void* stream) {
  if (count < 0 || (count > 0 && !out)) return SKR_ERR_ARG;
  if (count == 0) return SKR_OK;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32) ^ cid;
  k_normals<<<blocks_for(count / 2 + 1, 256), 256, 0, (cudaStream_t)stream>>>(
      count, idx, stream_id, k0, k1, scale, out);
  return cudaGetLastError() == cudaSuccess ? SKR_OK : SKR_ERR_CUDA;
}

extern "C" int skr_philox_uniforms(int32_t count, uint64_t seed, uint32_t cid, uint32_t idx,
                                   uint32_t stream_id, double* out, void* stream) {
  if (count < 0 || (count > 0 && !out)) return SKR_ERR_ARG;
  if (count == 0) return SKR_OK;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32) ^ cid;
  k_uniforms<<<(count / 2 + 256) / 256, 256, 0, (cudaStream_t)stream>>>(count, idx, stream_id,
                                                                        k0, k1, out);
  return cudaGetLastError() == cudaSuccess ? SKR_OK : SKR_ERR_CUDA;
}
