// Device assembly of the finite-difference systems of the benchmark configs
// (replaces the host loops of problems.py's assemble, the reference's
// problems.py:335-355 / :380-383): from the coefficient
// field (8 bytes per cell uploaded instead of the CSR's ~60), one thread per
// cell writes the stencil form (D, W, S, B; verified flag set) and the CSR
// values in the fixed natural-ordering pattern. Every value is computed with
// the host assembly's operation order and IEEE round-to-nearest (no FMA
// contraction), so the device matrix is bit-identical to the host one.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/skr.h"
#include "skr_device.cuh"

namespace skr {

// harmonic mean of the face between cells q (lower index) and p = q + stride,
// as problems.py _faces_flux: (2 a_p) a_q / (a_p + a_q)
__device__ __forceinline__ double face_hm(double ap, double aq) {
  return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, ap), aq), __dadd_rn(ap, aq));
}

// kind 0: -div(a grad u) h^2-scaled, negative diagonal (darcy / poisson):
//   off-diagonal = face coefficient, wall faces use the cell value,
//   diag = ((0 - lo_x) - hi_x) - lo_y - hi_y [- lo_z - hi_z]
// kind 1: Helmholtz, off-diagonal 1, diag = -2 dim + (k h)^2
__global__ void __launch_bounds__(NT) k_assemble_fd(int kind, int dim, int n, const double* f,
                                                    double h, const int32_t* rp, double* vals,
                                                    StenView sv) {
  const int N = dim == 3 ? n * n * n : n * n;
  const int sx = n, sxy = dim == 3 ? n * n : 0;
  double* D = const_cast<double*>(sv.D);
  double* W = const_cast<double*>(sv.W);
  double* S = const_cast<double*>(sv.S);
  double* B = const_cast<double*>(sv.B);
  for (int i = blockIdx.x * NT + threadIdx.x; i < N; i += gridDim.x * NT) {
    const int ix = i % n, iy = (i / n) % n, iz = dim == 3 ? i / (n * n) : 0;
    double lo[3], hi[3], d;
    const int st[3] = {1, sx, sxy};
    const int co[3] = {ix, iy, iz};
    if (kind == 0) {
      const double ai = __ldg(f + i);
      d = 0.0;
      for (int ax = 0; ax < dim; ++ax) {
        lo[ax] = co[ax] > 0 ? face_hm(ai, __ldg(f + i - st[ax])) : ai;
        hi[ax] = co[ax] < n - 1 ? face_hm(__ldg(f + i + st[ax]), ai) : ai;
        d = __dsub_rn(d, lo[ax]);
        d = __dsub_rn(d, hi[ax]);
      }
    } else {
      const double kh = __dmul_rn(__ldg(f + i), h);
      d = __dadd_rn(-2.0 * dim, __dmul_rn(kh, kh));
      for (int ax = 0; ax < dim; ++ax) lo[ax] = hi[ax] = 1.0;
    }
    // stencil form: lower entries (0 = absent) and the diagonal
    D[i] = d;
    W[i] = ix > 0 ? lo[0] : 0.0;
    S[i] = iy > 0 ? lo[1] : 0.0;
    if (dim == 3) B[i] = iz > 0 ? lo[2] : 0.0;
    // CSR values in column order: -sxy, -sx, -1, 0, +1, +sx, +sxy
    if (vals) {
      int q = __ldg(rp + i);
      if (dim == 3 && iz > 0) vals[q++] = lo[2];
      if (iy > 0) vals[q++] = lo[1];
      if (ix > 0) vals[q++] = lo[0];
      vals[q++] = d;
      if (ix < n - 1) vals[q++] = hi[0];
      if (iy < n - 1) vals[q++] = hi[1];
      if (dim == 3 && iz < n - 1) vals[q++] = hi[2];
    }
  }
}

__global__ void k_assemble_pad(StenView sv, int n, int sx, int sxy) {
  // zero padding past N (upper neighbours of the last rows) + verified flag
  double* W = const_cast<double*>(sv.W);
  double* S = const_cast<double*>(sv.S);
  double* B = const_cast<double*>(sv.B);
  for (int t = threadIdx.x; t < sx; t += blockDim.x) S[n + t] = 0.0;
  for (int t = threadIdx.x; t < sxy; t += blockDim.x) B[n + t] = 0.0;
  if (threadIdx.x == 0) {
    W[n] = 0.0;
    int* hdr = const_cast<int*>(sv.hdr);
    hdr[1] = 0;
    hdr[0] = 1;
  }
}

}  // namespace skr

using namespace skr;

extern "C" int skr_assemble_fd(int32_t kind, int32_t dim, int32_t n, const double* field,
                               double h, const int32_t* row_ptr, double* values, void* stencil,
                               size_t stencil_bytes, void* stream) {
  if ((kind != 0 && kind != 1) || (dim != 2 && dim != 3) || n < 2 || !field || !stencil)
    return SKR_ERR_ARG;
  if (values && !row_ptr) return SKR_ERR_ARG;
  const long long NN = dim == 3 ? (long long)n * n * n : (long long)n * n;
  if (NN >= (1ll << 31) - 1) return SKR_ERR_UNSUPPORTED;
  const int N = (int)NN, sx = n, sxy = dim == 3 ? n * n : 0;
  if (stencil_bytes < sten_doubles(N, sx, sxy) * sizeof(double)) return SKR_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  StenView v = sten_view(stencil, N, sx, sxy);
  int grid = (N + NT - 1) / NT;
  if (grid > 148 * 8) grid = 148 * 8;
  k_assemble_pad<<<1, 256, 0, s>>>(v, N, sx, sxy);
  k_assemble_fd<<<grid, NT, 0, s>>>(kind, dim, n, field, h, row_ptr, values, v);
  return cudaGetLastError() == cudaSuccess ? SKR_OK : SKR_ERR_CUDA;
}
