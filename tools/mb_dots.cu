// Microbenchmark for the k_cycle sweep-1 inner loop (tools/mb_dots.cu):
// partial dots Q^T [w z] of a column-major panel Q (N x P, ld = N) over each
// CTA's row slice, at C3 size (N = 2^21), persistent grid of 2 CTAs / SM.
//   v0: streaming ceiling (every element loaded once, summed per lane)
//   v1: the k_cycle scheme (64-row warp tiles, 8-column batches, butterfly)
//   v3: TMA (cp.async.bulk) ring, 2 stages x 32 KB, 2 CTAs / SM; v4: 6 stages, 1 CTA / SM
//   v2: DMMA m8n8k4 (rows = k; [w z] as the A operand, 8-column groups as B;
//       accumulators stay in registers for the whole sweep, no butterfly)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_dots tools/mb_dots.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 256, NW = 8;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(NT, 2) v0(const double* Q, int ld, int P, const double* w,
                                           const double* z, int rpb, int n, double* out) {
  const int r0 = blockIdx.x * rpb, r1 = min(n, r0 + rpb);
  double s = 0.0;
  for (int row = r0 + threadIdx.x; row < r1; row += NT) {
    double a = w[row] + z[row];
#pragma unroll 8
    for (int c = 0; c < P; ++c) a += Q[(size_t)c * ld + row];
    s += a;
  }
  if (s == 12345.0) out[blockIdx.x] = s;
}

template <int NV>
__device__ __forceinline__ double bfly(double (&v)[NV], int lane) {
  int off = 16;
#pragma unroll
  for (int h = NV / 2; h >= 1; h /= 2, off /= 2) {
    const bool hi = lane & off;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      double send = hi ? v[k] : v[k + h], keep = hi ? v[k + h] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  double r = v[0];
#pragma unroll
  for (; off >= 1; off /= 2) r += __shfl_xor_sync(0xffffffffu, r, off);
  return r;
}

__global__ void __launch_bounds__(NT, 2) v1(const double* Q, int ld, int P, const double* w,
                                           const double* z, int rpb, int n, double* out) {
  constexpr int R = 2, CB = 8, TR = 64;
  __shared__ double sacc[NW][2 * 64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = lane; c < 2 * 64; c += 32) sacc[warp][c] = 0.0;
  __syncwarp();
  const int r0 = blockIdx.x * rpb, r1 = min(n, r0 + rpb);
  const int ntile = (r1 - r0 + TR - 1) / TR;
  for (int tile = warp; tile < ntile; tile += NW) {
    const int base = r0 + tile * TR + lane;
    double wv[R], zv[R];
    bool ok[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      ok[i] = base + 32 * i < r1;
      wv[i] = ok[i] ? w[base + 32 * i] : 0.0;
      zv[i] = ok[i] ? z[base + 32 * i] : 0.0;
    }
    for (int c0 = 0; c0 < P; c0 += CB) {
      double qv[CB][R];
#pragma unroll
      for (int cc = 0; cc < CB; ++cc) {
        const double* Qc = Q + (size_t)min(c0 + cc, P - 1) * ld + base;
#pragma unroll
        for (int i = 0; i < R; ++i) qv[cc][i] = ok[i] ? Qc[32 * i] : 0.0;
      }
      double v[2 * CB];
#pragma unroll
      for (int cc = 0; cc < CB; ++cc) {
        double dw = 0.0, dz = 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          dw = fma(qv[cc][i], wv[i], dw);
          dz = fma(qv[cc][i], zv[i], dz);
        }
        v[cc] = dw;
        v[CB + cc] = dz;
      }
      const double tot = bfly<2 * CB>(v, lane);
      const int idx = (lane >> 1) & 15, col = c0 + (idx % CB);
      if (!(lane & 1) && col < P) sacc[warp][(idx / CB) * 64 + col] += tot;
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * P) {
    double s = 0.0;
    for (int q = 0; q < NW; ++q) s += sacc[q][(threadIdx.x / P) * 64 + threadIdx.x % P];
    out[(size_t)blockIdx.x * 128 + threadIdx.x] = s;
  }
}

// DMMA: per 16-row block rb of a warp's 64-row tile and 8-column group g,
// lane l (n = l / 4 column, kp = l % 4) loads Q rows rb + 4 kp .. + 3 of
// column 8 g + n (32 contiguous bytes); MMA q in 0..3 pairs k-position kp with
// row rb + 4 kp + q. A operand: lanes 0-3 hold w, lanes 4-7 z of those rows.
__global__ void __launch_bounds__(NT, 2) v2(const double* Q, int ld, int P, const double* w,
                                           const double* z, int rpb, int n, double* out) {
  constexpr int TR = 64, G = 8;  // up to 8 column groups of 8
  __shared__ double sres[NW][2][64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = blockIdx.x * rpb, r1 = min(n, r0 + rpb);
  const int ntile = (r1 - r0 + TR - 1) / TR;
  const int ng = (P + 7) / 8;
  const int kp = lane & 3, nn = lane >> 2;
  double acc[G][2];
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g][0] = acc[g][1] = 0.0;
  for (int tile = warp; tile < ntile; tile += NW) {
    const int tb = r0 + tile * TR;
    // A fragments of the tile: 4 blocks x 4 rows of w (lanes 0-3) / z (4-7)
    double af[4][4];
#pragma unroll
    for (int blk = 0; blk < 4; ++blk) {
      const int row = tb + 16 * blk + 4 * kp;
      const double* src = nn == 0 ? w : z;
      double2 p0 = make_double2(0.0, 0.0), p1 = p0;
      if (nn < 2 && row + 3 < r1) {
        p0 = *reinterpret_cast<const double2*>(src + row);
        p1 = *reinterpret_cast<const double2*>(src + row + 2);
      }
      af[blk][0] = p0.x; af[blk][1] = p0.y; af[blk][2] = p1.x; af[blk][3] = p1.y;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (g < ng) {
        const int col = min(8 * g + nn, P - 1);
        const double* Qc = Q + (size_t)col * ld;
        double qb[4][4];
#pragma unroll
        for (int blk = 0; blk < 4; ++blk) {
          const int row = tb + 16 * blk + 4 * kp;
          double2 p0 = make_double2(0.0, 0.0), p1 = p0;
          if (row + 3 < r1) {
            p0 = *reinterpret_cast<const double2*>(Qc + row);
            p1 = *reinterpret_cast<const double2*>(Qc + row + 2);
          }
          qb[blk][0] = p0.x; qb[blk][1] = p0.y; qb[blk][2] = p1.x; qb[blk][3] = p1.y;
        }
#pragma unroll
        for (int blk = 0; blk < 4; ++blk)
#pragma unroll
          for (int q = 0; q < 4; ++q) dmma(acc[g][0], acc[g][1], af[blk][q], qb[blk][q]);
      }
    }
  }
  // D[m][c]: lane l holds m = l / 4, c = 2 (l % 4) + {0, 1}
#pragma unroll
  for (int g = 0; g < G; ++g)
    if (g < ng && nn < 2) {
      sres[warp][nn][8 * g + 2 * kp] = acc[g][0];
      sres[warp][nn][8 * g + 2 * kp + 1] = acc[g][1];
    }
  __syncthreads();
  if (threadIdx.x < 2 * P) {
    const int m = threadIdx.x / P, c = threadIdx.x % P;
    double s = 0.0;
    for (int q = 0; q < NW; ++q) s += sres[q][m][c];
    out[(size_t)blockIdx.x * 128 + threadIdx.x] = s;
  }
}


// v3: CTA-level TMA ring. One producer thread issues 1-D bulk copies
// (cp.async.bulk, 4 KB = 512 rows of one column) into a ring of STAGES stages
// of [CBS columns x 512 rows]; the 8 consumer warps each take 64 rows of a
// stage (same butterfly as v1) and release it through an mbarrier.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}" ::"r"(smem_u32(b)),
      "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

template <int STAGES, int CBS>
__global__ void __launch_bounds__(NT + 32, 2) v3(const double* Q, int ld, int P, const double* w,
                                                const double* z, int rpb, int n, double* out) {
  constexpr int TRC = 512;  // rows per stage (8 warps x 64)
  extern __shared__ __align__(128) double dsm[];
  double* ring = dsm;                                  // STAGES x CBS x TRC
  double* wz = dsm + (size_t)STAGES * CBS * TRC;       // 2 x 2 x TRC (w, z; double-buffered)
  __shared__ double sacc[NW][2 * 64];
  __shared__ unsigned long long full[STAGES], empty[STAGES], wzfull[2], wzempty[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = blockIdx.x * rpb, r1 = min(n, r0 + rpb);
  const int nrb = (r1 - r0 + TRC - 1) / TRC;           // row blocks (rpb is a multiple of 64;
  const int ncb = (P + CBS - 1) / CBS;                 //  the last block may be short)
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&wzfull[s], 1);
      mbar_init(&wzempty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp < NW)
    for (int c = lane; c < 2 * 64; c += 32) sacc[warp][c] = 0.0;
  __syncthreads();
  if (warp == NW) {  // producer warp: one thread
    if (lane == 0) {
      int it = 0;
      for (int rb = 0; rb < nrb; ++rb) {
        const int row0 = r0 + rb * TRC;
        const int rows = min(TRC, r1 - row0);
        const unsigned cb = rows * 8;
        {
          const int s = rb & 1, ph = (rb >> 1) & 1;
          if (rb >= 2) mbar_wait(&wzempty[s], ph ^ 1);
          mbar_expect_tx(&wzfull[s], 2 * cb);
          bulk_g2s(wz + (size_t)s * 2 * TRC, w + row0, cb, &wzfull[s]);
          bulk_g2s(wz + (size_t)s * 2 * TRC + TRC, z + row0, cb, &wzfull[s]);
        }
        for (int b = 0; b < ncb; ++b, ++it) {
          const int s = it % STAGES, ph = (it / STAGES) & 1;
          if (it >= STAGES) mbar_wait(&empty[s], ph ^ 1);
          const int nc = min(CBS, P - b * CBS);
          mbar_expect_tx(&full[s], nc * cb);
          for (int c = 0; c < nc; ++c)
            bulk_g2s(ring + ((size_t)s * CBS + c) * TRC, Q + (size_t)(b * CBS + c) * ld + row0, cb,
                     &full[s]);
        }
      }
    }
    return;
  }
  int it = 0;
  for (int rb = 0; rb < nrb; ++rb) {
    const int row0 = r0 + rb * TRC;
    const int rows = min(TRC, r1 - row0);
    const int lr = 64 * warp + lane;  // this lane's rows lr, lr + 32 of the stage
    const bool ok0 = lr < rows, ok1 = lr + 32 < rows;
    const int ws = rb & 1;
    mbar_wait(&wzfull[ws], (rb >> 1) & 1);
    const double* wzb = wz + (size_t)ws * 2 * TRC;
    const double w0 = ok0 ? wzb[lr] : 0.0, w1 = ok1 ? wzb[lr + 32] : 0.0;
    const double z0 = ok0 ? wzb[TRC + lr] : 0.0, z1 = ok1 ? wzb[TRC + lr + 32] : 0.0;
    __syncwarp();
    if (lane == 0) mbar_arrive(&wzempty[ws]);
    for (int b = 0; b < ncb; ++b, ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      const double* st = ring + (size_t)s * CBS * TRC;
      const int nc = min(CBS, P - b * CBS);
      double v[2 * CBS];
#pragma unroll
      for (int cc = 0; cc < CBS; ++cc) {
        const double* qc = st + (size_t)min(cc, nc - 1) * TRC;
        const double q0 = ok0 ? qc[lr] : 0.0, q1 = ok1 ? qc[lr + 32] : 0.0;
        v[cc] = fma(q1, w1, q0 * w0);
        v[CBS + cc] = fma(q1, z1, q0 * z0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      const double tot = bfly<2 * CBS>(v, lane);
      constexpr int L2 = CBS == 8 ? 4 : CBS == 4 ? 3 : 5;
      constexpr int SH = 5 - L2;
      const int idx = (lane >> SH) & (2 * CBS - 1), col = b * CBS + (idx % CBS);
      if (!(lane & ((1 << SH) - 1)) && (idx % CBS) < nc) sacc[warp][(idx / CBS) * 64 + col] += tot;
    }
  }
  // consumers only (the producer warp has left): named barrier over 256 threads
  asm volatile("bar.sync 1, 256;" ::: "memory");
  if (threadIdx.x < 2 * P) {
    const int m = threadIdx.x / P, c = threadIdx.x % P;
    double s = 0.0;
    for (int q = 0; q < NW; ++q) s += sacc[q][m * 64 + c];
    out[(size_t)blockIdx.x * 128 + threadIdx.x] = s;
  }
}

int main() {
  const int n = 1 << 21;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nblk = 2 * sms;
  const int rpb = ((n + nblk - 1) / nblk + 63) / 64 * 64;
  double *Q, *w, *z, *out;
  const int PM = 64;
  cudaMalloc(&Q, (size_t)n * PM * 8);
  cudaMalloc(&w, n * 8);
  cudaMalloc(&z, n * 8);
  cudaMalloc(&out, (size_t)nblk * 128 * 8);
  // deterministic fill
  double* h = new double[n];
  for (int i = 0; i < n; ++i) h[i] = ((i * 7919) % 1000) * 1e-3 - 0.5;
  for (int c = 0; c < PM; ++c) cudaMemcpy(Q + (size_t)c * n, h, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(w, h, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(z, h, n * 8, cudaMemcpyHostToDevice);
  double* flush;
  cudaMalloc(&flush, 512 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double* o1 = new double[nblk * 128];
  double* o2 = new double[nblk * 128];
  double* o3 = new double[nblk * 128];
  const int smem3 = (2 * 8 * 512 + 4 * 512) * 8, smem4 = (6 * 8 * 512 + 4 * 512) * 8;
  cudaFuncSetAttribute(v3<2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
  cudaFuncSetAttribute(v3<6, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4);
  for (int P : {20, 32, 40, 60}) {
    for (int v = 0; v < 5; ++v) {
      float best = 1e9f;
      for (int rep = 0; rep < 8; ++rep) {
        cudaMemset(flush, rep, 512 << 20);
        cudaEventRecord(e0);
        if (v == 0) v0<<<nblk, NT>>>(Q, n, P, w, z, rpb, n, out);
        if (v == 1) v1<<<nblk, NT>>>(Q, n, P, w, z, rpb, n, out);
        if (v == 2) v2<<<nblk, NT>>>(Q, n, P, w, z, rpb, n, out);
        if (v == 3) v3<2, 8><<<nblk, NT + 32, smem3>>>(Q, n, P, w, z, rpb, n, out);
        if (v == 4) v3<6, 8><<<sms, NT + 32, smem4>>>(Q, n, P, w, z, 2 * rpb, n, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      if (v == 1) cudaMemcpy(o1, out, (size_t)nblk * 128 * 8, cudaMemcpyDeviceToHost);
      if (v == 2) cudaMemcpy(o2, out, (size_t)nblk * 128 * 8, cudaMemcpyDeviceToHost);
      if (v == 3) cudaMemcpy(o3, out, (size_t)nblk * 128 * 8, cudaMemcpyDeviceToHost);
      double gb = (double)(P + 2) * n * 8 / (best * 1e-3) / 1e9;
      printf("P=%d v%d: %.3f ms  %.0f GB/s  %s\n", P, v, best, gb, cudaGetErrorString(cudaGetLastError()));
    }
    double md = 0.0;
    for (int b = 0; b < nblk; ++b)
      for (int i = 0; i < 2 * P; ++i) {
        double d = o1[b * 128 + i] - o2[b * 128 + i];
        md = fmax(md, fabs(d) / (1e-30 + fabs(o1[b * 128 + i])));
      }
    printf("P=%d max rel diff v1 vs v2 %.2e\n", P, md);
    md = 0.0;
    for (int b = 0; b < nblk; ++b)
      for (int i = 0; i < 2 * P; ++i) {
        double d = o1[b * 128 + i] - o3[b * 128 + i];
        md = fmax(md, fabs(d) / (1e-30 + fabs(o1[b * 128 + i])));
      }
    printf("P=%d max rel diff v1 vs v3 (TMA ring) %.2e\n", P, md);
  }
  // leading-dimension padding: column stride 2^21 doubles (16 MiB) vs padded
  {
    double* Qp;
    const int P = 40;
    cudaMalloc(&Qp, ((size_t)n + 4096) * PM * 8);
    for (int pad : {0, 64, 192, 448, 1088, 2112}) {
      const int ldp = n + pad;
      for (int c = 0; c < PM; ++c) cudaMemcpy(Qp + (size_t)c * ldp, h, n * 8, cudaMemcpyHostToDevice);
      for (int v : {1, 3}) {
        float best = 1e9f;
        for (int rep = 0; rep < 8; ++rep) {
          cudaMemset(flush, rep, 512 << 20);
          cudaEventRecord(e0);
          if (v == 1) v1<<<nblk, NT>>>(Qp, ldp, P, w, z, rpb, n, out);
          if (v == 3) v3<2, 8><<<nblk, NT + 32, smem3>>>(Qp, ldp, P, w, z, rpb, n, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          best = ms < best ? ms : best;
        }
        printf("ld pad %4d doubles, P=40 v%d: %.3f ms  %.0f GB/s\n", pad, v, best,
               (double)(P + 2) * n * 8 / (best * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
