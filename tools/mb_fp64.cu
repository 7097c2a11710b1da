// FP64 throughput probe: DMMA m8n8k4 (mma.sync f64) vs DFMA, 8 independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kdmma(double* out, int iters) {
  double c[8][2];
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void kdfma(double* out, int iters) {
  double c[8];
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 16, 32}) {
    int it = 4096;
    float ms;
    kdmma<<<sms, 32 * warps>>>(o, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); kdmma<<<sms, 32 * warps>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = (double)sms * warps * it * 8 * 512;
    printf("DMMA warps/SM %d: %.1f TFLOP/s\n", warps, fl / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); kdfma<<<sms, 32 * warps>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = (double)sms * warps * 32 * it * 8 * 2;
    printf("DFMA warps/SM %d: %.1f TFLOP/s\n", warps, fl / (ms * 1e-3) / 1e12);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
