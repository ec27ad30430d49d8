// FP64 tensor-core (DMMA m8n8k4) vs DFMA throughput microbenchmark on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w : {4, 8, 16}) {
    int blocks = sms * 4, threads = 32 * w, iters = 4096;
    k_dmma<<<blocks, threads>>>(d, 16); cudaDeviceSynchronize();
    cudaEventRecord(a); k_dmma<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 8 * 8 * 4 * 8.0 * iters * blocks * (threads / 32);
    printf("DMMA warps/blk=%d: %.2f TFLOP/s (%s)\n", w, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(a); k_dfma<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    fl = 2.0 * 8 * (double)iters * blocks * threads;
    printf("DFMA warps/blk=%d: %.2f TFLOP/s\n", w, fl / ms / 1e9);
  }
  return 0;
}
