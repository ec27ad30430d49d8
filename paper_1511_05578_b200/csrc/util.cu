// FP64 roofline denominator: a register-resident DFMA loop on every SM.
#include "scv_internal.cuh"

__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the loop alive
}

extern "C" int scv_fp64_peak(scv_ctx* c, double* tflops) {
  if (!c || !tflops) return SCV_EINVAL;
  SCV_CUDA(c, cudaSetDevice(c->device));
  int sms = 0;
  SCV_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  double* d = nullptr;
  SCV_CUDA(c, cudaMalloc(&d, 8));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_dfma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);  // warm-up
  double best = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    k_dfma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 8.0 * (double)iters * blocks * threads;
    double tf = fl / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  SCV_CUDA(c, cudaGetLastError());
  *tflops = best;
  return SCV_OK;
}

// FP64 tensor-core (DMMA m8n8k4) roofline denominator: 8 independent
// accumulator chains per warp, 16 warps per SM (profiles/r01_fp64_pipe_microbench.log:
// that shape reaches the pipe's plateau).  512 flops per DMMA per warp.
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;  // keep the loop alive
}

extern "C" int scv_dmma_peak(scv_ctx* c, double* tflops) {
  if (!c || !tflops) return SCV_EINVAL;
  SCV_CUDA(c, cudaSetDevice(c->device));
  int sms = 0;
  SCV_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  double* d = nullptr;
  SCV_CUDA(c, cudaMalloc(&d, 8));
  const int blocks = sms * 2, threads = 256, iters = 1 << 12;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_dmma_peak<<<blocks, threads>>>(d, iters, 1e-3, 1e-3);  // warm-up
  double best = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    k_dmma_peak<<<blocks, threads>>>(d, iters, 1e-3, 1e-3);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double fl = 512.0 * 8.0 * (double)iters * blocks * (threads / 32);
    const double tf = fl / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  SCV_CUDA(c, cudaGetLastError());
  *tflops = best;
  return SCV_OK;
}
