// FP64 pipe microbenchmarks on sm_100a: DMMA m8n8k4 throughput vs independent
// chains per warp and warps per SM, DMMA latency, DFMA throughput, and whether
// DMMA and DFMA issued from the same warps overlap (separate pipes) or share
// one FP64 unit.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NC>
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  double c[NC][2];
#pragma unroll
  for (int i = 0; i < NC; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

template <int NC>
__global__ void k_dfma(double* out, int iters) {
  double x[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < NC; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
  double s = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

// mixed: per iteration ND DMMAs and NF DFMAs (independent chains)
template <int ND, int NF>
__global__ void k_mix(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  double c[ND + 1][2], x[NF + 1];
#pragma unroll
  for (int i = 0; i < ND; ++i) { c[i][0] = i; c[i][1] = -i; }
#pragma unroll
  for (int i = 0; i < NF; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ND; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NF; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ND; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

// DADD throughput (adds are the bulk of FFT butterflies)
template <int NC>
__global__ void k_dadd(double* out, int iters) {
  double x[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) x[i] = threadIdx.x + i;
  const double y = 1e-9 * threadIdx.x;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < NC; ++i) x[i] = x[i] + y;
  double s = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

static double g_ms;
template <class F>
static double timeit(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  g_ms = ms;
  return ms;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  const int iters = 2048;
  // DMMA: flops per mma = 2*8*8*4 = 512
#define DM(NC, W, BPS)                                                                            \
  {                                                                                               \
    int blocks = sms * BPS, threads = 32 * W;                                                     \
    double ms = timeit([&] { k_dmma<NC><<<blocks, threads>>>(d, iters); });                       \
    double n = (double)NC * iters * blocks * W;                                                   \
    printf("DMMA chains=%2d warps/SM=%3d : %7.2f TFLOP/s  %.3f mma/clk/SM\n", NC, W * BPS,        \
           n * 512 / ms / 1e9, n / (ms * 1e-3 * clk * 1e3) / sms);                                \
  }
  DM(1, 1, 1) DM(2, 1, 1) DM(4, 1, 1) DM(8, 1, 1) DM(16, 1, 1)
  DM(1, 4, 1) DM(2, 4, 1) DM(4, 4, 1) DM(8, 4, 1) DM(12, 4, 1)
  DM(1, 8, 1) DM(2, 8, 1) DM(4, 8, 1) DM(8, 8, 1)
  DM(1, 16, 1) DM(2, 16, 1) DM(4, 16, 1) DM(8, 16, 1)
  DM(4, 8, 4) DM(8, 8, 4)
#define DF(NC, W, BPS)                                                                      \
  {                                                                                         \
    int blocks = sms * BPS, threads = 32 * W;                                               \
    double ms = timeit([&] { k_dfma<NC><<<blocks, threads>>>(d, iters); });                 \
    double n = (double)NC * iters * blocks * threads;                                       \
    printf("DFMA chains=%2d warps/SM=%3d : %7.2f TFLOP/s\n", NC, W * BPS, n * 2 / ms / 1e9); \
  }
  DF(8, 8, 1) DF(8, 16, 1) DF(8, 8, 4)
#define DA(NC, W, BPS)                                                                       \
  {                                                                                          \
    int blocks = sms * BPS, threads = 32 * W;                                                \
    double ms = timeit([&] { k_dadd<NC><<<blocks, threads>>>(d, iters); });                  \
    double n = (double)NC * iters * blocks * threads;                                        \
    printf("DADD chains=%2d warps/SM=%3d : %7.2f Gop/s (lane ops)\n", NC, W * BPS, n / ms / 1e6); \
  }
  DA(8, 16, 1) DA(8, 8, 4)
#define MX(ND, NF, W, BPS)                                                                          \
  {                                                                                                 \
    int blocks = sms * BPS, threads = 32 * W;                                                       \
    double ms = timeit([&] { k_mix<ND, NF><<<blocks, threads>>>(d, iters); });                      \
    double nd = (double)ND * iters * blocks * W, nf = (double)NF * iters * blocks * threads;        \
    printf("MIX dmma=%2d dfma=%2d warps/SM=%3d : %.3f ms  dmma %.2f TF + dfma %.2f TF = %.2f TF\n", ND, NF, \
           W * BPS, ms, nd * 512 / ms / 1e9, nf * 2 / ms / 1e9, (nd * 512 + nf * 2) / ms / 1e9);  \
  }
  MX(8, 0, 16, 1) MX(0, 64, 16, 1) MX(8, 64, 16, 1) MX(8, 32, 16, 1) MX(8, 16, 16, 1) MX(4, 32, 16, 1)
  return 0;
}
