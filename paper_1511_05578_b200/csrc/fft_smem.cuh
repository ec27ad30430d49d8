// Power-of-two complex128 FFT held in shared memory, executed by a whole
// thread block: Stockham autosort, radix-4 stages (+ one radix-2 stage when
// log2 P is odd), twiddles from a P-entry table exp(-2 pi i k / P).
// Forward (DIR=-1) is sum x_j e^{-2 pi i jk/P}; inverse (DIR=+1) unnormalised.
#pragma once
#include "scv_internal.cuh"

template <int DIR>
__device__ __forceinline__ double2 tw_get(const double2* __restrict__ tw, int idx) {
  double2 w = __ldg(tw + idx);
  return DIR < 0 ? w : make_double2(w.x, -w.y);
}

// x: P complex in shared memory (natural order in and out).
template <int LOGP, int NT, int DIR>
__device__ __forceinline__ void fft_smem(double2* x, const double2* __restrict__ tw) {
  constexpr int P = 1 << LOGP;
  constexpr int Q4 = P / 4;
  constexpr int IT4 = (Q4 + NT - 1) / NT;
  const int tid = threadIdx.x;
  int Ns = 1;
#pragma unroll 1
  for (int st = 0; st < LOGP / 2; ++st) {
    double2 y[IT4][4];
#pragma unroll
    for (int it = 0; it < IT4; ++it) {
      const int j = tid + it * NT;
      if (j < Q4) {
        const int k = j & (Ns - 1);
        double2 v0 = x[j], v1 = x[j + Q4], v2 = x[j + 2 * Q4], v3 = x[j + 3 * Q4];
        if (Ns > 1) {
          const int step = (P / 4 / Ns) * k;  // r * k * P / (4 Ns)
          v1 = cmul(v1, tw_get<DIR>(tw, step));
          v2 = cmul(v2, tw_get<DIR>(tw, 2 * step));
          v3 = cmul(v3, tw_get<DIR>(tw, 3 * step));
        }
        double2 a0 = cadd(v0, v2), a1 = csub(v0, v2);
        double2 b0 = cadd(v1, v3), b1 = csub(v1, v3);
        // DIR*i*b1
        double2 ib1 = DIR < 0 ? make_double2(b1.y, -b1.x) : make_double2(-b1.y, b1.x);
        y[it][0] = cadd(a0, b0);
        y[it][1] = cadd(a1, ib1);
        y[it][2] = csub(a0, b0);
        y[it][3] = csub(a1, ib1);
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < IT4; ++it) {
      const int j = tid + it * NT;
      if (j < Q4) {
        const int k = j & (Ns - 1);
        const int o = (j - k) * 4 + k;
        x[o] = y[it][0];
        x[o + Ns] = y[it][1];
        x[o + 2 * Ns] = y[it][2];
        x[o + 3 * Ns] = y[it][3];
      }
    }
    __syncthreads();
    Ns *= 4;
  }
  if (LOGP & 1) {
    constexpr int Q2 = P / 2;
    constexpr int IT2 = (Q2 + NT - 1) / NT;
    double2 y[IT2][2];
#pragma unroll
    for (int it = 0; it < IT2; ++it) {
      const int j = tid + it * NT;
      if (j < Q2) {
        const int k = j & (Ns - 1);
        double2 v0 = x[j], v1 = x[j + Q2];
        if (Ns > 1) v1 = cmul(v1, tw_get<DIR>(tw, (P / 2 / Ns) * k));
        y[it][0] = cadd(v0, v1);
        y[it][1] = csub(v0, v1);
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < IT2; ++it) {
      const int j = tid + it * NT;
      if (j < Q2) {
        const int k = j & (Ns - 1);
        const int o = (j - k) * 2 + k;
        x[o] = y[it][0];
        x[o + Ns] = y[it][1];
      }
    }
    __syncthreads();
  }
}
