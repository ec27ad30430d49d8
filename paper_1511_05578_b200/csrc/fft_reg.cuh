// Register-resident power-of-two complex128 FFT for one block (Stockham).
//
// Thread t of NT = P/E threads holds E = 16 (or 8) points at positions
// t + s*NT ("natural distribution").  Each pass applies E/R radix-R
// butterflies per thread entirely in registers; between passes the data
// crosses shared memory ONCE (write at the Stockham output position, read
// back in the natural distribution), with a 1-in-16 padding that keeps the
// stride-16 writes of the first pass bank-conflict free.  Input and output are
// both in the natural distribution, so two transforms can be chained (and
// pointwise spectra applied) without an extra exchange.
// Twiddles: one base value w = e^{DIR 2 pi i a/P} per butterfly from a global
// table (L1-resident), powers w^r formed in registers by a depth-4 product tree.
#pragma once
#include "scv_internal.cuh"

namespace regfft {

__host__ __device__ constexpr double kC16_1 = 0.92387953251128675613;  // cos(pi/8)
__host__ __device__ constexpr double kS16_1 = 0.38268343236508977173;  // sin(pi/8)
__host__ __device__ constexpr double kR2 = 0.70710678118654752440;     // 1/sqrt(2)

// v * e^{DIR 2 pi i k / N} for compile-time k, N in {2,4,8,16}
template <int N, int k, int DIR>
__device__ __forceinline__ double2 rot(double2 v) {
  constexpr int kk = ((k % N) + N) % N;
  constexpr int q = kk * 16 / N;  // in sixteenths of a turn
  // e^{i theta} with theta = DIR * 2 pi q / 16
  if constexpr (q == 0) return v;
  else if constexpr (q == 4) return DIR < 0 ? make_double2(v.y, -v.x) : make_double2(-v.y, v.x);
  else if constexpr (q == 8) return make_double2(-v.x, -v.y);
  else if constexpr (q == 12) return DIR < 0 ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
  else {
    constexpr double c = (q == 2 || q == 14) ? kR2 : (q == 6 || q == 10) ? -kR2 :
                         (q == 1 || q == 15) ? kC16_1 : (q == 3 || q == 13) ? kS16_1 :
                         (q == 5 || q == 11) ? -kS16_1 : -kC16_1;
    constexpr double s0 = (q == 2 || q == 6) ? kR2 : (q == 10 || q == 14) ? -kR2 :
                          (q == 1 || q == 7) ? kS16_1 : (q == 3 || q == 5) ? kC16_1 :
                          (q == 9 || q == 15) ? -kS16_1 : -kC16_1;
    constexpr double s = DIR < 0 ? -s0 : s0;
    return make_double2(v.x * c - v.y * s, v.x * s + v.y * c);
  }
}

template <int DIR>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  const double2 t = a;
  a = make_double2(t.x + b.x, t.y + b.y);
  b = make_double2(t.x - b.x, t.y - b.y);
}

template <int DIR>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 a0 = make_double2(x0.x + x2.x, x0.y + x2.y), a1 = make_double2(x0.x - x2.x, x0.y - x2.y);
  const double2 b0 = make_double2(x1.x + x3.x, x1.y + x3.y), b1 = make_double2(x1.x - x3.x, x1.y - x3.y);
  const double2 ib1 = DIR < 0 ? make_double2(b1.y, -b1.x) : make_double2(-b1.y, b1.x);
  x0 = make_double2(a0.x + b0.x, a0.y + b0.y);
  x2 = make_double2(a0.x - b0.x, a0.y - b0.y);
  x1 = make_double2(a1.x + ib1.x, a1.y + ib1.y);
  x3 = make_double2(a1.x - ib1.x, a1.y - ib1.y);
}

// in-place R-point DFT of v[0..R-1] (natural order in and out)
template <int R, int DIR>
__device__ __forceinline__ void dft(double2* v) {
  if constexpr (R == 2) {
    dft2<DIR>(v[0], v[1]);
  } else if constexpr (R == 4) {
    dft4<DIR>(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<DIR>(e0, e1, e2, e3);
    dft4<DIR>(o0, o1, o2, o3);
    o1 = rot<8, 1, DIR>(o1);
    o2 = rot<8, 2, DIR>(o2);
    o3 = rot<8, 3, DIR>(o3);
    v[0] = make_double2(e0.x + o0.x, e0.y + o0.y); v[4] = make_double2(e0.x - o0.x, e0.y - o0.y);
    v[1] = make_double2(e1.x + o1.x, e1.y + o1.y); v[5] = make_double2(e1.x - o1.x, e1.y - o1.y);
    v[2] = make_double2(e2.x + o2.x, e2.y + o2.y); v[6] = make_double2(e2.x - o2.x, e2.y - o2.y);
    v[3] = make_double2(e3.x + o3.x, e3.y + o3.y); v[7] = make_double2(e3.x - o3.x, e3.y - o3.y);
  } else {  // 16 = 4 x 4
    double2 a[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      a[r][0] = v[r]; a[r][1] = v[r + 4]; a[r][2] = v[r + 8]; a[r][3] = v[r + 12];
      dft4<DIR>(a[r][0], a[r][1], a[r][2], a[r][3]);
    }
    a[1][1] = rot<16, 1, DIR>(a[1][1]); a[1][2] = rot<16, 2, DIR>(a[1][2]); a[1][3] = rot<16, 3, DIR>(a[1][3]);
    a[2][1] = rot<16, 2, DIR>(a[2][1]); a[2][2] = rot<16, 4, DIR>(a[2][2]); a[2][3] = rot<16, 6, DIR>(a[2][3]);
    a[3][1] = rot<16, 3, DIR>(a[3][1]); a[3][2] = rot<16, 6, DIR>(a[3][2]); a[3][3] = rot<16, 9, DIR>(a[3][3]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      double2 b0 = a[0][k1], b1 = a[1][k1], b2 = a[2][k1], b3 = a[3][k1];
      dft4<DIR>(b0, b1, b2, b3);
      v[k1] = b0; v[k1 + 4] = b1; v[k1 + 8] = b2; v[k1 + 12] = b3;
    }
  }
}

__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_size(int P) { return P + P / 16; }

__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// powers w^1..w^(R-1) in place: v[r] *= w^r (product tree of depth <= 4,
// each power applied as soon as it exists)
template <int R>
__device__ __forceinline__ void twiddle(double2* v, double2 w) {
  v[1] = cm(v[1], w);
  if constexpr (R > 2) {
    const double2 w2 = cm(w, w), w3 = cm(w2, w);
    v[2] = cm(v[2], w2);
    v[3] = cm(v[3], w3);
    if constexpr (R > 4) {
      const double2 w4 = cm(w2, w2);
      v[4] = cm(v[4], w4);
      v[5] = cm(v[5], cm(w4, w));
      v[6] = cm(v[6], cm(w4, w2));
      v[7] = cm(v[7], cm(w4, w3));
      if constexpr (R > 8) {
        const double2 w8 = cm(w4, w4), w5 = cm(w4, w), w6 = cm(w4, w2), w7 = cm(w4, w3);
        v[8] = cm(v[8], w8);
        v[9] = cm(v[9], cm(w8, w));
        v[10] = cm(v[10], cm(w8, w2));
        v[11] = cm(v[11], cm(w8, w3));
        v[12] = cm(v[12], cm(w8, w4));
        v[13] = cm(v[13], cm(w8, w5));
        v[14] = cm(v[14], cm(w8, w6));
        v[15] = cm(v[15], cm(w8, w7));
      }
    }
  }
}

// One Stockham pass with radix R on the natural distribution x[E].  Each
// butterfly is stored as soon as it is computed (no staging copy of the
// outputs, which keeps the live set at E + a few twiddle powers).  The LAST
// pass writes its outputs back into x in place: butterfly u reads
// x[u + r*BPT] and writes x[u + q*BPT], disjoint from every other butterfly.
template <int LOGP, int E, int R, int LOGNS, int DIR, bool LAST>
__device__ __forceinline__ void pass(double2 (&x)[E], double2* sm, const double2* __restrict__ tw, int t) {
  constexpr int P = 1 << LOGP, NT = P / E, NS = 1 << LOGNS, BPT = E / R;
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    const int j = t + u * NT;
    const int k = j & (NS - 1);
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = x[u + r * BPT];
    if constexpr (NS > 1) {
      double2 w = __ldg(tw + k * (P / (NS * R)));  // e^{-2 pi i a/P}
      if (DIR > 0) w.y = -w.y;
      twiddle<R>(v, w);
    }
    dft<R, DIR>(v);
    if constexpr (LAST) {
#pragma unroll
      for (int q = 0; q < R; ++q) x[u + q * BPT] = v[q];
    } else {
      const int ob = (j - k) * R + k;
#pragma unroll
      for (int q = 0; q < R; ++q) sm[pad16(ob + q * NS)] = v[q];
    }
  }
  if constexpr (!LAST) {
    __syncthreads();
#pragma unroll
    for (int s = 0; s < E; ++s) x[s] = sm[pad16(t + s * NT)];
    __syncthreads();
  }
}

template <int LOGP, int E, int LOGNS, int DIR>
__device__ __forceinline__ void passes(double2 (&x)[E], double2* sm, const double2* __restrict__ tw, int t) {
  constexpr int LOGE = E == 16 ? 4 : E == 8 ? 3 : 2;
  constexpr int REM = LOGP - LOGNS;
  constexpr int LOGR = REM < LOGE ? REM : LOGE;
  if constexpr (REM > 0) {
    pass<LOGP, E, (1 << LOGR), LOGNS, DIR, (REM == LOGR)>(x, sm, tw, t);
    passes<LOGP, E, LOGNS + LOGR, DIR>(x, sm, tw, t);
  }
}

// Full P-point FFT (DIR -1 forward, +1 inverse, unnormalised) of the block's
// natural-distribution registers.  sm: padded_size(P) double2 of shared memory.
// Precondition: no thread is still reading sm from a previous use (caller syncs).
// t = threadIdx.x; callers inside a persistent loop pass an opaque copy so the
// per-pass addresses are not hoisted out of the loop (hundreds of live values).
template <int LOGP, int E, int DIR>
__device__ __forceinline__ void fft(double2 (&x)[E], double2* sm, const double2* __restrict__ tw,
                                    int t = threadIdx.x) {
  passes<LOGP, E, 0, DIR>(x, sm, tw, t);
}

}  // namespace regfft
