// Alpha / gamma stages of the SO(3) transforms on the prime-factor DFT engine
// (pfa.cuh), for the Mersenne grid lengths K = 2^k - 1 of the lambda = 2
// tilings.  Other lengths fall back to cuFFT (so3.cu).
//
// Analysis  (so3.py:259-285 restated, see so3.cu for the closed form):
//   k_ana_alpha  : generate fac W_{mn} d^l_{mn}(beta_b) for R rows (n, b) in
//                  shared memory, inverse K-point DFT over m -> alpha, store
//                  rows of the (gamma-slot, beta, alpha) volume.  One HBM write.
//   k_ana_gamma  : R adjacent alpha columns of one beta slab, inverse DFT over
//                  n -> gamma in place (real path: Hermitian columns packed
//                  two per complex transform).
// Synthesis (so3.py:195-200 + the |m|<=|n| pruning of so3.py:240):
//   k_syn_alpha  : forward DFT of R rows (g, b) of the input into a beta-chunk
//                  buffer [b][g][m] (real input: two rows per complex transform).
//   k_syn_gamma  : R adjacent m columns of the chunk, forward DFT over
//                  g -> n, keep |m| <= |n| and scatter into the beta-contiguous
//                  columns W1p[(n,m)][b] consumed by the beta stage.
// All kernels are persistent (grid = resident CTAs) and stage the coefficient
// tables in shared memory once.

#include <algorithm>
#include <cmath>
#include <cstring>

#include "pfa.cuh"

typedef long double ld;

bool scv_pfa_supported(int K) {
  switch (K) {
    case 3: case 7: case 15: case 31: case 63: case 255: case 511: case 1023: case 2047:
    case 4095: return true;
    default: return false;
  }
}

static void factors_of(int K, int f[4]) {
  f[0] = f[1] = f[2] = f[3] = 1;
  switch (K) {
    case 3: f[0] = 3; break;
    case 7: f[0] = 7; break;
    case 15: f[0] = 3; f[1] = 5; break;
    case 31: f[0] = 31; break;
    case 63: f[0] = 7; f[1] = 9; break;
    case 127: f[0] = 127; break;
    case 255: f[0] = 3; f[1] = 5; f[2] = 17; break;
    case 511: f[0] = 7; f[1] = 73; break;
    case 1023: f[0] = 3; f[1] = 11; f[2] = 31; break;
    case 2047: f[0] = 23; f[1] = 89; break;
    case 4095: f[0] = 5; f[1] = 7; f[2] = 9; f[3] = 13; break;
  }
}

int scv_pfa_tables(scv_ctx* c, int K, const double2** out) {
  const std::string key = "pfa_" + std::to_string(K);
  auto it = c->aux.find(key);
  if (it != c->aux.end()) {
    *out = (const double2*)it->second;
    return SCV_OK;
  }
  int f[4];
  factors_of(K, f);
  std::vector<double2> tab;
  const ld twopi = 6.283185307179586476925286766559005768L;
  for (int s = 0; s < 4; ++s) {
    const int p = f[s];
    if (p == 1) continue;
    if (pfa_use_mma(p)) {
      // dense C and S matrices (M rows x pitch doubles each), row 0 = (1, 0)
      const int h = (p - 1) / 2, M = mma_M(p), PA = mma_pitch(mma_Kp(p));
      std::vector<double> C((size_t)M * PA, 0.0), S((size_t)M * PA, 0.0);
      for (int k = 0; k <= h; ++k)
        for (int j = 1; j <= h; ++j) {
          const ld a = twopi * (ld)(((long long)j * k) % p) / (ld)p;
          C[(size_t)k * PA + (j - 1)] = (double)cosl(a);
          S[(size_t)k * PA + (j - 1)] = (double)sinl(a);
        }
      const size_t base = tab.size();
      tab.resize(base + (size_t)M * PA);
      double* dst = (double*)(tab.data() + base);
      memcpy(dst, C.data(), C.size() * sizeof(double));
      memcpy(dst + C.size(), S.data(), S.size() * sizeof(double));
      continue;
    }
    for (int i = 0; i < p; ++i) {
      const ld a = twopi * (ld)i / (ld)p;
      tab.push_back(make_double2((double)cosl(a), (double)sinl(a)));
    }
  }
  if (tab.empty()) tab.push_back(make_double2(0.0, 0.0));
  void* d = nullptr;
  SCV_CUDA(c, cudaMalloc(&d, tab.size() * sizeof(double2)));
  SCV_CUDA(c, cudaMemcpy(d, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice));
  c->aux[key] = d;
  *out = (const double2*)d;
  return SCV_OK;
}

// Launch shapes per length.  ROW kernels (alpha passes) and COL kernels
// (gamma passes, R adjacent columns so each 16-byte element of a row is part
// of an R*16-byte contiguous segment) each use R transforms per batch, NT
// threads (every stage's work items fit one pass for the large radices) and
// MINB resident CTAs per SM.  Batches are double-buffered in shared memory:
// the next batch streams in with cp.async while the current one computes.
template <int K, bool COL> struct PfaCfg;
#define SCV_PFA_CFG(KK, CL, RR, NNT, MB) \
  template <> struct PfaCfg<KK, CL> { static constexpr int R = RR, NT = NNT, MINB = MB; };
SCV_PFA_CFG(3, false, 64, 128, 2)    SCV_PFA_CFG(3, true, 64, 128, 2)
SCV_PFA_CFG(7, false, 64, 128, 2)    SCV_PFA_CFG(7, true, 64, 128, 2)
SCV_PFA_CFG(15, false, 32, 128, 2)   SCV_PFA_CFG(15, true, 32, 128, 2)
SCV_PFA_CFG(31, false, 16, 128, 2)   SCV_PFA_CFG(31, true, 16, 128, 2)
SCV_PFA_CFG(63, false, 16, 256, 2)   SCV_PFA_CFG(63, true, 16, 256, 2)
SCV_PFA_CFG(255, false, 8, 256, 2)   SCV_PFA_CFG(255, true, 8, 256, 2)
SCV_PFA_CFG(511, false, 4, 256, 2)   SCV_PFA_CFG(511, true, 4, 256, 2)
#ifndef SCV_ROW2047
#define SCV_ROW2047 1, 192, 2
#endif
#ifndef SCV_COL2047
#define SCV_COL2047 2, 384, 1
#endif
#ifndef SCV_ROW1023
#define SCV_ROW1023 2, 224, 2
#endif
#define SCV_PFA_CFG_(KK, CL, ...) SCV_PFA_CFG(KK, CL, __VA_ARGS__)
SCV_PFA_CFG_(1023, false, SCV_ROW1023)  SCV_PFA_CFG(1023, true, 2, 224, 2)
SCV_PFA_CFG_(2047, false, SCV_ROW2047)  SCV_PFA_CFG_(2047, true, SCV_COL2047)
SCV_PFA_CFG(4095, false, 1, 320, 1)  SCV_PFA_CFG(4095, true, 1, 320, 1)

template <int K, bool COL>
static size_t pfa_smem() {
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, COL>::R;
  return ((size_t)2 * R * K + pfa_tab_total<PL>() + pfa_scratch<PL, R>()) * sizeof(double2) + R * sizeof(int4);
}

// ---------------------------------------------------------------------------
// batched rows (test / benchmark entry): out[r][k] = sum_n in[r][n] e^{DIR 2 pi i nk/K}
// ---------------------------------------------------------------------------
template <int K, int DIR>
__global__ void __launch_bounds__(PfaCfg<K, false>::NT, PfaCfg<K, false>::MINB)
    k_pfa_rows(long long nrows, const double2* __restrict__ in, double2* __restrict__ out,
               const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, false>::R, NT = PfaCfg<K, false>::NT;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const buf0 = scr + pfa_scratch<PL, R>();  // buffer c at buf0 + c * R * K (stays a shared pointer)
  pfa_load_tables<PL, NT>(tab, gtab);
  const long long nb = (nrows + R - 1) / R;
  auto issue = [&](long long bt, double2* X) {
    const long long r0 = bt * R;
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, n = i - r * K;
      if (r0 + r < nrows) cp_async16(X + i, in + (r0 + r) * K + n);
      else X[i] = make_double2(0.0, 0.0);
    }
    cp_async_commit();
  };
  long long bt = blockIdx.x;
  int cur = 0;
  if (bt < nb) issue(bt, buf0);
#pragma unroll 1
  for (; bt < nb; bt += gridDim.x) {
    const long long nx = bt + gridDim.x;
    if (nx < nb) issue(nx, buf0 + (cur ^ 1) * (R * K));
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double2* X = buf0 + cur * (R * K);
    pfa_dft<PL, DIR, R, NT, K>(X, tab, scr);
    const long long r0 = bt * R;
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, k = i - r * K;
      if (r0 + r < nrows) out[(r0 + r) * K + k] = X[r * K + pfa_pos<PL>(k)];
    }
    __syncthreads();
    cur ^= 1;
  }
}

// ---------------------------------------------------------------------------
// analysis alpha: generate + inverse DFT over m, R rows (gi, b) per batch
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(PfaCfg<K, false>::NT, PfaCfg<K, false>::MINB)
    k_ana_alpha(int real, const double2* __restrict__ w, const double* __restrict__ hlb,
                const double* __restrict__ lsin, const double* __restrict__ lcos, double2* __restrict__ out,
                const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, false>::R, NT = PfaCfg<K, false>::NT;
  constexpr int L = (K + 1) / 2;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* X = scr + pfa_scratch<PL, R>();
  int4* rp = (int4*)(X + 2 * R * K);  // per-row (gi, b, n, l)
  pfa_load_tables<PL, NT>(tab, gtab);
  const long long nrows = (long long)(real ? L : K) * L;
  const long long nb = (nrows + R - 1) / R;
#pragma unroll 1
  for (long long bt = blockIdx.x; bt < nb; bt += gridDim.x) {
    if (threadIdx.x < R) {
      const long long ri = bt * R + threadIdx.x;
      int gi = -1, b = 0, n = 0;
      if (ri < nrows) {
        gi = (int)(ri / L);
        b = (int)(ri - (long long)gi * L);
        n = real ? gi : (gi <= L - 1 ? gi : gi - K);
      }
      rp[threadIdx.x] = make_int4(gi, b, n, n < 0 ? -n : n);
    }
    __syncthreads();
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, q = i - r * K;
      const int4 P = rp[r];
      const int l = P.w, n = P.z;
      const int m = q <= L - 1 ? q : q - K;
      double2 v = make_double2(0.0, 0.0);
      if (P.x >= 0 && m >= -l && m <= l) {
        const int am = m < 0 ? -m : m;
        const int es = n >= 0 ? l - m : l + m;
        const int ec = n >= 0 ? l + m : l - m;
        double lg = hlb[(long long)l * (l + 1) / 2 + am];
        if (es) lg += (double)es * lsin[P.y];
        if (ec) lg += (double)ec * lcos[P.y];
        double d = exp(lg);
        if (n < 0 && ((l - m) & 1)) d = -d;
        const double2 cw = w[((long long)(n >= 0 ? 0 : 1) * L + l) * K + (L - 1) + m];
        const double f = (double)(2 * l + 1) / (8.0 * SCV_PI * SCV_PI) * d;
        v = make_double2(f * cw.x, f * cw.y);
      }
      X[i] = v;
    }
    __syncthreads();
    pfa_dft<PL, +1, R, NT, K>(X, tab, scr);
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, a = i - r * K;
      const int4 P = rp[r];
      if (P.x >= 0) out[((long long)P.x * L + P.y) * K + a] = X[r * K + pfa_pos<PL>(a)];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// analysis gamma: R adjacent alpha columns of one beta slab, inverse over n.
// complex: in place on sig (K, L, K), double-buffered.  real: src = T
// (L, L, K) complex half spectrum (n >= 0), dst = real sig (K, L, K); two
// Hermitian columns per complex transform.
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(PfaCfg<K, true>::NT, PfaCfg<K, true>::MINB)
    k_ana_gamma(int real, double2* __restrict__ src, double* __restrict__ dst_real,
                const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, true>::R, NT = PfaCfg<K, true>::NT;
  constexpr int L = (K + 1) / 2;
  constexpr long long LK = (long long)L * K;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const buf0 = scr + pfa_scratch<PL, R>();  // buffer c at buf0 + c * R * K (stays a shared pointer)
  pfa_load_tables<PL, NT>(tab, gtab);
  const int cpb = real ? 2 * R : R;  // columns per batch
  const int ngrp = (K + cpb - 1) / cpb;
  const long long nb = (long long)L * ngrp;
  auto issue = [&](long long bt, double2* X) {
    const int b = (int)(bt / ngrp);
    const int a0 = (int)(bt - (long long)b * ngrp) * cpb;
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int g = i / R, r = i - g * R;
      const int a = a0 + r;
      if (a < K) cp_async16(X + r * K + g, src + (long long)g * LK + (long long)b * K + a);
      else X[r * K + g] = make_double2(0.0, 0.0);
    }
    cp_async_commit();
  };
  long long bt = blockIdx.x;
  int cur = 0;
  if (!real && bt < nb) issue(bt, buf0);
#pragma unroll 1
  for (; bt < nb; bt += gridDim.x) {
    const int b = (int)(bt / ngrp);
    const int a0 = (int)(bt - (long long)b * ngrp) * cpb;
    double2* X = buf0 + cur * (R * K);
    if (!real) {
      const long long nx = bt + gridDim.x;
      if (nx < nb) issue(nx, buf0 + (cur ^ 1) * (R * K));
      else cp_async_commit();
      cp_async_wait<1>();
    } else {
      // Z[n] = T1[n] + i T2[n], Z[-n] = conj(T1[n]) + i conj(T2[n]); Im of n = 0 dropped
#pragma unroll 4
      for (int i = threadIdx.x; i < R * L; i += NT) {
        const int n = i / R, r = i - n * R;
        const int a1 = a0 + 2 * r, a2 = a1 + 1;
        double2 t1 = (a1 < K) ? src[(long long)n * LK + (long long)b * K + a1] : make_double2(0.0, 0.0);
        double2 t2 = (a2 < K) ? src[(long long)n * LK + (long long)b * K + a2] : make_double2(0.0, 0.0);
        if (n == 0) {
          t1.y = 0.0;
          t2.y = 0.0;
        }
        X[r * K + n] = make_double2(t1.x - t2.y, t1.y + t2.x);
        if (n > 0) X[r * K + K - n] = make_double2(t1.x + t2.y, -t1.y + t2.x);
      }
    }
    __syncthreads();
    pfa_dft<PL, +1, R, NT, K>(X, tab, scr);
    if (!real) {
#pragma unroll 4
      for (int i = threadIdx.x; i < R * K; i += NT) {
        const int g = i / R, r = i - g * R;
        const int a = a0 + r;
        if (a < K) src[(long long)g * LK + (long long)b * K + a] = X[r * K + pfa_pos<PL>(g)];
      }
    } else {
#pragma unroll 4
      for (int i = threadIdx.x; i < 2 * R * K; i += NT) {
        const int g = i / (2 * R), c = i - g * (2 * R);
        const int r = c >> 1;
        const int a = a0 + c;
        if (a < K) {
          const double2 z = X[r * K + pfa_pos<PL>(g)];
          dst_real[(long long)g * LK + (long long)b * K + a] = (c & 1) ? z.y : z.x;
        }
      }
    }
    __syncthreads();
    if (!real) cur ^= 1;
  }
}

// ---------------------------------------------------------------------------
// synthesis alpha: forward DFT of rows (g, b) for b in [b0, b0+nbb) into
// chunk[(b-b0)][g][m] (complex, double-buffered).  real input: two rows per
// complex transform.
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(PfaCfg<K, false>::NT, PfaCfg<K, false>::MINB)
    k_syn_alpha(int real, const void* __restrict__ in, int b0, int nbb, double2* __restrict__ chunk,
                const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, false>::R, NT = PfaCfg<K, false>::NT;
  constexpr int L = (K + 1) / 2;
  constexpr long long LK = (long long)L * K;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const buf0 = scr + pfa_scratch<PL, R>();  // buffer c at buf0 + c * R * K (stays a shared pointer)
  pfa_load_tables<PL, NT>(tab, gtab);
  const long long nrows = (long long)K * nbb;  // row index = bb*K + g
  const int rpb = real ? 2 * R : R;
  const long long nb = (nrows + rpb - 1) / rpb;
  const double2* F = (const double2*)in;
  auto issue = [&](long long bt, double2* X) {
    const long long r0 = bt * rpb;
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, a = i - r * K;
      const long long ri = r0 + r;
      if (ri < nrows) {
        const int bb = (int)(ri / K), g = (int)(ri - (long long)bb * K);
        cp_async16(X + i, F + (long long)g * LK + (long long)(b0 + bb) * K + a);
      } else {
        X[i] = make_double2(0.0, 0.0);
      }
    }
    cp_async_commit();
  };
  long long bt = blockIdx.x;
  int cur = 0;
  if (!real && bt < nb) issue(bt, buf0);
#pragma unroll 1
  for (; bt < nb; bt += gridDim.x) {
    const long long r0 = bt * rpb;
    double2* X = buf0 + cur * (R * K);
    if (!real) {
      const long long nx = bt + gridDim.x;
      if (nx < nb) issue(nx, buf0 + (cur ^ 1) * (R * K));
      else cp_async_commit();
      cp_async_wait<1>();
    } else {
      const double* Fr = (const double*)in;
#pragma unroll 4
      for (int i = threadIdx.x; i < R * K; i += NT) {
        const int r = i / K, a = i - r * K;
        double v1 = 0.0, v2 = 0.0;
        const long long ri1 = r0 + 2 * r, ri2 = ri1 + 1;
        if (ri1 < nrows) {
          const int bb = (int)(ri1 / K), g = (int)(ri1 - (long long)bb * K);
          v1 = Fr[(long long)g * LK + (long long)(b0 + bb) * K + a];
        }
        if (ri2 < nrows) {
          const int bb = (int)(ri2 / K), g = (int)(ri2 - (long long)bb * K);
          v2 = Fr[(long long)g * LK + (long long)(b0 + bb) * K + a];
        }
        X[i] = make_double2(v1, v2);
      }
    }
    __syncthreads();
    pfa_dft<PL, -1, R, NT, K>(X, tab, scr);
    if (!real) {
#pragma unroll 4
      for (int i = threadIdx.x; i < R * K; i += NT) {
        const int r = i / K, m = i - r * K;
        const long long ri = r0 + r;
        if (ri < nrows) chunk[ri * K + m] = X[r * K + pfa_pos<PL>(m)];
      }
    } else {
      // Z = X1 + i X2 (X1, X2 Hermitian): X1[k] = (Z[k] + conj Z[-k])/2, X2[k] = (Z[k] - conj Z[-k])/(2i)
#pragma unroll 4
      for (int i = threadIdx.x; i < 2 * R * K; i += NT) {
        const int c = i / K, m = i - c * K;
        const int r = c >> 1;
        const long long ri = r0 + c;
        if (ri < nrows) {
          const double2 z = X[r * K + pfa_pos<PL>(m)];
          const double2 zc = X[r * K + pfa_pos<PL>(m == 0 ? 0 : K - m)];
          double2 v;
          if ((c & 1) == 0) v = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
          else v = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
          chunk[ri * K + m] = v;
        }
      }
    }
    __syncthreads();
    if (!real) cur ^= 1;
  }
}

// ---------------------------------------------------------------------------
// synthesis gamma + extraction: columns (bb, m) of the chunk, forward over g.
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long w1p_colbase(int n, int real) {
  const long long l = n < 0 ? -n : n;
  if (real) return l * l;
  if (l == 0) return 0;
  return n > 0 ? 2 * l * l - 1 : 2 * l * l + 2 * l;
}

template <int K>
__global__ void __launch_bounds__(PfaCfg<K, true>::NT, PfaCfg<K, true>::MINB)
    k_syn_gamma(int real, const double2* __restrict__ chunk, int b0, int nbb, double2* __restrict__ W1p,
                const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, true>::R, NT = PfaCfg<K, true>::NT;
  constexpr int L = (K + 1) / 2;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const buf0 = scr + pfa_scratch<PL, R>();  // buffer c at buf0 + c * R * K (stays a shared pointer)
  pfa_load_tables<PL, NT>(tab, gtab);
  const int ngrp = (K + R - 1) / R;
  const long long nb = (long long)nbb * ngrp;
  auto issue = [&](long long bt, double2* X) {
    const int bb = (int)(bt / ngrp);
    const int q0 = (int)(bt - (long long)bb * ngrp) * R;
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int g = i / R, r = i - g * R;
      const int q = q0 + r;
      if (q < K) cp_async16(X + r * K + g, chunk + ((long long)bb * K + g) * K + q);
      else X[r * K + g] = make_double2(0.0, 0.0);
    }
    cp_async_commit();
  };
  long long bt = blockIdx.x;
  int cur = 0;
  if (bt < nb) issue(bt, buf0);
#pragma unroll 1
  for (; bt < nb; bt += gridDim.x) {
    const int bb = (int)(bt / ngrp);
    const int q0 = (int)(bt - (long long)bb * ngrp) * R;
    const long long nx = bt + gridDim.x;
    if (nx < nb) issue(nx, buf0 + (cur ^ 1) * (R * K));
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double2* X = buf0 + cur * (R * K);
    pfa_dft<PL, -1, R, NT, K>(X, tab, scr);
    // keep |m| <= |n| (real: n >= 0 only)
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, gn = i - r * K;
      const int q = q0 + r;
      if (q >= K) continue;
      const int m = q <= L - 1 ? q : q - K;
      const int n = gn <= L - 1 ? gn : gn - K;
      const int am = m < 0 ? -m : m, an = n < 0 ? -n : n;
      if (am > an || (real && n < 0)) continue;
      W1p[(w1p_colbase(n, real) + m + an) * (long long)L + b0 + bb] = X[r * K + pfa_pos<PL>(gn)];
    }
    __syncthreads();
    cur ^= 1;
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
template <typename Kern>
static int persistent_grid(scv_ctx* c, Kern k, int nt, size_t sm, long long nbatches, int* grid) {
  SCV_CUDA(c, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per = 0, sms = 0;
  SCV_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, nt, sm));
  SCV_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  if (per < 1) per = 1;
  long long g = (long long)per * sms;
  if (g > nbatches) g = nbatches;
  if (g < 1) g = 1;
  *grid = (int)g;
  return SCV_OK;
}

// ---------------------------------------------------------------------------
// beta stage + Delta contraction of the SO(3) forward transform on the
// prime-factor engine (restates so3.py:203-243; the packed-pair formulation
// is documented in beta.cu).  Per (n, column pair):
//   X1 <- packed extension of the two columns (natural b order)
//   X1 <- DFT_K (forward, CRT order);  F[m''] = (1/K) e^{-i m'' pi/K} X1[pos(m'' mod K)]
//   X1 <- F (natural);  X2 <- G = F - (gamma/2)(-1)^m'' wrapped mod K2 = 4L-1
//   X2 <- IDFT_K2( DFT_K2(X2) * DFT_K2(w_even)/K2 )   (the forward output is in
//         CRT order and the inverse consumes CRT order, returning natural order)
//   then Y_E / Y_O and the contraction exactly as in beta.cu.
// K2 = 4L-1 >= 4L-3 keeps the circular convolution alias-free for |m'| <= L-1.
// ---------------------------------------------------------------------------
int scv_pfa_pos_host(int K, int k) {
  int f[4];
  factors_of(K, f);
  long long a = 0;
  for (int s = 0; s < 4; ++s)
    if (f[s] > 1) a += (long long)(k % f[s]) * (K / f[s]);
  return (int)(a % K);
}

bool scv_pfa_beta_supported(int L) {
  return L >= 128 && L <= 1024 && scv_pfa_supported(2 * L - 1) && scv_pfa_supported(4 * L - 1);
}

// Three batched kernels over chunks of (n, pair) tasks; F and E go through a
// chunk scratch buffer so each transform runs as an efficient batch:
//   k_beta_f<K>   : packed extension -> DFT_K -> F (natural), gamma per task
//   k_beta_e<K2>  : G (wrapped) -> DFT_K2 -> * w spectrum -> IDFT_K2 -> E (|m'| <= L-1)
//   k_beta_c<L>   : Y_E / Y_O and the Delta contraction, one warp per task
template <int K>
__global__ void __launch_bounds__(PfaCfg<K, false>::NT, PfaCfg<K, false>::MINB)
    k_beta_f(int real, const double2* __restrict__ W1p, const int2* __restrict__ tasks, int t0, int ntask,
             const double2* __restrict__ phs, double2* __restrict__ Fbuf, double2* __restrict__ gam,
             const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, false>::R, NT = PfaCfg<K, false>::NT;
  constexpr int L = (K + 1) / 2;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* X = scr + pfa_scratch<PL, R>();
  pfa_load_tables<PL, NT>(tab, gtab);
  const long long nb = (ntask + R - 1) / R;
#pragma unroll 1
  for (long long bt = blockIdx.x; bt < nb; bt += gridDim.x) {
    const int r0 = (int)(bt * R);
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, b = i - r * K;
      double2 e = make_double2(0.0, 0.0);
      if (r0 + r < ntask) {
        const int2 tk = tasks[t0 + r0 + r];
        const int n = tk.x, l = n < 0 ? -n : n;
        const int m0 = -l + 2 * tk.y, m1 = m0 + 1;
        const long long cb = w1p_colbase(n, real);
        const bool even0 = ((n + m0) & 1) == 0;
        const int src = b < L ? b : 2 * L - 2 - b;
        const double2 v0 = W1p[(cb + m0 + l) * (long long)L + src];
        const double2 v1 = (m1 <= l) ? W1p[(cb + m1 + l) * (long long)L + src] : make_double2(0.0, 0.0);
        const double2 ve = even0 ? v0 : v1;
        double2 vo = even0 ? v1 : v0;
        if (b >= L) vo = make_double2(-vo.x, -vo.y);
        e = make_double2(ve.x + vo.x, ve.y + vo.y);
        if (b == L - 1) gam[r0 + r] = make_double2(vo.x * (2.0 / K), vo.y * (2.0 / K));
      }
      X[i] = e;
    }
    __syncthreads();
    pfa_dft<PL, -1, R, NT, K>(X, tab, scr);
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, q = i - r * K;
      if (r0 + r < ntask) {
        int kk = q - (L - 1);
        if (kk < 0) kk += K;
        Fbuf[(long long)(r0 + r) * K + q] = cmul(__ldg(phs + q), X[r * K + pfa_pos<PL>(kk)]);
      }
    }
    __syncthreads();
  }
}

template <int K2>
__global__ void __launch_bounds__(PfaCfg<K2, false>::NT, PfaCfg<K2, false>::MINB)
    k_beta_e(int ntask, const double2* __restrict__ Fbuf, const double2* __restrict__ gam,
             const double* __restrict__ wfpos, double2* __restrict__ Ebuf, const double2* __restrict__ gtab) {
  using PL = PfaPlan<K2>;
  constexpr int R = PfaCfg<K2, false>::R, NT = PfaCfg<K2, false>::NT;
  constexpr int L = (K2 + 1) / 4, K = 2 * L - 1;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* X = scr + pfa_scratch<PL, R>();
  pfa_load_tables<PL, NT>(tab, gtab);
  const long long nb = (ntask + R - 1) / R;
#pragma unroll 1
  for (long long bt = blockIdx.x; bt < nb; bt += gridDim.x) {
    const int r0 = (int)(bt * R);
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K2; i += NT) {
      const int r = i / K2, p = i - r * K2;
      const int mpp = p <= L - 1 ? p : p - K2;
      double2 v = make_double2(0.0, 0.0);
      if (r0 + r < ntask && mpp >= -(L - 1)) {
        const double2 F = Fbuf[(long long)(r0 + r) * K + mpp + L - 1];
        const double2 g = gam[r0 + r];
        const double hh = (mpp & 1) ? -0.5 : 0.5;
        v = make_double2(F.x - hh * g.x, F.y - hh * g.y);
      }
      X[i] = v;
    }
    __syncthreads();
    pfa_dft_ool<PL, -1, R, NT, K2>(X, tab, scr);
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K2; i += NT) {
      const int p = i - (i / K2) * K2;
      const double f = __ldg(wfpos + p);
      X[i] = make_double2(X[i].x * f, X[i].y * f);
    }
    __syncthreads();
    pfa_dft_ool<PL, +1, R, NT, K2>(X, tab, scr);
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, q = i - r * K;
      const int mp = q - (L - 1);
      if (r0 + r < ntask) Ebuf[(long long)(r0 + r) * K + q] = X[r * K2 + (mp >= 0 ? mp : mp + K2)];
    }
    __syncthreads();
  }
}

template <int L>
__global__ void __launch_bounds__(256) k_beta_c(int real, const int2* __restrict__ tasks, int t0, int ntask,
                                                const double2* __restrict__ Fbuf, const double2* __restrict__ Ebuf,
                                                const double2* __restrict__ gam, const double* __restrict__ Aalt,
                                                const double* __restrict__ delta, double pref,
                                                double2* __restrict__ wout) {
  constexpr int K = 2 * L - 1;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= ntask) return;
  const int2 tk = tasks[t0 + warp];
  const int n = tk.x, l = n < 0 ? -n : n;
  const int m0 = -l + 2 * tk.y, m1 = m0 + 1;
  const bool even0 = ((n + m0) & 1) == 0;
  const int mE = even0 ? m0 : m1, mO = even0 ? m1 : m0;
  const double2* F = Fbuf + (long long)warp * K + (L - 1);  // F[m''] at F[m'']
  const double2* E = Ebuf + (long long)warp * K + (L - 1);
  const double2 g = gam[warp];
  const double hp = 0.5 * SCV_PI;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int mp = -l + lane; mp <= l; mp += 32) {
    const double2 Ep = E[mp], Em = E[-mp];
    const double2 ee = make_double2(0.5 * (Ep.x + Em.x), 0.5 * (Ep.y + Em.y));
    const double2 eo = make_double2(0.5 * (Ep.x - Em.x), 0.5 * (Ep.y - Em.y));
    double2 xe[2], xo[2];
#pragma unroll
    for (int z = 0; z < 2; ++z) {
      const int k = z == 0 ? mp + 1 : mp - 1;
      if (k < -(L - 1) || k > L - 1) {
        xe[z] = make_double2(0.0, 0.0);
        xo[z] = make_double2(0.0, 0.0);
      } else {
        const double2 a = F[k], b = F[-k];
        const double hh = (k & 1) ? -1.0 : 1.0;
        xe[z] = make_double2(0.5 * (a.x + b.x - hh * g.x), 0.5 * (a.y + b.y - hh * g.y));
        xo[z] = make_double2(0.5 * (a.x - b.x + hh * g.x), 0.5 * (a.y - b.y + hh * g.y));
      }
    }
    const double2 dE = make_double2(xe[0].x - xe[1].x, xe[0].y - xe[1].y);
    const double2 dO = make_double2(xo[0].x - xo[1].x, xo[0].y - xo[1].y);
    const double2 yE = make_double2(ee.x - hp * dE.y, ee.y + hp * dE.x);
    const double aa = 0.5 * __ldg(Aalt + mp + L - 1);
    const double2 yO = make_double2(eo.x + aa * g.x - hp * dO.y, eo.y + aa * g.y + hp * dO.x);
    const double dn = wedge_get(delta, l, mp, n);
    const double dE2 = (mE <= l) ? wedge_get(delta, l, mp, mE) * dn : 0.0;
    const double dO2 = (mO <= l) ? wedge_get(delta, l, mp, mO) * dn : 0.0;
    acc[0] += dE2 * yE.x;
    acc[1] += dE2 * yE.y;
    acc[2] += dO2 * yO.x;
    acc[3] += dO2 * yO.y;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  if (lane == 0) {
    const int c = L - 1;
    const int sheet = n >= 0 ? 0 : 1;
    double2* row = wout + ((long long)sheet * L + l) * K;
    const int ms[2] = {mE, mO};
    for (int i = 0; i < 2; ++i) {
      const int m = ms[i];
      if (m > l) continue;
      const double2 v = cipow(make_double2(pref * acc[2 * i], pref * acc[2 * i + 1]), m - n);
      row[c + m] = v;
      if (real && n > 0) {  // row(-n)[m] = (-1)^{m+n} conj(row(n)[-m])  (so3.py:379-382)
        double2 cv = make_double2(v.x, -v.y);
        if ((m + n) & 1) cv = make_double2(-cv.x, -cv.y);
        wout[((long long)1 * L + l) * K + c - m] = cv;
      }
    }
  }
}

static int beta_pfa_tasks(scv_ctx* c, int L, int real, const int2** out, int* count) {
  const std::string key = "pfatasks_" + std::to_string(L) + "_" + std::to_string(real);
  std::vector<int2> v;
  for (int l = L - 1; l >= 0; --l)
    for (int sg = 0; sg < 2; ++sg) {
      const int n = sg == 0 ? l : -l;
      if (sg == 1 && (l == 0 || real)) continue;
      for (int i = 0; i <= l; ++i) v.push_back(make_int2(n, i));
    }
  *count = (int)v.size();
  auto it = c->aux.find(key);
  if (it != c->aux.end()) {
    *out = (const int2*)it->second;
    return SCV_OK;
  }
  void* d = nullptr;
  SCV_CUDA(c, cudaMalloc(&d, v.size() * sizeof(int2)));
  SCV_CUDA(c, cudaMemcpy(d, v.data(), v.size() * sizeof(int2), cudaMemcpyHostToDevice));
  c->aux[key] = d;
  *out = (const int2*)d;
  return SCV_OK;
}

template <int L>
static int run_beta_pfa(scv_ctx* c, int real, const double2* W1p, double2* w, double pref, const BetaTables* t,
                        cudaStream_t s) {
  constexpr int K = 2 * L - 1, K2 = 4 * L - 1;
  const double2 *tab1, *tab2;
  SCV_TRY(scv_pfa_tables(c, K, &tab1));
  SCV_TRY(scv_pfa_tables(c, K2, &tab2));
  const int2* tasks;
  int nt;
  SCV_TRY(beta_pfa_tasks(c, L, real, &tasks, &nt));
  // chunk scratch: F and E (K each) + gamma per task, in scratch slot 1 (free after the alpha/gamma passes)
  const size_t per_task = (size_t)(2 * K + 1) * sizeof(double2);
  size_t want = std::max<size_t>(per_task * 1024, (size_t)1 << 30);
  void* scr = nullptr;
  SCV_TRY(scv_scratch(c, 1, std::min(want, per_task * (size_t)nt), &scr));
  const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)nt, c->scratch_bytes[1] / per_task));
  double2* Fb = (double2*)scr;
  double2* Eb = Fb + (size_t)chunk * K;
  double2* gb = Eb + (size_t)chunk * K;
  const size_t smf = pfa_smem<K, false>(), sme = pfa_smem<K2, false>();
  for (int t0 = 0; t0 < nt; t0 += chunk) {
    const int ntask = std::min(chunk, nt - t0);
    int grid;
    SCV_TRY(persistent_grid(c, k_beta_f<K>, PfaCfg<K, false>::NT, smf, (ntask + PfaCfg<K, false>::R - 1) / PfaCfg<K, false>::R, &grid));
    k_beta_f<K><<<grid, PfaCfg<K, false>::NT, smf, s>>>(real, W1p, tasks, t0, ntask, t->phs, Fb, gb, tab1);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
    SCV_TRY(persistent_grid(c, k_beta_e<K2>, PfaCfg<K2, false>::NT, sme, (ntask + PfaCfg<K2, false>::R - 1) / PfaCfg<K2, false>::R, &grid));
    k_beta_e<K2><<<grid, PfaCfg<K2, false>::NT, sme, s>>>(ntask, Fb, gb, t->wfpos, Eb, tab2);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
    k_beta_c<L><<<(ntask * 32 + 255) / 256, 256, 0, s>>>(real, tasks, t0, ntask, Fb, Eb, gb, t->Aalt, c->delta,
                                                          pref, w);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
  }
  return SCV_OK;
}

int scv_pfa_beta_so3(scv_ctx* c, int L, int real, const double2* W1p, double2* w, double pref,
                     const BetaTables* t, cudaStream_t s) {
  switch (L) {
    case 128: return run_beta_pfa<128>(c, real, W1p, w, pref, t, s);
    case 256: return run_beta_pfa<256>(c, real, W1p, w, pref, t, s);
    case 512: return run_beta_pfa<512>(c, real, W1p, w, pref, t, s);
    case 1024: return run_beta_pfa<1024>(c, real, W1p, w, pref, t, s);
    default: return scv_fail(c, SCV_EINVAL, "no prime-factor beta stage for L=" + std::to_string(L));
  }
}

#define PFA_SWITCH(K, CALL)                                                                 \
  switch (K) {                                                                              \
    case 3: return CALL(3); case 7: return CALL(7); case 15: return CALL(15);              \
    case 31: return CALL(31); case 63: return CALL(63);                                     \
    case 255: return CALL(255); case 511: return CALL(511); case 1023: return CALL(1023);   \
    case 2047: return CALL(2047); case 4095: return CALL(4095);                             \
    default: return scv_fail(c, SCV_EINVAL, "no prime-factor plan for length " + std::to_string(K)); \
  }

template <int K, int DIR>
static int run_rows(scv_ctx* c, long long nrows, const double2* in, double2* out, cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  const size_t sm = pfa_smem<K, false>();
  int grid;
  const long long nb = (nrows + PfaCfg<K, false>::R - 1) / PfaCfg<K, false>::R;
  SCV_TRY(persistent_grid(c, k_pfa_rows<K, DIR>, PfaCfg<K, false>::NT, sm, nb, &grid));
  k_pfa_rows<K, DIR><<<grid, PfaCfg<K, false>::NT, sm, s>>>(nrows, in, out, tab);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

template <int K>
static int run_ana_alpha(scv_ctx* c, int real, const double2* w, const double* hlb, const double* ls,
                         const double* lc, double2* out, cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  const size_t sm = pfa_smem<K, false>();
  constexpr int L = (K + 1) / 2;
  const long long nb = ((long long)(real ? L : K) * L + PfaCfg<K, false>::R - 1) / PfaCfg<K, false>::R;
  int grid;
  SCV_TRY(persistent_grid(c, k_ana_alpha<K>, PfaCfg<K, false>::NT, sm, nb, &grid));
  k_ana_alpha<K><<<grid, PfaCfg<K, false>::NT, sm, s>>>(real, w, hlb, ls, lc, out, tab);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

template <int K>
static int run_ana_gamma(scv_ctx* c, int real, double2* src, double* dst, cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  const size_t sm = pfa_smem<K, true>();
  constexpr int L = (K + 1) / 2;
  const int cpb = real ? 2 * PfaCfg<K, true>::R : PfaCfg<K, true>::R;
  const long long nb = (long long)L * ((K + cpb - 1) / cpb);
  int grid;
  SCV_TRY(persistent_grid(c, k_ana_gamma<K>, PfaCfg<K, true>::NT, sm, nb, &grid));
  k_ana_gamma<K><<<grid, PfaCfg<K, true>::NT, sm, s>>>(real, src, dst, tab);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

template <int K>
static int run_syn_alpha(scv_ctx* c, int real, const void* in, int b0, int nbb, double2* chunk, cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  const size_t sm = pfa_smem<K, false>();
  const int rpb = real ? 2 * PfaCfg<K, false>::R : PfaCfg<K, false>::R;
  const long long nb = ((long long)K * nbb + rpb - 1) / rpb;
  int grid;
  SCV_TRY(persistent_grid(c, k_syn_alpha<K>, PfaCfg<K, false>::NT, sm, nb, &grid));
  k_syn_alpha<K><<<grid, PfaCfg<K, false>::NT, sm, s>>>(real, in, b0, nbb, chunk, tab);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

template <int K>
static int run_syn_gamma(scv_ctx* c, int real, const double2* chunk, int b0, int nbb, double2* W1p, cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  const size_t sm = pfa_smem<K, true>();
  const long long nb = (long long)nbb * ((K + PfaCfg<K, true>::R - 1) / PfaCfg<K, true>::R);
  int grid;
  SCV_TRY(persistent_grid(c, k_syn_gamma<K>, PfaCfg<K, true>::NT, sm, nb, &grid));
  k_syn_gamma<K><<<grid, PfaCfg<K, true>::NT, sm, s>>>(real, chunk, b0, nbb, W1p, tab);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

int scv_pfa_ana_alpha(scv_ctx* c, int K, int real, const double2* w, const double* hlb, const double* ls,
                      const double* lc, double2* out, cudaStream_t s) {
#define CALL(KK) run_ana_alpha<KK>(c, real, w, hlb, ls, lc, out, s)
  PFA_SWITCH(K, CALL)
#undef CALL
}
int scv_pfa_ana_gamma(scv_ctx* c, int K, int real, double2* src, double* dst, cudaStream_t s) {
#define CALL(KK) run_ana_gamma<KK>(c, real, src, dst, s)
  PFA_SWITCH(K, CALL)
#undef CALL
}
int scv_pfa_syn_alpha(scv_ctx* c, int K, int real, const void* in, int b0, int nbb, double2* chunk,
                      cudaStream_t s) {
#define CALL(KK) run_syn_alpha<KK>(c, real, in, b0, nbb, chunk, s)
  PFA_SWITCH(K, CALL)
#undef CALL
}
int scv_pfa_syn_gamma(scv_ctx* c, int K, int real, const double2* chunk, int b0, int nbb, double2* W1p,
                      cudaStream_t s) {
#define CALL(KK) run_syn_gamma<KK>(c, real, chunk, b0, nbb, W1p, s)
  PFA_SWITCH(K, CALL)
#undef CALL
}

extern "C" int scv_debug_dft(scv_ctx* c, int K, int dir, int nrows, const double* in, double* out,
                             void* stream) {
  if (!c) return SCV_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "debug_dft");
  if (dir < 0) {
#define CALL(KK) run_rows<KK, -1>(c, nrows, (const double2*)in, (double2*)out, s)
    PFA_SWITCH(K, CALL)
#undef CALL
  }
#define CALL(KK) run_rows<KK, +1>(c, nrows, (const double2*)in, (double2*)out, s)
  PFA_SWITCH(K, CALL)
#undef CALL
}
