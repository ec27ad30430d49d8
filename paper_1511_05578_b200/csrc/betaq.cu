// beta quadrature table of the SO(3) forward transform (synthesis direction).
//
// For a curvelet column (n, m), |m| <= l = |n|, the reference's beta stage
// (so3.py:203-243: parity extension, K-point DFT / K, phase e^{-i m'' pi/K},
// 4 pi^2 * weights convolution, Delta contraction with i^{m-n}) is a LINEAR
// functional of the column's L beta samples.  Written out:
//
//   W_{mn} = sum_b S(b) q_{nm}(b),
//   q_ext(b) = i^{m-n} (pref/K) sum_{|m''|<=L-1} U(m'') e^{-i m'' beta_b},
//   U(m'')  = sum_{|m'|<=l} w(m''-m') c(m'),   c(m') = D^l_{m'm} D^l_{m'n},
//   q(b)    = q_ext(b) + (-1)^{n+m} q_ext(2L-2-b)  (b <= L-2),  q(L-1) = q_ext(L-1),
//
// with beta_b = pi(2b+1)/K and pref = 4 pi^2 / K^2 (the alpha/gamma DFT
// normalisation folded in).  c(-m') = (-1)^{n+m} c(m'), so with U = U_e + U_o
// (even taps 2/(1-k^2), odd taps +-i pi/2):
//   b <= L-2:  q = 2 i^{m-n} (pref/K) sum U_e(m'') e^{-i m'' beta_b}
//              (the odd taps cancel between b and its reflection), which is
//              a cosine (n+m even) or sine (n+m odd) transform of U_e, real;
//   b = L-1:   q = i^{m-n} (pref/K) sum (U_e + U_o)(m'') (-1)^{m''}, real.
// The table depends on L only (like the Delta table), is built once per
// context, and replaces the per-map beta FFTs and the Delta contraction by one
// multiply-accumulate per (n, m, b) fused into the gamma pass (pfa.cu,
// k_syn_gamma_q).  Checked against the reference pipeline by
// tests/test_formulation.py (unit-vector probes) and on the GPU against the
// FFT beta stage (tests/test_gpu_parity.py).
//
// Storage (n = +l only; q_{-l,m} = (-1)^{l+m} q_{l,-m}):
//   q[mbase(m) + b * (L-|m|) + (l-|m|)],  m in [-(L-1), L-1], b < L, |m| <= l < L,
//   mbase(m) = L * sum_{j < m} (L - |j|)        -> L^3 doubles (8.6 GB at L=1024).

#include <algorithm>
#include <cmath>
#include <vector>

#include "scv_internal.cuh"

namespace {

typedef long double ld;
constexpr int QG_MAX = 8;   // consecutive degrees per task (coalesced 64-byte stores)
constexpr int QNT = 256;    // threads per block

__global__ void __launch_bounds__(QNT) k_betaq_build(int L, int QG, double pref, const double* __restrict__ delta,
                                                     const double* __restrict__ trig, const long long* __restrict__ mbase,
                                                     const int2* __restrict__ tasks, int ntasks, double* __restrict__ q) {
  const int K = 2 * L - 1;
  extern __shared__ double smq[];
  double* cosT = smq;                  // 2K
  double* sinT = cosT + 2 * K;         // 2K
  double* cb = sinT + 2 * K;           // 2L+2 : c(m') at m'+L, zero outside [-l, l]
  double* ue = cb + 2 * L + 2;         // L    : U_e(m''), m'' >= 0
  double* qg = ue + L;                 // QG * L
  double* red = qg + QG * L;           // 32
  const int t = threadIdx.x;
  for (int i = t; i < 2 * K; i += QNT) {
    cosT[i] = trig[2 * i];
    sinT[i] = trig[2 * i + 1];
  }
  __syncthreads();
  for (int task = blockIdx.x; task < ntasks; task += gridDim.x) {
    const int m = tasks[task].x, l0 = tasks[task].y;
    const int am = m < 0 ? -m : m;
    const int nl = min(QG, L - l0);
    for (int li = 0; li < nl; ++li) {
      const int l = l0 + li;
      const bool even = ((l + m) & 1) == 0;  // parity (-1)^{n+m}, n = l
      for (int i = t; i < 2 * L + 2; i += QNT) {
        const int mp = i - L;
        cb[i] = (mp >= -l && mp <= l) ? wedge_get(delta, l, mp, m) * wedge_get(delta, l, mp, l) : 0.0;
      }
      __syncthreads();
      // U_e(m'') = sum over m' == m'' (mod 2) of c(m') 2/(1-(m''-m')^2)
      for (int mpp = t; mpp < L; mpp += QNT) {
        double acc = 0.0;
        int mp = -l + (((mpp + l) & 1) ? 1 : 0);
        for (; mp <= l; mp += 2) {
          const double d = (double)(mpp - mp);
          acc += cb[mp + L] * (2.0 / (1.0 - d * d));
        }
        ue[mpp] = acc;
      }
      __syncthreads();
      // b = L-1: sum_{m''} (U_e + U_o)(m'') (-1)^{m''}; U_e(-m'') = par U_e(m''),
      // U_o(m'') = (i pi/2)(c(m''-1) - c(m''+1))
      double se = 0.0, so = 0.0;
      for (int mpp = -(L - 1) + t; mpp <= L - 1; mpp += QNT) {
        const double sg = (mpp & 1) ? -1.0 : 1.0;
        const int a = mpp < 0 ? -mpp : mpp;
        const double u = (mpp < 0 && !even) ? -ue[a] : ue[a];
        se += sg * u;
        so += sg * (cb[mpp - 1 + L] - cb[mpp + 1 + L]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        se += __shfl_xor_sync(0xffffffffu, se, o);
        so += __shfl_xor_sync(0xffffffffu, so, o);
      }
      if ((t & 31) == 0) {
        red[(t >> 5) * 2] = se;
        red[(t >> 5) * 2 + 1] = so;
      }
      // q(b), b <= L-2: 2 i^{m-n} (pref/K) sum_{m''} U_e(m'') e^{-i m'' beta_b}
      const double f = pref / (double)K;
      const int mn = m - l;  // m - n
      for (int b = t; b < L - 1; b += QNT) {
        const int step = 2 * b + 1;
        int j = 0;
        double acc = 0.0;
        if (even) {
          for (int mpp = 1; mpp < L; ++mpp) {
            j += step;
            if (j >= 2 * K) j -= 2 * K;
            acc += ue[mpp] * cosT[j];
          }
          acc = ue[0] + 2.0 * acc;
          // i^{m-n}, m-n even
          qg[li * L + b] = 2.0 * f * ((mn / 2) & 1 ? -acc : acc);
        } else {
          for (int mpp = 1; mpp < L; ++mpp) {
            j += step;
            if (j >= 2 * K) j -= 2 * K;
            acc += ue[mpp] * sinT[j];
          }
          // 2 i^{m-n} (-2i) acc = 4 i^{m-n-1} acc, m-n odd
          const int e = (mn - 1) / 2;
          qg[li * L + b] = 4.0 * f * ((e & 1) ? -acc : acc);
        }
      }
      __syncthreads();
      if (t == 0) {
        double te = 0.0, to = 0.0;
        for (int w = 0; w < QNT / 32; ++w) {
          te += red[2 * w];
          to += red[2 * w + 1];
        }
        // i^{m-n} (pref/K) (te + (i pi/2) to): even -> i^{m-n} real; odd -> i^{m-n+1} (pi/2) to
        double v;
        if (even) v = ((mn / 2) & 1) ? -te : te;
        else {
          const int e = (mn + 1) / 2;
          v = 0.5 * SCV_PI * (((e % 2) + 2) % 2 ? -to : to);
        }
        qg[li * L + L - 1] = f * v;
      }
      __syncthreads();
    }
    // store: q[mbase(m) + b*(L-|m|) + (l-|m|)]
    const long long base = mbase[m + L - 1];
    const int row = L - am;
    for (int i = t; i < nl * L; i += QNT) {
      const int b = i / nl, li = i - b * nl;
      q[base + (long long)b * row + (l0 + li - am)] = qg[li * L + b];
    }
    __syncthreads();
  }
}

}  // namespace

bool scv_betaq_enabled(int L) {
  static const char* e = getenv("SCV_BETAQ");
  if (e && e[0] == '0') return false;
  return L >= 2;
}

// Build (once per context and L) the beta quadrature table and the per-m bases.
int scv_betaq_table(scv_ctx* c, int L, cudaStream_t s, const double** qtab, const long long** mbase) {
  const std::string key = "betaq_" + std::to_string(L);
  const std::string kb = "betaqb_" + std::to_string(L);
  auto it = c->aux.find(key);
  if (it != c->aux.end()) {
    *qtab = (const double*)it->second;
    *mbase = (const long long*)c->aux[kb];
    return SCV_OK;
  }
  SCV_TRY(scv_ensure_delta(c, L, s));
  const int K = 2 * L - 1;
  std::vector<long long> mb(2 * L - 1);
  long long acc = 0;
  for (int m = -(L - 1); m <= L - 1; ++m) {
    mb[m + L - 1] = acc;
    acc += (long long)L * (L - std::abs(m));
  }
  // degrees per task: as many as fit next to the trig tables in shared memory
  // (8 up to L = 1024, fewer at L = 2048)
  const size_t fixed = (size_t)4 * K + 2 * L + 2 + L + 32;
  const int QG = (int)std::max<long long>(1, std::min<long long>(QG_MAX, ((long long)(232448 / sizeof(double)) - (long long)fixed) / L));
  std::vector<int2> tasks;
  for (int m = -(L - 1); m <= L - 1; ++m)
    for (int l0 = std::abs(m); l0 < L; l0 += QG) tasks.push_back(make_int2(m, l0));
  const ld pi = 3.141592653589793238462643383279502884L;
  std::vector<double> trig(4 * (size_t)K);
  for (int j = 0; j < 2 * K; ++j) {
    trig[2 * j] = (double)cosl(pi * (ld)j / (ld)K);
    trig[2 * j + 1] = (double)sinl(pi * (ld)j / (ld)K);
  }
  double* dq = nullptr;
  long long* dmb = nullptr;
  void *dtrig = nullptr, *dtask = nullptr;
  SCV_CUDA(c, cudaMalloc(&dq, (size_t)acc * sizeof(double)));
  SCV_CUDA(c, cudaMalloc(&dmb, mb.size() * sizeof(long long)));
  SCV_CUDA(c, cudaMalloc(&dtrig, trig.size() * sizeof(double)));
  SCV_CUDA(c, cudaMalloc(&dtask, tasks.size() * sizeof(int2)));
  SCV_CUDA(c, cudaMemcpyAsync(dmb, mb.data(), mb.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  SCV_CUDA(c, cudaMemcpyAsync(dtrig, trig.data(), trig.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  SCV_CUDA(c, cudaMemcpyAsync(dtask, tasks.data(), tasks.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
  const size_t sm = (fixed + (size_t)QG * L) * sizeof(double);
  SCV_CUDA(c, cudaFuncSetAttribute(k_betaq_build, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per = 0, sms = 0;
  SCV_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_betaq_build, QNT, sm));
  SCV_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  const int grid = std::max(1, std::min((int)tasks.size(), std::max(per, 1) * sms));
  const double pref = 4.0 * SCV_PI * SCV_PI / ((double)K * (double)K);
  {
    SCV_PROF(c, s, "betaq_build");
    k_betaq_build<<<grid, QNT, sm, s>>>(L, QG, pref, c->delta, (const double*)dtrig, dmb, (const int2*)dtask,
                                        (int)tasks.size(), dq);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
  }
  SCV_CUDA(c, cudaStreamSynchronize(s));
  cudaFree(dtrig);
  cudaFree(dtask);
  c->aux[key] = dq;
  c->aux[kb] = dmb;
  c->table_bytes += (long long)acc * (long long)sizeof(double) + (long long)mb.size() * (long long)sizeof(long long);
  *qtab = dq;
  *mbase = dmb;
  return SCV_OK;
}
