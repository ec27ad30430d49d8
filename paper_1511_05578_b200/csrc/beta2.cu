// SO(3) forward beta stage + Delta contraction on the register-resident
// power-of-two FFT (fft_reg.cuh).  Same linear map as beta.cu / the reference
// (so3.py:203-243, fourier.py:41-119); differences are in the data flow only:
//
//  * centred Bluestein: the K extended samples are indexed b' = b-(L-1) in
//    [-(L-1), L-1] and stored wrapped mod P, so the chirp filter h'[j],
//    |j| <= 2L-2, is even and its spectrum (P/2+1 entries) plus the pre/post
//    chirp exp(-i pi b'^2/K) (L entries) are the only Bluestein tables; the
//    post-chirp with the offset phase is (1/K)(-1)^{m''} exp(-i pi m''^2/K);
//  * the Bluestein output F lands at positions m'' mod P, which is exactly
//    where the (wrapped, even, real-spectrum) weight convolution wants G, so
//    DFT -> filter -> IDFT -> post-chirp -> DFT -> filter -> IDFT runs on
//    registers with no relayout between the four transforms;
//  * all tables (~72 KB at L=1024) live in shared memory for the lifetime of
//    a persistent block and are read once per element per column pair.
// Packing of two opposite-parity columns per transform: see beta.cu.

#include <algorithm>

#include "fft_reg.cuh"
#include "scv_internal.cuh"

namespace {

#ifndef SCV_B2_E
#define SCV_B2_E 8
#endif
template <int LOGP>
struct B2Cfg {
  static constexpr int P = 1 << LOGP;
  static constexpr int E = (LOGP >= 12 || SCV_B2_E < 16) ? SCV_B2_E : 8;
  static constexpr int NT = P / E;
#ifdef SCV_B2_MINB
  static constexpr int MINB = SCV_B2_MINB;
#else
  static constexpr int MINB = NT >= 512 ? 1 : 2;
#endif
};

__device__ __forceinline__ long long colbase(int n, int real) {
  const long long l = n < 0 ? -n : n;
  if (real) return l * l;
  if (l == 0) return 0;
  return n > 0 ? 2 * l * l - 1 : 2 * l * l + 2 * l;
}

template <int LOGP>
__global__ void __launch_bounds__(B2Cfg<LOGP>::NT, B2Cfg<LOGP>::MINB)
    k_beta2(int L, int real, const double2* __restrict__ W1p, double2* __restrict__ wout,
            const double2* __restrict__ g_a2, const double2* __restrict__ g_hf2, const double* __restrict__ g_vf2,
            const double* __restrict__ g_aalt, const double2* __restrict__ tw, const double* __restrict__ delta,
            double pref, const int2* __restrict__ tasks, int ntasks) {
  constexpr int P = 1 << LOGP, E = B2Cfg<LOGP>::E, NT = B2Cfg<LOGP>::NT;
  const int K = 2 * L - 1;
  extern __shared__ double2 sm[];
  double2* ex = sm;                                  // padded exchange buffer, later E (unpadded)
  double2* Fs = ex + regfft::padded_size(P);         // F[m''] at m''+L-1
  double2* A2 = Fs + K;                              // L
  double2* gsh = A2 + L;                             // 1 (gamma of the odd column)
  double2* HF = gsh + 1;                             // P/2+1
  double* VF = (double*)(HF + P / 2 + 1);            // P/2+1
  double* AL = VF + P / 2 + 1;                       // Aalt[m'] for m' = 0..L-1 (even)
  double* red = AL + L;                              // 4 * NT/32
  const int t = threadIdx.x;
  for (int i = t; i < L; i += NT) {
    A2[i] = g_a2[i];
    AL[i] = g_aalt[i + L - 1];
  }
  for (int i = t; i <= P / 2; i += NT) {
    HF[i] = g_hf2[i];
    VF[i] = g_vf2[i];
  }
  __syncthreads();
  const double invK = 1.0 / (double)K;
#pragma unroll 1
  for (int task = blockIdx.x; task < ntasks; task += gridDim.x) {
    // opaque per-iteration copy of the thread index: keeps the compiler from
    // hoisting every table / exchange address of the 4 FFTs out of the loop
    int t = threadIdx.x;
    asm volatile("" : "+r"(t));
    const int2 tk = tasks[task];
    const int n = tk.x, l = n < 0 ? -n : n;
    const int m0 = -l + 2 * tk.y, m1 = m0 + 1;
    const bool has1 = m1 <= l;
    const bool even0 = ((n + m0) & 1) == 0;
    const long long cb = colbase(n, real);
    const double2* c0 = W1p + (cb + m0 + l) * (long long)L;
    const double2* c1 = has1 ? W1p + (cb + m1 + l) * (long long)L : nullptr;
    const double2* colE = even0 ? c0 : c1;
    const double2* colO = even0 ? c1 : c0;
    // 1. centred, packed, pre-chirped input at positions b' mod P
    double2 x[E];
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k = t + s * NT;
      const int bp = k <= L - 1 ? k : k - P;  // b'
      double2 u = make_double2(0.0, 0.0);
      if (bp >= -(L - 1) && bp <= L - 1) {
        const int b = bp + L - 1;
        const int src = b < L ? b : 2 * L - 2 - b;
        double2 e = colE ? colE[src] : make_double2(0.0, 0.0);
        if (colO) {
          const double2 o = colO[src];
          if (b >= L) e = make_double2(e.x - o.x, e.y - o.y);
          else e = make_double2(e.x + o.x, e.y + o.y);
          if (b == L - 1) *gsh = make_double2(o.x * (2.0 * invK), o.y * (2.0 * invK));
        } else if (b == L - 1) {
          *gsh = make_double2(0.0, 0.0);
        }
        u = cmul(e, A2[bp < 0 ? -bp : bp]);
      }
      x[s] = u;
    }
    regfft::fft<LOGP, E, -1>(x, ex, tw, t);
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k = t + s * NT;
      x[s] = cmul(x[s], HF[k <= P / 2 ? k : P - k]);
    }
    __syncthreads();  // ex reuse + gsh visibility
    regfft::fft<LOGP, E, +1>(x, ex, tw, t);
    const double2 g = *gsh;
    // 2. F = (1/K)(-1)^{m''} A2[|m''|] c ; G = F - (gamma/2)(-1)^{m''} at the same positions
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k = t + s * NT;
      const int mpp = k <= L - 1 ? k : k - P;
      double2 v = make_double2(0.0, 0.0);
      if (mpp >= -(L - 1) && mpp <= L - 1) {
        const double sg = (mpp & 1) ? -invK : invK;
        double2 F = cmul(x[s], A2[mpp < 0 ? -mpp : mpp]);
        F = make_double2(F.x * sg, F.y * sg);
        Fs[mpp + L - 1] = F;
        const double hh = (mpp & 1) ? -0.5 : 0.5;
        v = make_double2(F.x - hh * g.x, F.y - hh * g.y);
      }
      x[s] = v;
    }
    __syncthreads();
    regfft::fft<LOGP, E, -1>(x, ex, tw, t);
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k = t + s * NT;
      const double f = VF[k <= P / 2 ? k : P - k];
      x[s] = make_double2(x[s].x * f, x[s].y * f);
    }
    __syncthreads();
    regfft::fft<LOGP, E, +1>(x, ex, tw, t);
    // 3. E[m'] for |m'| <= L-1 into ex (unpadded, index m' mod P)
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k = t + s * NT;
      if (k <= L - 1 || k >= P - (L - 1)) ex[k] = x[s];
    }
    __syncthreads();
    // 4. Y_E / Y_O and the Delta contraction
    const int mE = even0 ? m0 : m1, mO = even0 ? m1 : m0;
    const double hp = 0.5 * SCV_PI;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int mp = -l + t; mp <= l; mp += NT) {
      const double2 Ep = ex[mp >= 0 ? mp : mp + P], Em = ex[mp <= 0 ? -mp : P - mp];
      const double2 ee = make_double2(0.5 * (Ep.x + Em.x), 0.5 * (Ep.y + Em.y));
      const double2 eo = make_double2(0.5 * (Ep.x - Em.x), 0.5 * (Ep.y - Em.y));
      double2 xe[2], xo[2];
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int kk = z == 0 ? mp + 1 : mp - 1;
        if (kk < -(L - 1) || kk > L - 1) {
          xe[z] = make_double2(0.0, 0.0);
          xo[z] = make_double2(0.0, 0.0);
        } else {
          const double2 a = Fs[kk + L - 1], b = Fs[-kk + L - 1];
          const double h2 = (kk & 1) ? -1.0 : 1.0;
          xe[z] = make_double2(0.5 * (a.x + b.x - h2 * g.x), 0.5 * (a.y + b.y - h2 * g.y));
          xo[z] = make_double2(0.5 * (a.x - b.x + h2 * g.x), 0.5 * (a.y - b.y + h2 * g.y));
        }
      }
      const double2 dE = make_double2(xe[0].x - xe[1].x, xe[0].y - xe[1].y);
      const double2 dO = make_double2(xo[0].x - xo[1].x, xo[0].y - xo[1].y);
      const double2 yE = make_double2(ee.x - hp * dE.y, ee.y + hp * dE.x);
      const double aa = 0.5 * AL[mp < 0 ? -mp : mp];
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
    if ((t & 31) == 0)
#pragma unroll
      for (int i = 0; i < 4; ++i) red[(t >> 5) * 4 + i] = acc[i];
    __syncthreads();
    if (t == 0) {
      double tot[4] = {0.0, 0.0, 0.0, 0.0};
      for (int wv = 0; wv < NT / 32; ++wv)
        for (int i = 0; i < 4; ++i) tot[i] += red[wv * 4 + i];
      const int c = L - 1;
      double2* row = wout + ((long long)(n >= 0 ? 0 : 1) * L + l) * K;
      const int ms[2] = {mE, mO};
      for (int i = 0; i < 2; ++i) {
        const int m = ms[i];
        if (m > l) continue;
        const double2 v = cipow(make_double2(pref * tot[2 * i], pref * tot[2 * i + 1]), m - n);
        row[c + m] = v;
        if (real && n > 0) {  // row(-n)[m] = (-1)^{m+n} conj(row(n)[-m])  (so3.py:379-382)
          double2 cv = make_double2(v.x, -v.y);
          if ((m + n) & 1) cv = make_double2(-cv.x, -cv.y);
          wout[((long long)1 * L + l) * K + c - m] = cv;
        }
      }
    }
    __syncthreads();
  }
}

template <int LOGP>
size_t b2_smem(int L) {
  constexpr int P = 1 << LOGP, NT = B2Cfg<LOGP>::NT;
  const int K = 2 * L - 1;
  return (size_t)(regfft::padded_size(P) + K + L + P / 2 + 1) * sizeof(double2) +
         (size_t)(P / 2 + 1 + L + 4 * (NT / 32) + 2) * sizeof(double) + 2 * sizeof(double2);
}

template <int LOGP>
int launch_b2(scv_ctx* c, int L, int real, const double2* W1p, double2* w, double pref, const BetaTables* t,
              const int2* tasks, int ntasks, cudaStream_t s) {
  const size_t sm = b2_smem<LOGP>(L);
  auto kern = k_beta2<LOGP>;
  SCV_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per = 0, sms = 0;
  SCV_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, B2Cfg<LOGP>::NT, sm));
  SCV_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  const int grid = std::max(1, std::min(ntasks, std::max(per, 1) * sms));
  kern<<<grid, B2Cfg<LOGP>::NT, sm, s>>>(L, real, W1p, w, t->a2, t->hf2, t->vf2, t->Aalt, t->tw, c->delta, pref,
                                         tasks, ntasks);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

}  // namespace

bool scv_beta2_supported(int L) {
  int lg = next_pow2_log(4 * L - 3);
  return lg >= 8 && lg <= 12;  // P = 256 .. 4096
}

int scv_beta2_so3(scv_ctx* c, int L, int real, const double2* W1p, double2* w, double pref,
                  const BetaTables* t, const int2* tasks, int ntasks, cudaStream_t s) {
  switch (t->logP) {
    case 8: return launch_b2<8>(c, L, real, W1p, w, pref, t, tasks, ntasks, s);
    case 9: return launch_b2<9>(c, L, real, W1p, w, pref, t, tasks, ntasks, s);
    case 10: return launch_b2<10>(c, L, real, W1p, w, pref, t, tasks, ntasks, s);
    case 11: return launch_b2<11>(c, L, real, W1p, w, pref, t, tasks, ntasks, s);
    case 12: return launch_b2<12>(c, L, real, W1p, w, pref, t, tasks, ntasks, s);
    default: return scv_fail(c, SCV_EINVAL, "beta2: unsupported transform size");
  }
}
