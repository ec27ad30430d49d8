// The beta (colatitude) stage of the forward transforms, hand-written.
//
// Reference (per column of beta samples s[b], b<L, with parity p):
//   extend to K=2L-1 nodes, node b>=L = p*s[2L-2-b]          fourier.py:41-55
//   X[m''] = fftshift(fft(ext)/K) * exp(-i m'' pi/K)          so3.py:203-209, sphere.py:166-169
//   Y[m']  = pref * sum_m'' X[m''] w(m''-m')                  fourier.py:84-119
// then the Delta contraction
//   SO(3):  W_{m,n} = i^{m-n} sum_m' D^l_{m'm} D^l_{m'n} Y[m']  (l=|n|)  so3.py:236-243
//   SHT:    done by k_sht_contract in sht.cu                     sphere.py:171-181
//
// B200 formulation (same linear map, fewer FP64 flops):
//  * The K-point DFT at the offset nodes is a Bluestein chirp-z transform
//    built from two P-point power-of-two FFTs (P >= 4L-3) in shared memory.
//  * Two columns of opposite parity are packed into ONE transform.  With
//    the reflection b -> 2L-2-b, beta_b -> 2pi-beta_b, so an even column
//    has X[-k] = X[k] and an odd one X[-k] = -X[k] + gamma (-1)^k,
//    gamma = (2/K) s[L-1] (the beta=pi node is not reflected).  From
//    F = X_E + X_O both come back exactly:
//        X_E[k] = (F[k] + F[-k] - gamma(-1)^k)/2,  X_O[k] = (F[k] - F[-k] + gamma(-1)^k)/2.
//  * w(k) splits into a real even part (even k: 2/(1-k^2)) and the two odd
//    taps w(+-1) = +-i pi/2.  The even part preserves parity, so ONE padded
//    convolution of G = F - (gamma/2)(-1)^k serves both columns:
//        W_e X_E = even part of W_e G,  W_e X_O = odd part + (gamma/2) A_alt,
//    with A_alt = W_e (-1)^k tabulated; the odd taps are two-term
//    differences.  Net: 4 P-point FFTs per PAIR of columns instead of
//    3-4 per column.

#include <cstdlib>

#include "fft_smem.cuh"
#include "scv_internal.cuh"

struct BetaDev {
  const double2* tw;
  const double2* A;
  const double2* Hf;
  const double2* C;
  const double2* Vf;
  const double* Aalt;
};

static BetaDev dev_of(const BetaTables* t) {
  return BetaDev{t->tw, t->chirpA, t->Hf, t->chirpC, t->Vf, t->Aalt};
}

// Steps common to both epilogues.  On exit:
//   xs[q] = F[q-(L-1)], q in [0,K)      (packed DFT, no pref)
//   buf[3L-3+m'] = (W_e G)[m']          for |m'| <= L-1
//   *gam = gamma of the odd column
// colE/colO: global pointers to the even/odd columns' L samples (nullptr = zero column),
// with element stride `cs`.
template <int LOGP, int NT>
__device__ void beta_pair_core(int L, const double2* __restrict__ colE, const double2* __restrict__ colO,
                               long long cs, const BetaDev& T, double2* buf, double2* xs,
                               double2* gam_sh) {
  constexpr int P = 1 << LOGP;
  const int K = 2 * L - 1;
  const int tid = threadIdx.x;
  // 1. packed, extended, chirped input
  for (int b = tid; b < P; b += NT) {
    double2 u = make_double2(0.0, 0.0);
    if (b < K) {
      double2 e = make_double2(0.0, 0.0), o = make_double2(0.0, 0.0);
      const int src = (b < L) ? b : (2 * L - 2 - b);
      if (colE) e = colE[src * cs];
      if (colO) {
        o = colO[src * cs];
        if (b >= L) o = make_double2(-o.x, -o.y);
      }
      u = cmul(cadd(e, o), __ldg(T.A + b));
    }
    buf[b] = u;
  }
  if (tid == 0) {
    double2 g = make_double2(0.0, 0.0);
    if (colO) g = cscale(colO[(L - 1) * cs], 2.0 / (double)K);
    *gam_sh = g;
  }
  __syncthreads();
  fft_smem<LOGP, NT, -1>(buf, T.tw);
  for (int k = tid; k < P; k += NT) buf[k] = cmul(buf[k], __ldg(T.Hf + k));
  __syncthreads();
  fft_smem<LOGP, NT, +1>(buf, T.tw);
  // 2. post-chirp -> F; then G = F - (gamma/2)(-1)^k into the padded buffer
  const double2 g = *gam_sh;
  double2 Fv[(P / 2 + NT - 1) / NT + 1];
  int cnt = 0;
  for (int q = tid; q < K; q += NT) {
    const int mpp = q - (L - 1);
    const double2 F = cmul(__ldg(T.C + q), buf[mpp & (P - 1)]);
    Fv[cnt++] = F;
  }
  __syncthreads();
  cnt = 0;
  for (int q = tid; q < P; q += NT) {
    if (q < K) {
      const double2 F = Fv[cnt++];
      xs[q] = F;
      const int mpp = q - (L - 1);
      const double h = (mpp & 1) ? -0.5 : 0.5;
      buf[q] = make_double2(F.x - h * g.x, F.y - h * g.y);
    } else {
      buf[q] = make_double2(0.0, 0.0);
    }
  }
  __syncthreads();
  fft_smem<LOGP, NT, -1>(buf, T.tw);
  for (int k = tid; k < P; k += NT) buf[k] = cmul(buf[k], __ldg(T.Vf + k));
  __syncthreads();
  fft_smem<LOGP, NT, +1>(buf, T.tw);
}

// X_E / X_O at integer bin k from the packed F (0 outside [-(L-1), L-1]).
__device__ __forceinline__ double2 x_even(const double2* xs, int L, int k, double2 g) {
  if (k < -(L - 1) || k > L - 1) return make_double2(0.0, 0.0);
  double2 a = xs[k + L - 1], b = xs[-k + L - 1];
  double h = (k & 1) ? -1.0 : 1.0;
  return make_double2(0.5 * (a.x + b.x - h * g.x), 0.5 * (a.y + b.y - h * g.y));
}
__device__ __forceinline__ double2 x_odd(const double2* xs, int L, int k, double2 g) {
  if (k < -(L - 1) || k > L - 1) return make_double2(0.0, 0.0);
  double2 a = xs[k + L - 1], b = xs[-k + L - 1];
  double h = (k & 1) ? -1.0 : 1.0;
  return make_double2(0.5 * (a.x - b.x + h * g.x), 0.5 * (a.y - b.y + h * g.y));
}

// Y_E[m'] and Y_O[m'] (without pref) from the core's outputs.
__device__ __forceinline__ void y_pair(const double2* buf, const double2* xs, const double* __restrict__ Aalt,
                                       int L, int mp, double2 g, double2* yE, double2* yO) {
  const double2 Ep = buf[3 * L - 3 + mp], Em = buf[3 * L - 3 - mp];
  double2 ee = make_double2(0.5 * (Ep.x + Em.x), 0.5 * (Ep.y + Em.y));
  double2 eo = make_double2(0.5 * (Ep.x - Em.x), 0.5 * (Ep.y - Em.y));
  const double hp = 0.5 * SCV_PI;
  double2 dE = csub(x_even(xs, L, mp + 1, g), x_even(xs, L, mp - 1, g));
  double2 dO = csub(x_odd(xs, L, mp + 1, g), x_odd(xs, L, mp - 1, g));
  // (i pi/2) * d
  *yE = make_double2(ee.x - hp * dE.y, ee.y + hp * dE.x);
  const double aa = 0.5 * __ldg(Aalt + mp + L - 1);
  *yO = make_double2(eo.x + aa * g.x - hp * dO.y, eo.y + aa * g.y + hp * dO.x);
}

template <int NT>
__device__ __forceinline__ void block_sum4(double v[4], double* red) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < 4; ++i) red[w * 4 + i] = v[i];
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double t = (lane < NT / 32) ? red[lane * 4 + i] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      v[i] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// SO(3) forward: one block per (n, column pair); W1p holds the pruned
// alpha/gamma spectrum, column (n, m) at W1p[col(n,m)*L + b].
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long so3_colbase(int n, int real) {
  const long long l = n < 0 ? -n : n;
  if (real) return l * l;
  if (l == 0) return 0;
  return n > 0 ? 2 * l * l - 1 : 2 * l * l + 2 * l;
}

template <int LOGP, int NT>
__global__ void __launch_bounds__(NT) k_beta_so3(int L, int real, const double2* __restrict__ W1p,
                                                 double2* __restrict__ wout, BetaDev T,
                                                 const double* __restrict__ delta, double pref,
                                                 const int2* __restrict__ tasks) {
  extern __shared__ double2 smem[];
  constexpr int P = 1 << LOGP;
  const int K = 2 * L - 1;
  double2* buf = smem;
  double2* xs = smem + P;
  double2* gsh = xs + K;
  double* red = (double*)(gsh + 1);
  const int2 task = tasks[blockIdx.x];
  const int n = task.x, l = n < 0 ? -n : n;
  const int m0 = -l + 2 * task.y, m1 = m0 + 1;
  const bool has1 = m1 <= l;
  const bool even0 = ((n + m0) & 1) == 0;
  const long long cb = so3_colbase(n, real);
  const double2* c0 = W1p + (cb + m0 + l) * (long long)L;
  const double2* c1 = has1 ? W1p + (cb + m1 + l) * (long long)L : nullptr;
  const double2* colE = even0 ? c0 : c1;
  const double2* colO = even0 ? c1 : c0;
  beta_pair_core<LOGP, NT>(L, colE, colO, 1, T, buf, xs, gsh);
  const double2 g = *gsh;
  const int mE = even0 ? m0 : m1, mO = even0 ? m1 : m0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int mp = -l + (int)threadIdx.x; mp <= l; mp += NT) {
    double2 yE, yO;
    y_pair(buf, xs, T.Aalt, L, mp, g, &yE, &yO);
    const double dn = wedge_get(delta, l, mp, n);
    const double dE = (mE <= l) ? wedge_get(delta, l, mp, mE) * dn : 0.0;
    const double dO = (mO <= l) ? wedge_get(delta, l, mp, mO) * dn : 0.0;
    acc[0] += dE * yE.x;
    acc[1] += dE * yE.y;
    acc[2] += dO * yO.x;
    acc[3] += dO * yO.y;
  }
  block_sum4<NT>(acc, red);
  if (threadIdx.x == 0) {
    const int c = L - 1;
    const int sheet = n >= 0 ? 0 : 1;
    double2* row = wout + ((long long)sheet * L + l) * K;
    const int ms[2] = {mE, mO};
    for (int i = 0; i < 2; ++i) {
      const int m = ms[i];
      if (m > l) continue;
      double2 v = cipow(make_double2(pref * acc[2 * i], pref * acc[2 * i + 1]), m - n);
      row[c + m] = v;
      if (real && n > 0) {  // row(-n)[m] = (-1)^{m+n} conj(row(n)[-m])  (so3.py:379-382)
        double2 cv = make_double2(v.x, -v.y);
        if ((m + n) & 1) cv = make_double2(-cv.x, -cv.y);
        wout[((long long)1 * L + l) * K + c - m] = cv;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// SHT forward beta stage: columns m of G (rows t<L), full Y written to Gw.
//   complex: G[t*K + (m mod K)], m in [-(L-1), L-1], parity (-1)^{m+s};
//            Gw[(m'+L-1)*K + m+L-1]
//   real:    G[t*L + m], m in [0, L-1], parity (-1)^m;  Gw[(m'+L-1)*L + m]
// one block per column pair (m0, m0+1).
// ---------------------------------------------------------------------------
template <int LOGP, int NT>
__global__ void __launch_bounds__(NT) k_beta_sht(int L, int spin, int real, const double2* __restrict__ G,
                                                 double2* __restrict__ Gw, BetaDev T, double pref) {
  extern __shared__ double2 smem[];
  constexpr int P = 1 << LOGP;
  const int K = 2 * L - 1;
  double2* buf = smem;
  double2* xs = smem + P;
  double2* gsh = xs + K;
  const int mlo = real ? 0 : -(L - 1);
  const int m0 = mlo + 2 * (int)blockIdx.x, m1 = m0 + 1;
  const bool has1 = m1 <= L - 1;
  const int par0 = real ? (m0 & 1) : ((m0 + spin) & 1);
  const bool even0 = par0 == 0;
  const int pitch = real ? L : K;
  auto colptr = [&](int m) -> const double2* {
    const int idx = real ? m : ((m % K) + K) % K;
    return G + idx;
  };
  const double2* c0 = colptr(m0);
  const double2* c1 = has1 ? colptr(m1) : nullptr;
  beta_pair_core<LOGP, NT>(L, even0 ? c0 : c1, even0 ? c1 : c0, pitch, T, buf, xs, gsh);
  const double2 g = *gsh;
  const int mE = even0 ? m0 : m1, mO = even0 ? m1 : m0;
  const int ncol = real ? L : K;
  const int off = real ? 0 : (L - 1);
  for (int mp = -(L - 1) + (int)threadIdx.x; mp <= L - 1; mp += NT) {
    double2 yE, yO;
    y_pair(buf, xs, T.Aalt, L, mp, g, &yE, &yO);
    double2* orow = Gw + (long long)(mp + L - 1) * ncol;
    if (mE <= L - 1) orow[mE + off] = cscale(yE, pref);
    if (mO <= L - 1) orow[mO + off] = cscale(yO, pref);
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
template <int LOGP>
struct NTof { static constexpr int v = LOGP >= 13 ? 512 : 256; };

static size_t beta_smem(int P, int K) { return (size_t)(P + K + 1) * 16 + 64 * 8; }

template <int LOGP>
static int launch_so3(scv_ctx* c, int L, int real, const double2* W1p, double2* w, const BetaTables* t,
                      double pref, const int2* tasks, int ntasks, cudaStream_t s) {
  constexpr int NT = NTof<LOGP>::v;
  size_t sm = beta_smem(1 << LOGP, 2 * L - 1);
  SCV_CUDA(c, cudaFuncSetAttribute(k_beta_so3<LOGP, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_beta_so3<LOGP, NT><<<ntasks, NT, sm, s>>>(L, real, W1p, w, dev_of(t), c->delta, pref, tasks);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

template <int LOGP>
static int launch_sht(scv_ctx* c, int L, int spin, int real, const double2* G, double2* Gw,
                      const BetaTables* t, double pref, cudaStream_t s) {
  constexpr int NT = NTof<LOGP>::v;
  size_t sm = beta_smem(1 << LOGP, 2 * L - 1);
  int ncols = real ? L : 2 * L - 1;
  int npairs = (ncols + 1) / 2;
  SCV_CUDA(c, cudaFuncSetAttribute(k_beta_sht<LOGP, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_beta_sht<LOGP, NT><<<npairs, NT, sm, s>>>(L, spin, real, G, Gw, dev_of(t), pref);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

#define SCV_DISPATCH_LOGP(lg, CALL)                                            \
  switch (lg) {                                                                \
    case 4: return CALL(4); case 5: return CALL(5); case 6: return CALL(6);    \
    case 7: return CALL(7); case 8: return CALL(8); case 9: return CALL(9);    \
    case 10: return CALL(10); case 11: return CALL(11); case 12: return CALL(12); \
    case 13: return CALL(13);                                                  \
    default: return scv_fail(c, SCV_EINVAL, "band limit too large for the beta stage"); \
  }

// task table: (n, pair index), largest degree first (load balance)
static int so3_tasks(scv_ctx* c, int L, int real, const int2** out, int* count, cudaStream_t s) {
  std::string key = "so3tasks_" + std::to_string(L) + "_" + std::to_string(real);
  std::vector<int2> v;
  for (int l = L - 1; l >= 0; --l) {
    for (int sg = 0; sg < 2; ++sg) {
      int n = sg == 0 ? l : -l;
      if (sg == 1 && (l == 0 || real)) continue;
      for (int i = 0; i <= l; ++i) v.push_back(make_int2(n, i));
    }
  }
  *count = (int)v.size();
  auto it = c->aux.find(key);
  if (it != c->aux.end()) {
    *out = (const int2*)it->second;
    return SCV_OK;
  }
  void* d = nullptr;
  SCV_CUDA(c, cudaMalloc(&d, v.size() * sizeof(int2)));
  SCV_CUDA(c, cudaMemcpyAsync(d, v.data(), v.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
  SCV_CUDA(c, cudaStreamSynchronize(s));
  c->aux[key] = d;
  *out = (const int2*)d;
  return SCV_OK;
}

int scv_beta_so3(scv_ctx* c, int L, int real, const double2* W1p, double2* w, double pref,
                 cudaStream_t s) {
  const BetaTables* t = nullptr;
  SCV_TRY(scv_get_beta_tables(c, L, s, &t));
  const int2* tasks = nullptr;
  int nt = 0;
  SCV_TRY(so3_tasks(c, L, real, &tasks, &nt, s));
  static const bool use_v1 = getenv("SCV_BETA_V1") != nullptr;
  if (!use_v1 && scv_beta2_supported(L)) return scv_beta2_so3(c, L, real, W1p, w, pref, t, tasks, nt, s);
#define CALL_SO3(LG) launch_so3<LG>(c, L, real, W1p, w, t, pref, tasks, nt, s)
  SCV_DISPATCH_LOGP(t->logP, CALL_SO3)
#undef CALL_SO3
}

int scv_beta_sht(scv_ctx* c, int L, int spin, int real, const double2* G, double2* Gw, double pref,
                 cudaStream_t s) {
  const BetaTables* t = nullptr;
  SCV_TRY(scv_get_beta_tables(c, L, s, &t));
#define CALL_SHT(LG) launch_sht<LG>(c, L, spin, real, G, Gw, t, pref, s)
  SCV_DISPATCH_LOGP(t->logP, CALL_SHT)
#undef CALL_SHT
}
