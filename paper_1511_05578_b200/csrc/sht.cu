// Spin spherical harmonic transforms on the MW grid (sphere.py:155-260).
//
// forward: phi FFT (cuFFT) -> hand-written beta stage (beta.cu) ->
//          Delta contraction over n=-s (k_sht_contract, one warp per (l,m))
// inverse: Delta outer-product sum into the centred bin plane
//          (k_sht_bins, one thread per bin (m',m), loop over l) ->
//          2-D inverse FFT (cuFFT), rows t<L kept.

#include <cmath>

#include "scv_internal.cuh"

__device__ __forceinline__ double sht_amp(int l, int spin) {
  double a = sqrt((double)(2 * l + 1) / (4.0 * SCV_PI));
  return (spin & 1) ? -a : a;
}

// flm[l^2+l+m] = amp(l,s) i^{m+s} sum_m' D_{m'm} D_{m',-s} Gw[m',m]   (sphere.py:171-181)
// real: m>=0 half + conjugate fill (sphere.py:226-236)
__global__ void k_sht_contract(int L, int spin, int real, const double2* __restrict__ Gw,
                               const double* __restrict__ delta, double2* __restrict__ flm) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= L * L) return;
  int ll = (int)sqrt((double)warp);
  while (ll * ll > warp) --ll;
  while ((ll + 1) * (ll + 1) <= warp) ++ll;
  const int m = warp - ll * ll - ll;
  if (real && m < 0) return;
  const int as = spin < 0 ? -spin : spin;
  if (ll < as) {
    if (lane == 0) flm[warp] = make_double2(0.0, 0.0);
    return;
  }
  const int ncol = real ? L : 2 * L - 1;
  const int coff = real ? 0 : L - 1;
  double sx = 0.0, sy = 0.0;
  for (int mp = -ll + lane; mp <= ll; mp += 32) {
    const double d = wedge_get(delta, ll, mp, m) * wedge_get(delta, ll, mp, -spin);
    const double2 g = Gw[(long long)(mp + L - 1) * ncol + m + coff];
    sx += d * g.x;
    sy += d * g.y;
  }
  for (int o = 16; o > 0; o >>= 1) {
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
  }
  if (lane == 0) {
    const double a = sht_amp(ll, spin);
    double2 v = cipow(make_double2(sx * a, sy * a), m + spin);
    flm[warp] = v;
    if (real && m > 0) {
      double2 cv = make_double2(v.x, -v.y);
      if (m & 1) cv = make_double2(-cv.x, -cv.y);
      flm[ll * ll + ll - m] = cv;
    }
  }
}


// Wedge-pair form of k_sht_contract (SCV_SHT_CONTRACT_WEDGE=1): one thread per
// (l, b = |m|) accumulates f_{l,+b} and f_{l,-b} over a = |m'| = 0..l; the four
// terms (+-a, +-b) share one wedge value, U(+-a) = Delta^l_{+-a,-s} are warp
// broadcasts and Gw[+-a][+-b] are contiguous across the warp's b.
#ifndef SCV_SHT_CONTRACT_WEDGE
#define SCV_SHT_CONTRACT_WEDGE 1
#endif
__global__ void __launch_bounds__(128) k_sht_contract_w(int L, int spin, int real, const double2* __restrict__ Gw,
                                                        const double* __restrict__ delta,
                                                        const double* __restrict__ U, double2* __restrict__ flm) {
  const int K = 2 * L - 1;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)L * (L + 1) / 2) return;
  int l = (int)((sqrt(8.0 * (double)i + 1.0) - 1.0) * 0.5);
  while ((long long)l * (l + 1) / 2 > i) --l;
  while ((long long)(l + 1) * (l + 2) / 2 <= i) ++l;
  const int b = (int)(i - (long long)l * (l + 1) / 2);
  const int as = spin < 0 ? -spin : spin;
  if (l < as) {
    flm[(long long)l * l + l + b] = make_double2(0.0, 0.0);
    if (b > 0) flm[(long long)l * l + l - b] = make_double2(0.0, 0.0);
    return;
  }
  const int ncol = real ? L : K;
  const int coff = real ? 0 : L - 1;
  const bool negm = b > 0 && !real;  // compute m = -b directly (real: conjugate fill)
  const double* Ul = U + (long long)l * K + (L - 1);
  const double* Wl = delta + wedge_plane_base(l);
  double px = 0.0, py = 0.0, nx = 0.0, ny = 0.0;
#pragma unroll 4
  for (int a = 0; a <= l; ++a) {
    const double w = a >= b ? __ldg(Wl + (long long)a * (a + 1) / 2 + b) : __ldg(Wl + (long long)b * (b + 1) / 2 + a);
    const int swp = a < b ? ((b - a) & 1) : 0;  // transpose sign (m'-m parity)
#pragma unroll
    for (int sa = 0; sa < 2; ++sa) {
      if (sa && a == 0) continue;
      const int mp = sa ? -a : a;
      const double u = __ldg(Ul + mp);
      const double2* grow = Gw + (long long)(mp + L - 1) * ncol + coff;
      {  // m = +b
        int neg = swp;
        if (mp < 0) neg ^= (l + b) & 1;
        const double d = (neg ? -w : w) * u;
        const double2 g = __ldg(grow + b);
        px += d * g.x;
        py += d * g.y;
      }
      if (negm) {  // m = -b
        int neg = swp;
        if (mp < 0) neg ^= (l - b) & 1;
        neg ^= (l + a) & 1;
        const double d = (neg ? -w : w) * u;
        const double2 g = __ldg(grow - b);
        nx += d * g.x;
        ny += d * g.y;
      }
    }
  }
  const double amp = sht_amp(l, spin);
  const double2 v = cipow(make_double2(px * amp, py * amp), b + spin);
  flm[(long long)l * l + l + b] = v;
  if (b > 0) {
    if (real) {
      double2 cv = make_double2(v.x, -v.y);
      if (b & 1) cv = make_double2(-cv.x, -cv.y);
      flm[(long long)l * l + l - b] = cv;
    } else {
      flm[(long long)l * l + l - b] = cipow(make_double2(nx * amp, ny * amp), -b + spin);
    }
  }
}

// k_sht_contract_w for SCV_SHT_LC consecutive degrees per thread (r02): the bins Gw[+-a][+-b] of an
// (a, b) are loaded once for the chunk instead of once per degree.  k_sht_contract_w moved 24.9 GB
// between L2 and the SMs at L = 1024 (ncu, profiles/r03_ncu_k_sht_contract_w.txt: 81% of its stall
// samples wait on those loads), 4/5 of it the bins.  Per (l, b) the terms are added in the same
// order with the same operands, so the coefficients are bit-identical.  Measured at L = 1024
// (ms): 1 degree per thread 3.04, 2: 1.83, 4: 2.62, 8: 4.86 (too few threads, longer loops).
#ifndef SCV_SHT_LC
#define SCV_SHT_LC 2
#endif
__global__ void __launch_bounds__(128) k_sht_contract_c(int L, int spin, int real, const double2* __restrict__ Gw,
                                                        const double* __restrict__ delta,
                                                        const double* __restrict__ U, double2* __restrict__ flm) {
  constexpr int LC = SCV_SHT_LC;
  const int K = 2 * L - 1;
  const int nch = (L + LC - 1) / LC;
  const int l0 = (nch - 1 - (int)blockIdx.y) * LC;  // large degrees (long loops) first
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int ltop = min(l0 + LC, L) - 1;
  if (b > ltop) return;
  const int as = spin < 0 ? -spin : spin;
  const int ncol = real ? L : K;
  const int coff = real ? 0 : L - 1;
  const bool negm = b > 0 && !real;  // compute m = -b directly (real: conjugate fill)
  double px[LC], py[LC], nx[LC], ny[LC];
#pragma unroll
  for (int i = 0; i < LC; ++i) px[i] = py[i] = nx[i] = ny[i] = 0.0;
#pragma unroll 2
  for (int a = 0; a <= ltop; ++a) {
    const int swp = a < b ? ((b - a) & 1) : 0;  // transpose sign (m'-m parity)
    const long long widx = a >= b ? (long long)a * (a + 1) / 2 + b : (long long)b * (b + 1) / 2 + a;
    const double2* gp = Gw + (long long)(a + L - 1) * ncol + coff;
    const double2* gn = Gw + (long long)(-a + L - 1) * ncol + coff;
    const double2 gpp = __ldg(gp + b);
    const double2 gpn = negm ? __ldg(gp - b) : make_double2(0.0, 0.0);
    const double2 gnp = a ? __ldg(gn + b) : make_double2(0.0, 0.0);
    const double2 gnn = (a && negm) ? __ldg(gn - b) : make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < LC; ++i) {
      const int l = l0 + i;
      if (l > ltop || l < as || a > l || b > l) continue;
      const double w = __ldg(delta + wedge_plane_base(l) + widx);
      const double* Ul = U + (long long)l * K + (L - 1);
#pragma unroll
      for (int sa = 0; sa < 2; ++sa) {
        if (sa && a == 0) continue;
        const int mp = sa ? -a : a;
        const double u = __ldg(Ul + mp);
        {  // m = +b
          int neg = swp;
          if (mp < 0) neg ^= (l + b) & 1;
          const double d = (neg ? -w : w) * u;
          const double2 g = sa ? gnp : gpp;
          px[i] += d * g.x;
          py[i] += d * g.y;
        }
        if (negm) {  // m = -b
          int neg = swp;
          if (mp < 0) neg ^= (l - b) & 1;
          neg ^= (l + a) & 1;
          const double d = (neg ? -w : w) * u;
          const double2 g = sa ? gnn : gpn;
          nx[i] += d * g.x;
          ny[i] += d * g.y;
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < LC; ++i) {
    const int l = l0 + i;
    if (l > ltop || b > l) continue;
    if (l < as) {
      flm[(long long)l * l + l + b] = make_double2(0.0, 0.0);
      if (b > 0) flm[(long long)l * l + l - b] = make_double2(0.0, 0.0);
      continue;
    }
    const double amp = sht_amp(l, spin);
    const double2 v = cipow(make_double2(px[i] * amp, py[i] * amp), b + spin);
    flm[(long long)l * l + l + b] = v;
    if (b > 0) {
      if (real) {
        double2 cv = make_double2(v.x, -v.y);
        if (b & 1) cv = make_double2(-cv.x, -cv.y);
        flm[(long long)l * l + l - b] = cv;
      } else {
        flm[(long long)l * l + l - b] = cipow(make_double2(nx[i] * amp, ny[i] * amp), -b + spin);
      }
    }
  }
}

// B[m' mod K][m mod K] = e^{i m' pi/K} i^{-(m+s)} sum_{l} amp D_{m'm} D_{m',-s} f_lm   (sphere.py:191-203)
// real: B[m' mod K][m], m in [0,L)   (sphere.py:245-252)
__global__ void k_sht_bins(int L, int spin, int real, const double2* __restrict__ flm,
                           const double* __restrict__ delta, double2* __restrict__ B) {
  const int K = 2 * L - 1;
  const int ncol = real ? L : K;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)K * ncol) return;
  const int r = (int)(idx / ncol), cidx = (int)(idx % ncol);
  const int mp = r - (L - 1);
  const int m = real ? cidx : cidx - (L - 1);
  const int as = spin < 0 ? -spin : spin;
  int l0 = mp < 0 ? -mp : mp;
  const int am = m < 0 ? -m : m;
  if (am > l0) l0 = am;
  if (as > l0) l0 = as;
  double sx = 0.0, sy = 0.0;
  for (int l = l0; l < L; ++l) {
    const double a = sht_amp(l, spin);
    const double2 f = flm[l * l + l + m];
    const double u = wedge_get(delta, l, mp, -spin);
    const double d = wedge_get(delta, l, mp, m);
    // (u * (amp f)) * d  -- reference order
    sx += (u * (a * f.x)) * d;
    sy += (u * (a * f.y)) * d;
  }
  double2 v = cipow(make_double2(sx, sy), -(m + spin));
  double sn, cs;
  sincos((double)mp * (SCV_PI / (double)K), &sn, &cs);
  v = cmul(v, make_double2(cs, sn));
  const int row = ((mp % K) + K) % K;
  const int col = real ? m : ((m % K) + K) % K;
  B[(long long)row * ncol + col] = v;
}


// Wedge-pair form of k_sht_bins (default, SCV_SHT_BINS_WEDGE=1): one thread
// per Delta wedge pair (a, b), 0 <= b <= a < L, produces every bin (m', m) in
// {(+-a, +-b), (+-b, +-a)} from ONE wedge load per degree: the eight bins
// share |Delta^l_{ab}|, and consecutive threads take consecutive b, so the
// wedge, the u column and the f_{l,+-b} loads are contiguous.  The per-bin
// arithmetic is k_sht_bins' (same operands, same order).
#ifndef SCV_SHT_BINS_WEDGE
#define SCV_SHT_BINS_WEDGE 1
#endif

// U[l][mp + L - 1] = Delta^l_{mp,-s}, |mp| <= l
__global__ void k_sht_ucol(int L, int spin, const double* __restrict__ delta, double* __restrict__ U) {
  const int K = 2 * L - 1;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)L * K) return;
  const int l = (int)(t / K), mp = (int)(t - (long long)l * K) - (L - 1);
  const int as = spin < 0 ? -spin : spin;
  U[t] = (mp >= -l && mp <= l && l >= as) ? wedge_get(delta, l, mp, -spin) : 0.0;
}

__global__ void __launch_bounds__(128) k_sht_bins_w(int L, int spin, int real, const double2* __restrict__ flm,
                                                    const double* __restrict__ delta, const double* __restrict__ U,
                                                    double2* __restrict__ B) {
  const int K = 2 * L - 1;
  const int ncol = real ? L : K;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)L * (L + 1) / 2) return;
  int a = (int)((sqrt(8.0 * (double)i + 1.0) - 1.0) * 0.5);
  while ((long long)a * (a + 1) / 2 > i) --a;
  while ((long long)(a + 1) * (a + 2) / 2 <= i) ++a;
  const int b = (int)(i - (long long)a * (a + 1) / 2);
  const int as = spin < 0 ? -spin : spin;
  // slot k: swap = k >> 2 (m' = +-b, m = +-a), sign of m' = bit 1, sign of m = bit 0
  int mpk[8], mk[8];
  bool ok[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int sw = k >> 2, s1 = (k >> 1) & 1, s2 = k & 1;
    const int x = sw ? b : a, y = sw ? a : b;
    mpk[k] = s1 ? -x : x;
    mk[k] = s2 ? -y : y;
    ok[k] = !(s1 && x == 0) && !(s2 && y == 0) && !(sw && a == b) && !(real && mk[k] < 0);
  }
  double sx[8], sy[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) sx[k] = sy[k] = 0.0;
  const int l0 = a > as ? a : as;
  // the wedge loads of successive degrees are independent DRAM accesses one
  // plane apart: unrolled so several are in flight per thread
#pragma unroll 4
  for (int l = l0; l < L; ++l) {
    const double amp = sht_amp(l, spin);
    const double w = __ldg(delta + wedge_plane_base(l) + (long long)a * (a + 1) / 2 + b);
    const double* Ul = U + (long long)l * K + (L - 1);
    const double2* fl = flm + (long long)l * l + l;
    const double uap = __ldg(Ul + a), uan = __ldg(Ul - a), ubp = __ldg(Ul + b), ubn = __ldg(Ul - b);
    const double2 fap = __ldg(fl + a), fbp = __ldg(fl + b);
    const double2 fan = real ? fap : __ldg(fl - a), fbn = real ? fbp : __ldg(fl - b);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (!ok[k]) continue;
      const int sw = k >> 2, s1 = (k >> 1) & 1, s2 = k & 1;
      const int mp = mpk[k], m = mk[k];
      // sign of Delta^l_{mp,m} relative to the wedge value (wedge_get's rules)
      int neg = 0;
      if (mp < 0) neg ^= (l + m) & 1;
      if (m < 0) neg ^= (l + (mp < 0 ? -mp : mp)) & 1;
      if (sw) neg ^= (a - b) & 1;
      const double d = neg ? -w : w;
      const double u = sw ? (s1 ? ubn : ubp) : (s1 ? uan : uap);
      const double2 f = sw ? (s2 ? fan : fap) : (s2 ? fbn : fbp);
      sx[k] += (u * (amp * f.x)) * d;
      sy[k] += (u * (amp * f.y)) * d;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (!ok[k]) continue;
    const int mp = mpk[k], m = mk[k];
    double2 v = cipow(make_double2(sx[k], sy[k]), -(m + spin));
    double sn, cs;
    sincos((double)mp * (SCV_PI / (double)K), &sn, &cs);
    v = cmul(v, make_double2(cs, sn));
    const int row = ((mp % K) + K) % K;
    const int col = real ? m : ((m % K) + K) % K;
    B[(long long)row * ncol + col] = v;
  }
}

__global__ void k_zero_imag_col0(double2* B, int rows, int pitch) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < rows) B[(long long)t * pitch].y = 0.0;
}

static int check_sht_args(scv_ctx* c, int L, int spin, int real) {
  if (L < 1) return scv_fail(c, SCV_EINVAL, "band limit must be positive, got " + std::to_string(L));
  if (std::abs(spin) >= L)
    return scv_fail(c, SCV_EINVAL, "spin " + std::to_string(spin) + " out of range for band limit " + std::to_string(L));
  if (real && spin != 0) return scv_fail(c, SCV_EINVAL, "real signals must have spin 0");
  return SCV_OK;
}

extern "C" int scv_sht_forward(scv_ctx* c, int L, int spin, int real, const void* f, double* flm,
                               void* stream) {
  if (!c) return SCV_EINVAL;
  SCV_TRY(check_sht_args(c, L, spin, real));
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_TRY(scv_ensure_delta(c, L, s));
  const int K = 2 * L - 1;
  const int ncol = real ? L : K;
  void* G = nullptr;
  void* Gw = nullptr;
  SCV_TRY(scv_scratch(c, 1, (size_t)L * ncol * 16, &G));
  SCV_TRY(scv_scratch(c, 2, (size_t)K * ncol * 16, &Gw));
  cufftHandle h;
  int n[1] = {K};
  {
  SCV_PROF(c, s, "sht_phi_fft");
  if (real) {
    int on[1] = {L};
    SCV_TRY(scv_plan(c, "sht_phi_d2z_" + std::to_string(L), 1, n, n, 1, K, on, 1, L, CUFFT_D2Z, L, &h));
    SCV_TRY(scv_plan_exec_setup(c, h, s));
    SCV_CUFFT(c, cufftExecD2Z(h, (double*)f, (cufftDoubleComplex*)G));
  } else {
    SCV_TRY(scv_plan(c, "sht_phi_z2z_" + std::to_string(L), 1, n, n, 1, K, n, 1, K, CUFFT_Z2Z, L, &h));
    SCV_TRY(scv_plan_exec_setup(c, h, s));
    SCV_CUFFT(c, cufftExecZ2Z(h, (cufftDoubleComplex*)f, (cufftDoubleComplex*)G, CUFFT_FORWARD));
  }
  }
  {
  SCV_PROF(c, s, "beta_sht");
  SCV_TRY(scv_beta_sht(c, L, spin, real, (const double2*)G, (double2*)Gw, 2.0 * SCV_PI / (double)K, s));
  }
  SCV_PROF(c, s, "sht_contract");
  if (SCV_SHT_CONTRACT_WEDGE) {
    void* U = nullptr;
    SCV_TRY(scv_scratch(c, 0, (size_t)L * K * 8, &U));
    k_sht_ucol<<<(int)(((long long)L * K + 255) / 256), 256, 0, s>>>(L, spin, c->delta, (double*)U);
    c->launches++;
    if (SCV_SHT_LC > 1) {
      k_sht_contract_c<<<dim3((L + 127) / 128, (L + SCV_SHT_LC - 1) / SCV_SHT_LC), 128, 0, s>>>(
          L, spin, real, (const double2*)Gw, c->delta, (const double*)U, (double2*)flm);
    } else {
      const long long np = (long long)L * (L + 1) / 2;
      k_sht_contract_w<<<(int)((np + 127) / 128), 128, 0, s>>>(L, spin, real, (const double2*)Gw, c->delta,
                                                               (const double*)U, (double2*)flm);
    }
    c->launches++;
  } else {
    const long long warps = (long long)L * L;
    k_sht_contract<<<(int)((warps * 32 + 255) / 256), 256, 0, s>>>(L, spin, real, (const double2*)Gw,
                                                                   c->delta, (double2*)flm);
    c->launches++;
  }
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

extern "C" int scv_sht_inverse(scv_ctx* c, int L, int spin, int real, const double* flm, void* f,
                               void* stream) {
  if (!c) return SCV_EINVAL;
  SCV_TRY(check_sht_args(c, L, spin, real));
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_TRY(scv_ensure_delta(c, L, s));
  const int K = 2 * L - 1;
  const int ncol = real ? L : K;
  void* B = nullptr;
  SCV_TRY(scv_scratch(c, 1, (size_t)K * ncol * 16, &B));
  const long long tot = (long long)K * ncol;
  {
  SCV_PROF(c, s, "sht_bins");
  if (SCV_SHT_BINS_WEDGE) {
    void* U = nullptr;
    SCV_TRY(scv_scratch(c, 2, (size_t)L * K * 8, &U));
    k_sht_ucol<<<(int)(((long long)L * K + 255) / 256), 256, 0, s>>>(L, spin, c->delta, (double*)U);
    c->launches++;
    const long long np = (long long)L * (L + 1) / 2;
    k_sht_bins_w<<<(int)((np + 127) / 128), 128, 0, s>>>(L, spin, real, (const double2*)flm, c->delta,
                                                         (const double*)U, (double2*)B);
    c->launches++;
  } else {
    k_sht_bins<<<(int)((tot + 127) / 128), 128, 0, s>>>(L, spin, real, (const double2*)flm, c->delta,
                                                        (double2*)B);
    c->launches++;
  }
  SCV_CUDA(c, cudaGetLastError());
  }
  SCV_PROF(c, s, "sht_ifft");
  cufftHandle h;
  if (!real) {
    int n2[2] = {K, K};
    SCV_TRY(scv_plan(c, "sht_inv2d_" + std::to_string(L), 2, n2, n2, 1, K * K, n2, 1, K * K, CUFFT_Z2Z, 1, &h));
    SCV_TRY(scv_plan_exec_setup(c, h, s));
    SCV_CUFFT(c, cufftExecZ2Z(h, (cufftDoubleComplex*)B, (cufftDoubleComplex*)B, CUFFT_INVERSE));
    SCV_CUDA(c, cudaMemcpyAsync(f, B, (size_t)L * K * 16, cudaMemcpyDeviceToDevice, s));
    return SCV_OK;
  }
  // theta: inverse along axis 0 of the (K, L) plane, columns strided by L
  int n1[1] = {K};
  int emb[1] = {K * L};
  SCV_TRY(scv_plan(c, "sht_inv_theta_" + std::to_string(L), 1, n1, emb, L, 1, emb, L, 1, CUFFT_Z2Z, L, &h));
  SCV_TRY(scv_plan_exec_setup(c, h, s));
  SCV_CUFFT(c, cufftExecZ2Z(h, (cufftDoubleComplex*)B, (cufftDoubleComplex*)B, CUFFT_INVERSE));
  // irfft discards Im of the DC bin (scipy semantics); make that explicit for cuFFT
  k_zero_imag_col0<<<(L + 127) / 128, 128, 0, s>>>((double2*)B, L, L);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  int on[1] = {K}, in1[1] = {L};
  SCV_TRY(scv_plan(c, "sht_inv_phi_z2d_" + std::to_string(L), 1, n1, in1, 1, L, on, 1, K, CUFFT_Z2D, L, &h));
  SCV_TRY(scv_plan_exec_setup(c, h, s));
  SCV_CUFFT(c, cufftExecZ2D(h, (cufftDoubleComplex*)B, (double*)f));
  return SCV_OK;
}
