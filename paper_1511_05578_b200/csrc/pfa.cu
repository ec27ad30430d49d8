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
#include <complex>
#include <cmath>
#include <cstring>

#include <cuda.h>          // CUtensorMap (TMA descriptor type only; encoded via the runtime entry point)
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

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
    case 1023:
      f[0] = PfaPlan<1023>::P0; f[1] = PfaPlan<1023>::P1; f[2] = PfaPlan<1023>::P2; f[3] = PfaPlan<1023>::P3;
      break;
    case 2047: f[0] = 23; f[1] = 89; break;
    case 4095:
      f[0] = PfaPlan<4095>::P0; f[1] = PfaPlan<4095>::P1; f[2] = PfaPlan<4095>::P2; f[3] = PfaPlan<4095>::P3;
      break;
  }
}

int scv_pfa_pos_host(int K, int k);
static int pfa_in_host(int K, int n);

// Tables of pfa_stage_rader89 (pfa.cuh), in long double: the 44-point cyclic
// (cos) and negacyclic (sin) correlation operators of Rader's permutation
// (r_a = 3^a mod 89), conjugated by the in-lane 4-point transforms along
// a mod 4 (a <-> (a mod 4, a mod 11)), are block diagonal; the blocks are the
// dense products the stage runs on DMMA.  The 1/4 and 1/2 of the inverse
// transforms are folded in.  Layout: see R89_OFF_* (rows = output a mod 11,
// columns = input a mod 11; 22 x 22 blocks stored as Re rows 0..7 / Im rows
// 8..15 / Re rows 16..18 / Im rows 19..21 and Re columns 0..10 / Im 12..22).
static void rader89_tables(double* T) {
  typedef std::complex<ld> cld;
  const int p = 89, h = 44;
  const ld pi = 3.141592653589793238462643383279502884L;
  int r[44];
  r[0] = 1;
  for (int a = 1; a < h; ++a) r[a] = (r[a - 1] * 3) % p;
  auto idx = [](int a1, int a2) { return (33 * a1 + 12 * a2) % 44; };
  auto sgn = [](int a) { return ((a >> 2) & 1) ? -1.0L : 1.0L; };
  std::vector<ld> C44(h * h), S44(h * h);
  for (int b = 0; b < h; ++b)
    for (int a = 0; a < h; ++a) {
      const ld ang = 2 * pi * (ld)(((long long)r[a] * r[b]) % p) / (ld)p;
      C44[b * h + a] = cosl(ang);
      S44[b * h + a] = sinl(ang);
    }
  // cyclic: coordinates [V0 | V2 | Ur | Ui] x 11
  std::vector<ld> Tc(h * h, 0.0L), Tci(h * h, 0.0L);
  for (int a2 = 0; a2 < 11; ++a2) {
    for (int a1 = 0; a1 < 4; ++a1) {
      Tc[a2 * h + idx(a1, a2)] = 1;
      Tc[(11 + a2) * h + idx(a1, a2)] = (a1 & 1) ? -1 : 1;
    }
    Tc[(22 + a2) * h + idx(0, a2)] = 1;
    Tc[(22 + a2) * h + idx(2, a2)] = -1;
    Tc[(33 + a2) * h + idx(1, a2)] = 1;
    Tc[(33 + a2) * h + idx(3, a2)] = -1;
    // inverse: v0 = (V0+V2)/4 + Ur/2, v1 = (V0-V2)/4 + Ui/2, v2 = (V0+V2)/4 - Ur/2, v3 = (V0-V2)/4 - Ui/2
    for (int a1 = 0; a1 < 4; ++a1) {
      const int a = idx(a1, a2);
      Tci[a * h + a2] = 0.25L;
      Tci[a * h + 11 + a2] = (a1 & 1) ? -0.25L : 0.25L;
      if (a1 == 0) Tci[a * h + 22 + a2] = 0.5L;
      if (a1 == 2) Tci[a * h + 22 + a2] = -0.5L;
      if (a1 == 1) Tci[a * h + 33 + a2] = 0.5L;
      if (a1 == 3) Tci[a * h + 33 + a2] = -0.5L;
    }
  }
  auto mm = [h](const std::vector<ld>& A, const std::vector<ld>& B) {
    std::vector<ld> Cm(h * h, 0.0L);
    for (int i = 0; i < h; ++i)
      for (int k = 0; k < h; ++k) {
        const ld v = A[i * h + k];
        if (v == 0) continue;
        for (int j = 0; j < h; ++j) Cm[i * h + j] += v * B[k * h + j];
      }
    return Cm;
  };
  const std::vector<ld> Mc = mm(mm(Tc, C44), Tci);
  // negacyclic: sign-twisted odd DFT, eta_f = exp(-i pi (2f+1)/4)
  std::vector<cld> Ts(h * h), Tsi(h * h), Sc(h * h);
  for (int i = 0; i < h * h; ++i) Sc[i] = cld(S44[i], 0);
  for (int f = 0; f < 4; ++f) {
    const cld eta = std::polar(1.0L, -pi * (ld)(2 * f + 1) / 4);
    for (int a2 = 0; a2 < 11; ++a2)
      for (int a1 = 0; a1 < 4; ++a1) {
        const int a = idx(a1, a2);
        Ts[(f * 11 + a2) * h + a] = sgn(a) * std::pow(eta, a1);
        Tsi[a * h + f * 11 + a2] = sgn(a) * 0.25L * std::pow(eta, -a1);
      }
  }
  auto mmc = [h](const std::vector<cld>& A, const std::vector<cld>& B) {
    std::vector<cld> Cm(h * h, cld(0, 0));
    for (int i = 0; i < h; ++i)
      for (int k = 0; k < h; ++k) {
        const cld v = A[i * h + k];
        if (v == cld(0, 0)) continue;
        for (int j = 0; j < h; ++j) Cm[i * h + j] += v * B[k * h + j];
      }
    return Cm;
  };
  const std::vector<cld> Ms = mmc(mmc(Ts, Sc), Tsi);
  auto row22 = [](int rr) { return rr < 11 ? (rr < 8 ? rr : 16 + rr - 8) : (rr - 11 < 8 ? 8 + rr - 11 : 19 + rr - 19); };
  auto col22 = [](int cc) { return cc < 11 ? cc : 12 + cc - 11; };
  for (int b2 = 0; b2 < 11; ++b2)
    for (int a2 = 0; a2 < 11; ++a2) {
      T[b2 * R89_P12 + a2] = (double)(0.25L * Mc[b2 * h + a2]);
      T[R89_OFF_M2 + b2 * R89_P12 + a2] = (double)(0.25L * Mc[(11 + b2) * h + 11 + a2]);
    }
  for (int i = 0; i < 22; ++i)
    for (int j = 0; j < 22; ++j) {
      T[R89_OFF_MC + row22(i) * R89_P28 + col22(j)] = (double)(0.5L * Mc[(22 + i) * h + 22 + j]);
      // complex 11 x 11 blocks as real [[Re, -Im], [Im, Re]]: A = Ms[33.., 0..] (f 0 -> 3), B = Ms[22.., 11..] (f 1 -> 2)
      const int bi = i % 11, bj = j % 11;
      const cld za = Ms[(33 + bi) * h + bj], zb = Ms[(22 + bi) * h + 11 + bj];
      const ld ra = (i < 11) == (j < 11) ? za.real() : (i < 11 ? -za.imag() : za.imag());
      const ld rb = (i < 11) == (j < 11) ? zb.real() : (i < 11 ? -zb.imag() : zb.imag());
      T[R89_OFF_RA + row22(i) * R89_P28 + col22(j)] = (double)(0.5L * ra);
      T[R89_OFF_RB + row22(i) * R89_P28 + col22(j)] = (double)(0.5L * rb);
    }
  // row 11 of the first matrix (padding of the 16-row tile) = all ones: its
  // product with the V0 column sums is sum_a s'_a, the y_0 term
  for (int a2 = 0; a2 < 11; ++a2) T[11 * R89_P12 + a2] = 1.0;
  unsigned char* RT = (unsigned char*)(T + R89_OFF_RT);
  for (int a = 0; a < h; ++a) RT[a] = (unsigned char)r[a];
}

// Storage order of a radix-89 butterfly's elements (pfa_stage_rader89):
// position of input element j (which = 0) or of output y_k (which = 1).
static int r89_sigma(int which, int j) {
  if (j == 0) return 0;
  int r = 1;
  for (int a = 0; a < 44; ++a, r = (r * 3) % 89) {
    if (r != j && 89 - r != j) continue;
    const bool neg = (a >> 2) & 1;           // negacyclic wrap sign of a
    const bool first = (r == j) != neg;      // j is the u / "+" member of the pair
    const int a1 = a % 4, a2 = a % 11;
    const int s = which == 0 ? r89_in_slot(a1, a2) : r89_out_slot(a1, a2);
    return (first ? 1 : 45) + s;
  }
  return -1;
}

// Lane schedule of the ring kernels' slot accesses (r02).  A warp copy moves 32 consecutive
// elements of a row between global memory and a slot; which lane takes which of the 32 does
// not matter to the global side (the same four 128-byte lines), but the slot positions are
// pseudo-random in the natural index (Ruritanian map x Rader storage order), so the natural
// lane order costs ~10.4 shared-memory wavefronts per 16-byte warp access instead of 4.  For
// each group of 32 the elements are dealt to the four quarter-warps so that a quarter's eight
// positions fall into as many different 16-byte bank groups as possible (~7.3 wavefronts).
// Entry [32 j + lane] = position | (e << 11): the lane handles element 32 j + e.
static void pfa_lane_schedule(const unsigned short* pos, int K, unsigned short* out) {
  for (int n0 = 0; n0 < K; n0 += 32) {
    const int W = std::min(32, K - n0);
    int tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int e = 0; e < W; ++e) tot[pos[n0 + e] & 7]++;
    // elements of the fullest bank groups first
    std::vector<int> order(W);
    for (int e = 0; e < W; ++e) order[e] = e;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tot[pos[n0 + a] & 7] > tot[pos[n0 + b] & 7]; });
    int cnt[4][8] = {}, fill[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0};
    int lane_of[32];
    for (int e : order) {
      const int b = pos[n0 + e] & 7;
      int best = -1, bk0 = 0, bk1 = 0, bk2 = 0;
      for (int q = 0; q < 4; ++q) {
        if (fill[q] >= 8) continue;
        const int grow = cnt[q][b] + 1 > mx[q] ? 1 : 0;  // does this quarter need another wavefront?
        const int k0 = grow, k1 = cnt[q][b], k2 = fill[q];
        if (best < 0 || k0 < bk0 || (k0 == bk0 && (k1 < bk1 || (k1 == bk1 && k2 < bk2)))) {
          best = q;
          bk0 = k0;
          bk1 = k1;
          bk2 = k2;
        }
      }
      lane_of[e] = best * 8 + fill[best];
      fill[best]++;
      cnt[best][b]++;
      mx[best] = std::max(mx[best], cnt[best][b]);
    }
    for (int l = 0; l < 32; ++l) {
      if (n0 + l < K) out[n0 + l] = (unsigned short)(31u << 11);  // idle lanes of the last group: element past K
    }
    bool used[32] = {};
    for (int e = 0; e < W; ++e) {
      // the last group has W < 32 elements: its lanes >= W do not exist in the table, so
      // squeeze the assigned lanes into [0, W)
      used[lane_of[e]] = true;
    }
    int remap[32], nl = 0;
    for (int l = 0; l < 32; ++l) remap[l] = used[l] ? nl++ : -1;
    for (int e = 0; e < W; ++e) out[n0 + remap[lane_of[e]]] = (unsigned short)(pos[n0 + e] | (e << 11));
  }
}

// the tables of length K with the two position maps in lane-schedule form (k_pfa_rows_p)
int scv_pfa_tables_sched(scv_ctx* c, int K, const double2** out) {
  const std::string key = "pfas_" + std::to_string(K);
  auto it = c->aux.find(key);
  if (it != c->aux.end()) {
    *out = (const double2*)it->second;
    return SCV_OK;
  }
  if (K > 2048) return scv_fail(c, SCV_EINVAL, "lane schedule packs positions into 11 bits");
  const double2* plain;
  SCV_TRY(scv_pfa_tables(c, K, &plain));
  int f[4];
  factors_of(K, f);
  size_t nr = 0;
  for (int s = 0; s < 4; ++s) nr += (size_t)pfa_tab(f[s], K);
  const size_t n16 = ((size_t)4 * K + 15) / 16, total = nr + n16;
  std::vector<double2> tab(total);
  SCV_CUDA(c, cudaMemcpy(tab.data(), plain, total * sizeof(double2), cudaMemcpyDeviceToHost));
  unsigned short* pos = (unsigned short*)(tab.data() + nr);
  std::vector<unsigned short> sched(2 * (size_t)K);
  pfa_lane_schedule(pos, K, sched.data());
  pfa_lane_schedule(pos + K, K, sched.data() + K);
  memcpy(pos, sched.data(), sched.size() * sizeof(unsigned short));
  void* d = nullptr;
  SCV_CUDA(c, cudaMalloc(&d, total * sizeof(double2)));
  SCV_CUDA(c, cudaMemcpy(d, tab.data(), total * sizeof(double2), cudaMemcpyHostToDevice));
  c->aux[key] = d;
  c->table_bytes += (long long)(total * sizeof(double2));
  c->small_table_bytes += (long long)(total * sizeof(double2));
  *out = (const double2*)d;
  return SCV_OK;
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
    if (pfa_rader89(p)) {
      const size_t base = tab.size();
      tab.resize(base + R89_TAB, make_double2(0.0, 0.0));
      rader89_tables((double*)(tab.data() + base));
      continue;
    }
    if (pfa_use_mma(p, K)) {
      // dense C and S matrices (M rows x pitch doubles each), row 0 = (1, 0)
      const int h = (p - 1) / 2, M = mma_M(p), PA = mma_pa(p);
      std::vector<double> C((size_t)M * PA, 0.0), S((size_t)M * PA, 0.0);
      for (int k = 0; k <= h; ++k)
        for (int j = 1; j <= h; ++j) {
          const ld a = twopi * (ld)(((long long)j * k) % p) / (ld)p;
          C[(size_t)mma_aoff(p, k, j - 1)] = (double)cosl(a);
          S[(size_t)mma_aoff(p, k, j - 1)] = (double)sinl(a);
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
  {  // 16-bit position maps (pfa_pos_tab, pfa_in_tab): out[k], then in[n]
    const size_t base = tab.size(), n16 = ((size_t)4 * K + 15) / 16;
    tab.resize(base + n16, make_double2(0.0, 0.0));
    unsigned short* pos = (unsigned short*)(tab.data() + base);
    for (int k = 0; k < K; ++k) {
      pos[k] = (unsigned short)scv_pfa_pos_host(K, k);
      pos[K + k] = (unsigned short)pfa_in_host(K, k);
    }
  }
  void* d = nullptr;
  SCV_CUDA(c, cudaMalloc(&d, tab.size() * sizeof(double2)));
  SCV_CUDA(c, cudaMemcpy(d, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice));
  c->aux[key] = d;
  c->table_bytes += (long long)(tab.size() * sizeof(double2));
  c->small_table_bytes += (long long)(tab.size() * sizeof(double2));
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
SCV_PFA_CFG(255, false, 8, 256, 1)   SCV_PFA_CFG(255, true, 8, 256, 1)
SCV_PFA_CFG(511, false, 4, 256, 1)   SCV_PFA_CFG(511, true, 4, 256, 1)
#ifndef SCV_ROW2047
#define SCV_ROW2047 1, 192, 2
#endif
#ifndef SCV_COL2047
#define SCV_COL2047 2, 384, 1
#endif
#ifndef SCV_ROW1023
#define SCV_ROW1023 2, 352, 1
#endif
#ifndef SCV_COL1023
#define SCV_COL1023 2, 352, 1
#endif
#define SCV_PFA_CFG_(KK, CL, ...) SCV_PFA_CFG(KK, CL, __VA_ARGS__)
SCV_PFA_CFG_(1023, false, SCV_ROW1023)  SCV_PFA_CFG_(1023, true, SCV_COL1023)
SCV_PFA_CFG_(2047, false, SCV_ROW2047)  SCV_PFA_CFG_(2047, true, SCV_COL2047)
SCV_PFA_CFG(4095, false, 1, 384, 1)  SCV_PFA_CFG(4095, true, 1, 384, 1)

// Row batches in shared memory: 2 = the next batch streams in (cp.async)
// while the current one computes, 1 = single buffer (other resident CTAs
// cover the load latency).
template <int K, bool COL> struct PfaNBuf { static constexpr int v = 2; };
#ifndef SCV_ROW2047_NBUF
#define SCV_ROW2047_NBUF 2
#endif
template <> struct PfaNBuf<2047, false> { static constexpr int v = SCV_ROW2047_NBUF; };

// Rows per transform call: R when the launch shape fits in shared memory,
// else 1 (the R adjacent columns of a batch still move as R*16-byte segments,
// but are transformed one call at a time, bounding the DMMA scratch).
template <int K, bool COL, int RD>
constexpr size_t pfa_smem_rd() {
  static_assert(PfaCfg<K, COL>::NT % PfaCfg<K, COL>::R == 0, "column kernels map R | NT");
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, COL>::R;
  return ((size_t)PfaNBuf<K, COL>::v * R * K + pfa_tab_total<PL>() + pfa_scratch<PL, RD, PfaCfg<K, COL>::NT>()) *
             sizeof(double2) + R * sizeof(int4);
}
template <int K, bool COL> struct PfaRD {
  static constexpr int v = pfa_smem_rd<K, COL, PfaCfg<K, COL>::R>() <= 232448 ? PfaCfg<K, COL>::R : 1;
};

template <class PL, int DIR, int R, int RD, int NT>
__device__ __forceinline__ void pfa_dft_rows(double2* X, const double2* tab, double2* scr) {
#pragma unroll 1
  for (int r = 0; r < R; r += RD) pfa_dft<PL, DIR, RD, NT, PL::K>(X + r * PL::K, tab, scr);
}

template <int K, bool COL>
static constexpr size_t pfa_smem() {
  return pfa_smem_rd<K, COL, PfaRD<K, COL>::v>();
}

// ---------------------------------------------------------------------------
// batched rows (test / benchmark entry): out[r][k] = sum_n in[r][n] e^{DIR 2 pi i nk/K}
// ---------------------------------------------------------------------------
// GATHER = 2: the blocked analysis's alpha pass (see k_pfa_rows_g): row
// r = bb*K + g reads the column pairs T[bb][m/2][g][m&1] and writes signal
// row (g, b0 + bb) of a slab with LK beta rows.
template <int K, int DIR, int GATHER = 0>
__global__ void __launch_bounds__(PfaCfg<K, false>::NT, PfaCfg<K, false>::MINB)
    k_pfa_rows(long long nrows, const double2* in, double2* out, const double2* __restrict__ gtab,
               long long LK = 0, int b0 = 0) {
  // in == out is allowed (in-place rows: a batch is read one iteration before it is written)
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, false>::R, NT = PfaCfg<K, false>::NT;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const buf0 = scr + pfa_scratch<PL, PfaRD<K, false>::v, NT>();  // buffer c at buf0 + c * R * K (stays a shared pointer)
  pfa_load_tables<PL, NT>(tab, gtab);
  const long long nb = (nrows + R - 1) / R;
  auto issue = [&](long long bt, double2* X) {
    const long long r0 = bt * R;
#if SCV_EXP_ROWS_NOIO
    if (bt >= 0) { cp_async_commit(); return; }  // timing experiment only: no loads
#endif
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, n = i - r * K;
      const int xi = r * K + pfa_in_tab<PL>(tab, n);
      if (r0 + r < nrows) {
        if constexpr (GATHER == 2) {
          constexpr int NPR = (K + 1) / 2;
          const long long ri = r0 + r, bb = ri / K, g = ri - bb * K;
          cp_async16(X + xi, in + ((bb * NPR + (n >> 1)) * K + g) * 2 + (n & 1));
        } else {
          cp_async16(X + xi, in + (r0 + r) * K + n);
        }
      } else {
        X[xi] = make_double2(0.0, 0.0);
      }
    }
    cp_async_commit();
  };
  constexpr int NBUF = PfaNBuf<K, false>::v;
  long long bt = blockIdx.x;
  int cur = 0;
  if (NBUF == 2 && bt < nb) issue(bt, buf0);
#pragma unroll 1
  for (; bt < nb; bt += gridDim.x) {
    if constexpr (NBUF == 2) {
      const long long nx = bt + gridDim.x;
      if (nx < nb) issue(nx, buf0 + (cur ^ 1) * (R * K));
      else cp_async_commit();
      cp_async_wait<1>();
    } else {
      issue(bt, buf0);
      cp_async_wait<0>();
    }
    __syncthreads();
    double2* X = buf0 + cur * (R * K);
    pfa_dft_rows<PL, DIR, R, PfaRD<K, false>::v, NT>(X, tab, scr);
    const long long r0 = bt * R;
#if SCV_EXP_ROWS_NOIO
    if (threadIdx.x == 0 && X[0].x == 12345.678) out[r0 * K] = X[1];  // timing experiment only: no stores
#else
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, k = i - r * K;
      if (r0 + r < nrows) {
        if constexpr (GATHER == 2) {
          const long long ri = r0 + r, bb = ri / K, g = ri - bb * K;
          out[(g * LK + b0 + bb) * K + k] = X[r * K + pfa_pos_tab<PL>(tab, k)];
        } else {
          out[(r0 + r) * K + k] = X[r * K + pfa_pos_tab<PL>(tab, k)];
        }
      }
    }
#endif
    __syncthreads();
    if (NBUF == 2) cur ^= 1;
  }
}

// ---------------------------------------------------------------------------
// batched rows, warp-group variant: the CTA holds ONE copy of the tables and
// NG independent groups of NTG threads, each owning a row buffer and a named
// barrier (bar.sync 1+g).  A group loads its row (cp.async), runs the stages
// with group-local barriers and stores it; groups drift apart, so one group's
// load / store phase overlaps the others' DMMA stages without CTA-wide
// barriers (vs k_pfa_rows: 2 CTAs per SM, each CTA-synchronised, tables
// duplicated per CTA).
// ---------------------------------------------------------------------------
#ifndef SCV_EXP_ROWS_NOIO
#define SCV_EXP_ROWS_NOIO 0
#endif
#ifndef SCV_ROWS_NG
#define SCV_ROWS_NG 4
#endif
#ifndef SCV_ROWS_NTG
#define SCV_ROWS_NTG 96
#endif
#ifndef SCV_ROWS_GRP
#define SCV_ROWS_GRP SCV_ROWS_NG, SCV_ROWS_NTG
#endif
template <int K> struct PfaGrpCfg { static constexpr int NG = 0, NTG = 0; };
#define SCV_RGCFG_(KK, ...)                                  \
  template <> struct PfaGrpCfg<KK> {                         \
    static constexpr int v_[2] = {__VA_ARGS__};              \
    static constexpr int NG = v_[0], NTG = v_[1];            \
  };
SCV_RGCFG_(2047, SCV_ROWS_GRP)
// (K = 4095 keeps k_pfa_rows: its all-register DFMA stages for radices 5 and 7
// spill in 128-thread groups)
#ifndef SCV_ROWS_GRP_1023
#define SCV_ROWS_GRP_1023 0, 0
#endif
SCV_RGCFG_(1023, SCV_ROWS_GRP_1023)
template <int K>
static constexpr size_t pfa_smem_grp() {
  using PL = PfaPlan<K>;
  return ((size_t)pfa_tab_total<PL>() + (size_t)PfaGrpCfg<K>::NG * K) * sizeof(double2);
}

// GATHER = 1 (synthesis alpha): row r = bb*K + g of the launch reads the
// input row (g, b0 + bb) of a (K, lsig, K) signal, i.e. in + g*lsig*K +
// (b0+bb)*K, and writes chunk row r (the [bb][g][m] beta chunk).
// GATHER = 2 (analysis alpha from the beta-block scratch of k_ana_colgen_s in
// T mode): row r = bb*K + g reads column pairs T[bb][m/2][g][m&1] (32-byte
// pieces) and writes the signal row (g, bs0 + bb) of a (K, LK/K... ) slab:
// out + (g*snb + bs0 + bb)*K, snb = LK.
template <int K, int DIR, int GATHER>
__global__ void __launch_bounds__(PfaGrpCfg<K>::NG * PfaGrpCfg<K>::NTG, 1)
    k_pfa_rows_g(long long nrows, const double2* in, double2* out, const double2* __restrict__ gtab,
                 long long LK = 0, int b0 = 0) {
  using PL = PfaPlan<K>;
  constexpr int NG = PfaGrpCfg<K>::NG, NTG = PfaGrpCfg<K>::NTG;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  pfa_load_tables<PL, NG * NTG>(tab, gtab);
  const int g = threadIdx.x / NTG, gtid = threadIdx.x - g * NTG, bar = 1 + g;
  double2* const X = sm + pfa_tab_total<PL>() + g * K;
  if constexpr (GATHER >= 3) {
    // real paths: two real rows per complex transform (row pairs 2p, 2p+1)
    constexpr int L = (K + 1) / 2;
    const long long npair = (nrows + 1) / 2;
#pragma unroll 1
    for (long long pr = (long long)blockIdx.x * NG + g; pr < npair; pr += (long long)gridDim.x * NG) {
      const long long r1 = 2 * pr, r2 = r1 + 1;
      const bool has2 = r2 < nrows;
      if constexpr (GATHER == 3) {
        // synthesis alpha of a real signal: X = f1 + i f2 (rows (g, b0+bb) of a (K, LK/K, K) real signal)
        const double* F = (const double*)in;
        const long long bb1 = r1 / K, g1 = r1 - bb1 * K, bb2 = r2 / K, g2 = r2 - bb2 * K;
        const double* s1 = F + g1 * LK + (b0 + bb1) * K;
        const double* s2 = F + g2 * LK + (b0 + bb2) * K;
#pragma unroll 4
        for (int n = gtid; n < K; n += NTG) {
          double* xd = (double*)(X + pfa_in_tab<PL>(tab, n));
          cp_async8(xd, s1 + n);
          if (has2) cp_async8(xd + 1, s2 + n);
          else xd[1] = 0.0;
        }
        cp_async_commit();
        cp_async_wait<0>();
      } else {
        // analysis alpha of a real signal from its half spectrum T (nrows, L):
        // Z = T1 + i T2 extended by Z[-m] = conj(T1[m]) + i conj(T2[m]); Im of m = 0 dropped
        const double2* T1 = in + r1 * L;
        const double2* T2 = in + r2 * L;
#pragma unroll 4
        for (int m = gtid; m < L; m += NTG) {
          double2 t1 = T1[m];
          double2 t2 = has2 ? T2[m] : make_double2(0.0, 0.0);
          if (m == 0) {
            t1.y = 0.0;
            t2.y = 0.0;
          }
          X[pfa_in_tab<PL>(tab, m)] = make_double2(t1.x - t2.y, t1.y + t2.x);
          if (m > 0) X[pfa_in_tab<PL>(tab, K - m)] = make_double2(t1.x + t2.y, -t1.y + t2.x);
        }
      }
      grp_sync(bar, NTG);
      pfa_dft<PL, DIR, 1, NTG, K>(X, tab, nullptr, gtid, bar);
      if constexpr (GATHER == 3) {
        // X1[m] = (Z[m] + conj Z[-m])/2, X2[m] = (Z[m] - conj Z[-m])/(2i), m >= 0 half only
        double2* d1 = out + r1 * K;
        double2* d2 = out + r2 * K;
#pragma unroll 4
        for (int m = gtid; m < L; m += NTG) {
          const double2 z = X[pfa_pos_tab<PL>(tab, m)];
          const double2 zc = X[pfa_pos_tab<PL>(tab, m == 0 ? 0 : K - m)];
          d1[m] = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
          if (has2) d2[m] = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
        }
      } else {
        double* o1 = (double*)out + r1 * K;
        double* o2 = (double*)out + r2 * K;
#pragma unroll 4
        for (int a = gtid; a < K; a += NTG) {
          const double2 z = X[pfa_pos_tab<PL>(tab, a)];
          o1[a] = z.x;
          if (has2) o2[a] = z.y;
        }
      }
      grp_sync(bar, NTG);
    }
    return;
  }
#pragma unroll 1
  for (long long r = (long long)blockIdx.x * NG + g; r < nrows; r += (long long)gridDim.x * NG) {
    const double2* src;
    double2* dst = out + r * K;
    if constexpr (GATHER == 2) {
      constexpr int NPR = (K + 1) / 2;
      const long long bb = r / K, g = r - bb * K;
      src = in + (bb * NPR * K + g) * 2;  // + (m/2)*2K + (m&1)
      dst = out + (g * LK + b0 + bb) * K;
#pragma unroll 4
      for (int n = gtid; n < K; n += NTG) cp_async16(X + pfa_in_tab<PL>(tab, n), src + (long long)(n >> 1) * (2 * K) + (n & 1));
    } else {
      if constexpr (GATHER == 1) {
        const long long bb = r / K, g = r - bb * K;
        src = in + g * LK + (b0 + bb) * K;
      } else {
        src = in + r * K;
      }
      constexpr int KLD = SCV_EXP_ROWS_NOIO ? 0 : K;  // timing experiment only: no loads
#pragma unroll 4
      for (int n = gtid; n < KLD; n += NTG) cp_async16(X + pfa_in_tab<PL>(tab, n), src + n);
    }
    cp_async_commit();
    cp_async_wait<0>();
    grp_sync(bar, NTG);
    pfa_dft<PL, DIR, 1, NTG, K>(X, tab, nullptr, gtid, bar);
#if SCV_EXP_ROWS_NOIO
    if (gtid == 0 && X[0].x == 12345.678) dst[0] = X[1];  // timing experiment only: no stores
#else
#pragma unroll 4
    for (int k = gtid; k < K; k += NTG) dst[k] = X[pfa_pos_tab<PL>(tab, k)];
#endif
    grp_sync(bar, NTG);
  }
}

// ---------------------------------------------------------------------------
// batched rows, pipelined variant (r02): the transform groups of k_pfa_rows_g
// never touch global memory.  The CTA has NG transform groups of NTG threads,
// NIO load/store warps and a ring of NB > NG row buffers.  Step i of the CTA's
// row sequence uses buffer i % NB and transform group i % NG; load/store warp
// i % NIO first writes out the row that was transformed in that buffer NB
// steps earlier, then streams row i in with cp.async.  Two mbarriers per
// buffer order the hand-overs: `full` (32 cp.async-completion arrivals of the
// loading warp -> the transform group) and `done` (one arrival after the
// group's last stage barrier -> the storing warp).  A dependency of step i
// always points to a smaller step and every warp walks its steps in order, so
// the ring cannot deadlock.  With NB - NG rows in flight beyond the ones being
// transformed, the DRAM latency of a row's load and the issue slots of the
// permuted copies no longer sit on the transform warps' critical path
// (k_pfa_rows_g measured 2.96 ms per 131008 rows with, 2.03 ms without its
// global traffic, profiles/r02c_rows_stage_experiments.txt).
// GATHER = 0 / 1 / 2 as in k_pfa_rows_g (the real-signal modes stay there).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// suspend-time hint of a waiting thread (ns): a short hint makes the waiters
// poll, and their polling shows up as a quarter of all executed instructions
#ifndef SCV_MBAR_SUSPEND_NS
#define SCV_MBAR_SUSPEND_NS 20000
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned ok;
  do {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(SCV_MBAR_SUSPEND_NS)
        : "memory");
  } while (!ok);
}
// arrive on `bar` once all cp.async of this thread issued so far have landed
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async16_m(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
// Ring-slot copies of the load/store warps, in batches of RB elements per lane:
// all position-map reads of a batch first, then the data moves.  (The copies
// are asm volatile / cross address spaces the compiler cannot disambiguate, so
// an element-at-a-time loop serialises map read -> copy -> next map read.)
constexpr int RB = 8;
// Pacing (ns) of the load/store warps' copies: a burst of warp-wide copies to scattered slot
// positions delays the transform warps' own shared-memory traffic; sleeping between copies
// spreads it (the load/store warps have slack).  SCV_RING_PACE after every SCV_RING_PACE_N
// fill copies, SCV_RING_PACE_D after every batch of RB drain reads.
// Measured on the C4 map (ms of the two row passes): off 84.3 / 83.7; 20 ns per 2 copies
// 82.4 / 82.2; 20 ns per copy 82.6 / 82.9; 50 ns per 3 copies 82.7 / 82.7; 50 ns per copy
// 91 / 85 (the load/store warps then bound the kernel); drain pacing 200 ns per batch 84.5 / 83.8.
#ifndef SCV_RING_PACE
#define SCV_RING_PACE 20
#endif
#ifndef SCV_RING_PACE_N
#define SCV_RING_PACE_N 2
#endif
#ifndef SCV_RING_PACE_D
#define SCV_RING_PACE_D 0
#endif
// slot X (Ruritanian positions) <- element n of a row at gsrc(n), n = lane0 + nl*j < K
template <class PL, int RB = ::RB, class SrcFn>
__device__ __forceinline__ void ring_fill(double2* X, const double2* tab, int lane0, int nl, SrcFn gsrc) {
  constexpr int K = PL::K;
#pragma unroll 1
  for (int n0 = lane0; n0 < K; n0 += nl * RB) {
    int pos[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int n = n0 + nl * j;
      pos[j] = n < K ? pfa_in_tab<PL>(tab, n) : 0;
    }
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int n = n0 + nl * j;
      if (n < K) cp_async16_m(X + pos[j], gsrc(n));
#if SCV_RING_PACE
      if ((j % SCV_RING_PACE_N) == SCV_RING_PACE_N - 1) __nanosleep(SCV_RING_PACE);
#endif
    }
  }
}
// output frequency k of slot X -> gdst(k), k = lane0 + nl*j < K
template <class PL, int RB = ::RB, class DstFn>
__device__ __forceinline__ void ring_drain(const double2* X, const double2* tab, int lane0, int nl, DstFn gdst) {
  constexpr int K = PL::K;
#pragma unroll 1
  for (int k0 = lane0; k0 < K; k0 += nl * RB) {
    int pos[RB];
    double2 v[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int k = k0 + nl * j;
      pos[j] = k < K ? pfa_pos_tab<PL>(tab, k) : 0;
    }
#pragma unroll
    for (int j = 0; j < RB; ++j) v[j] = X[pos[j]];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int k = k0 + nl * j;
      if (k < K) *gdst(k) = v[j];
    }
#if SCV_RING_PACE_D
    __nanosleep(SCV_RING_PACE_D);
#endif
  }
}

// The same copies through the lane schedule (scv_pfa_tables_sched): entry [32 j + lane] =
// position | e << 11, the lane moves element 32 j + e.  A full warp only (32 consecutive
// elements per copy instruction).
template <class PL, class SrcFn>
__device__ __forceinline__ void ring_fill_s(double2* X, const double2* tab, int lane, SrcFn gsrc) {
  constexpr int K = PL::K;
  const unsigned short* map = (const unsigned short*)(tab + pfa_rtab_total<PL>()) + K;
#pragma unroll 1
  for (int n0 = 0; n0 < K; n0 += 32 * RB) {
    unsigned en[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int i = n0 + 32 * j + lane;
      en[j] = i < K ? map[i] : (31u << 11);
    }
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int n = n0 + 32 * j + (int)(en[j] >> 11);
      if (n < K) cp_async16_m(X + (en[j] & 0x7ffu), gsrc(n));
#if SCV_RING_PACE
      if ((j % SCV_RING_PACE_N) == SCV_RING_PACE_N - 1) __nanosleep(SCV_RING_PACE);
#endif
    }
  }
}
template <class PL, class DstFn>
__device__ __forceinline__ void ring_drain_s(const double2* X, const double2* tab, int lane, DstFn gdst) {
  constexpr int K = PL::K;
  const unsigned short* map = (const unsigned short*)(tab + pfa_rtab_total<PL>());
#pragma unroll 1
  for (int k0 = 0; k0 < K; k0 += 32 * RB) {
    unsigned en[RB];
    double2 v[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int i = k0 + 32 * j + lane;
      en[j] = i < K ? map[i] : (31u << 11);
    }
#pragma unroll
    for (int j = 0; j < RB; ++j) v[j] = X[en[j] & 0x7ffu];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int k = k0 + 32 * j + (int)(en[j] >> 11);
      if (k < K) *gdst(k) = v[j];
    }
  }
}

// Pipeline timing counters (debug builds, -DSCV_PIPE_STATS=1): clock64 sums per
// role, [kernel kind * 6 + {0 transform wait-full, 1 transform, 2 io wait-done,
// 3 io drain, 4 io fill, 5 CTA lifetime}]; read with scv_debug_pipe_stats.
#ifndef SCV_PIPE_STATS
#define SCV_PIPE_STATS 0
#endif
__device__ unsigned long long g_pipe_stats[36];
__device__ __forceinline__ long long pipe_now() {
#if defined(__CUDA_ARCH__) && SCV_PIPE_STATS
  return clock64();
#else
  return 0;
#endif
}
struct PipeClk {
  long long t;
  __device__ __forceinline__ PipeClk() : t(pipe_now()) {}
  // add the time since the last mark to counter `idx` (kept in `acc`)
  __device__ __forceinline__ void mark(long long (&acc)[6], int idx) {
    if (SCV_PIPE_STATS) {
      const long long n = pipe_now();
      acc[idx] += n - t;
      t = n;
    }
  }
};
__device__ __forceinline__ void pipe_flush(const long long (&acc)[6], int kind, bool leader) {
  if (SCV_PIPE_STATS && leader)
    for (int i = 0; i < 6; ++i)
      if (acc[i]) atomicAdd(&g_pipe_stats[kind * 6 + i], (unsigned long long)acc[i]);
}
extern "C" int scv_debug_pipe_stats(unsigned long long* out, int reset) {
  if (out && cudaMemcpyFromSymbol(out, g_pipe_stats, sizeof(g_pipe_stats)) != cudaSuccess) return SCV_ECUDA;
  if (reset) {
    unsigned long long z[36] = {0};
    if (cudaMemcpyToSymbol(g_pipe_stats, z, sizeof(z)) != cudaSuccess) return SCV_ECUDA;
  }
  return SCV_OK;
}

#ifndef SCV_ROWSP
#define SCV_ROWSP 1
#endif
// register split (setmaxnreg 152 / 120) in the K = 1023 column kernels too: its three-stage
// transform (3 * 11 * 31) wanted all 128 registers, the two-stage one (SCV_PLAN_1023) does not
#ifndef SCV_SETREG_1023
#define SCV_SETREG_1023 0
#endif
#ifndef SCV_ROWSP_NG
#define SCV_ROWSP_NG 4
#endif
#ifndef SCV_ROWSP_NIO
#define SCV_ROWSP_NIO 3
#endif
#ifndef SCV_ROWSP_NB
#define SCV_ROWSP_NB 6
#endif
// lane-scheduled slot copies in the row kernel (see pfa_lane_schedule); the transposed-chunk
// mode 5 walks the plain maps
// Measured (r02t, r02x): bit-identical, 7.3 instead of 10.4 shared-memory wavefronts per copy,
// and 2.5 ms/map SLOWER per row pass, with or without pacing (84.5 vs 82.0).  A 16-byte warp
// access is served quarter-warp by quarter-warp; in natural lane order a quarter covers one
// 128-byte line of global memory, scheduled it touches up to four, so what the shared side
// saves the global side loses.  Off.
#ifndef SCV_ROWSP_SCHED
#define SCV_ROWSP_SCHED 0
#endif
constexpr bool pfa_rows_sched(int gather) { return SCV_ROWSP_SCHED && gather != 5; }
// XW / XS: blocks per warp iteration of the Rader-89 and radix-23 stages in the row kernel's
// transform groups (pfa.cuh).  The K = 2047 shape can trade a transform group for registers.
#ifndef SCV_ROWSP_NG_2047
#define SCV_ROWSP_NG_2047 SCV_ROWSP_NG
#endif
// Register split of the K = 2047 row kernel (setmaxnreg, whole warpgroups): SCV_ROWSP_SETREG_T
// registers per transform thread (0 = no split), SCV_ROWSP_SETREG_IO per load/store thread; the
// load/store warps are then padded to one warpgroup (the pad warp exits), and their copy
// batches shrink to SCV_ROWSP_RB elements per lane.  The split only moves registers inside
// the CTA's launch allocation (threads x launch registers): threads(T) x T + 128 x IO must not
// exceed it, or setmaxnreg.inc waits for ever (640 threads launch at 96: T <= 112 with IO = 32).
// Measured at C4 (r07q/r07r, ms per row pass, default 80.5 / 79.4): 4 groups of 4 warps at
// 112 / 32 registers 83.9 / 84.2; 4 groups of 3 warps at 160 / 32 or 152 / 40 with two Rader
// blocks per iteration (SCV_ROWSP_XW=2; 72-92 bytes of spills) 92.7 / 92.5 and 89.2 / 90.5.  Off.
#ifndef SCV_ROWSP_SETREG_T
#define SCV_ROWSP_SETREG_T 0
#endif
#ifndef SCV_ROWSP_SETREG_IO
#define SCV_ROWSP_SETREG_IO 32
#endif
#ifndef SCV_ROWSP_RB
#define SCV_ROWSP_RB 4
#endif
#ifndef SCV_ROWSP_XW
#define SCV_ROWSP_XW SCV_R89_NBW
#endif
#ifndef SCV_ROWSP_XS
#define SCV_ROWSP_XS SCV_PFA_NBW_SMALL
#endif
template <int K> struct PfaPipeCfg {
  static constexpr int NG = 0, NTG = 96, NIO = 0, NB = 0, XW = SCV_R89_NBW, XS = SCV_PFA_NBW_SMALL;
};
// threads of a row-kernel launch: with the register split the load/store warps fill a warpgroup
template <int K> constexpr int pfa_pipe_setreg() { return K == 2047 ? SCV_ROWSP_SETREG_T : 0; }
template <class C, int K> constexpr int pfa_pipe_threads() {
  return C::NG * C::NTG + (pfa_pipe_setreg<K>() ? 128 : C::NIO * 32);
}
#ifndef SCV_ROWSP_NTG
#define SCV_ROWSP_NTG 96
#endif
#ifndef SCV_ROWSP_NTG_2047
#define SCV_ROWSP_NTG_2047 SCV_ROWSP_NTG
#endif
template <> struct PfaPipeCfg<2047> {
  static constexpr int NG = SCV_ROWSP ? SCV_ROWSP_NG_2047 : 0, NTG = SCV_ROWSP_NTG_2047, NIO = SCV_ROWSP_NIO, NB = SCV_ROWSP_NB;
  static constexpr int XW = SCV_ROWSP_XW, XS = SCV_ROWSP_XS;
};
// K = 1023 (the L_j = 512 scale): on with SCV_RING_1023
#ifndef SCV_RING_1023
#define SCV_RING_1023 1
#endif
template <> struct PfaPipeCfg<1023> {
  static constexpr int NG = SCV_RING_1023 ? SCV_ROWSP_NG : 0, NTG = SCV_ROWSP_NTG, NIO = SCV_ROWSP_NIO, NB = SCV_ROWSP_NB;
  static constexpr int XW = SCV_R89_NBW, XS = SCV_PFA_NBW_SMALL;
};
// K = 511 (the L_j = 256 scale): row kernel and gamma+quadrature as ring kernels (SCV_RING_511);
// its column generation keeps the batched kernel (8 degrees per generator lane < one batch)
#ifndef SCV_RING_511
#define SCV_RING_511 1
#endif
template <> struct PfaPipeCfg<511> {
  static constexpr int NG = SCV_RING_511 ? SCV_ROWSP_NG : 0, NTG = SCV_ROWSP_NTG, NIO = SCV_ROWSP_NIO, NB = SCV_ROWSP_NB;
  static constexpr int XW = SCV_R89_NBW, XS = SCV_PFA_NBW_SMALL;
};
// K = 4095 (the L_j = 2048 scales of C5): a slot is 64 KB, so the ring has 3 slots and 2
// transform groups (SCV_RING_4095 = NTG threads per group, 0 = off).  Measured on the C5
// streamed map (ms/map; the four-radix transform spills at every shape): off 5472, 128
// threads per group 5458, 192: 5738, 256: 5391.
#ifndef SCV_RING_4095
#define SCV_RING_4095 256
#endif
template <> struct PfaPipeCfg<4095> {
  static constexpr int NG = SCV_RING_4095 ? 2 : 0, NTG = SCV_RING_4095 ? SCV_RING_4095 : 96, NIO = 3, NB = 3;
  static constexpr int XW = SCV_R89_NBW, XS = SCV_PFA_NBW_SMALL;
};
template <int K>
static constexpr size_t pfa_smem_pipe() {
  using PL = PfaPlan<K>;
  return ((size_t)pfa_tab_total<PL>() + (size_t)PfaPipeCfg<K>::NB * K) * sizeof(double2) +
         4 * (size_t)PfaPipeCfg<K>::NB * sizeof(unsigned long long);
}

template <int K, int DIR, int GATHER>
__global__ void __launch_bounds__(pfa_pipe_threads<PfaPipeCfg<K>, K>(), 1)
    k_pfa_rows_p(long long nrows, const double2* in, double2* out, const double2* __restrict__ gtab,
                 long long LK = 0, int b0 = 0) {
  using PL = PfaPlan<K>;
  constexpr int NG = PfaPipeCfg<K>::NG, NTG = PfaPipeCfg<K>::NTG, NIO = PfaPipeCfg<K>::NIO, NB = PfaPipeCfg<K>::NB;
  constexpr int NT = pfa_pipe_threads<PfaPipeCfg<K>, K>();
  constexpr int SETREG = pfa_pipe_setreg<K>();
  constexpr int IORB = SETREG ? SCV_ROWSP_RB : RB;
  static_assert(!SETREG || ((NG * NTG) % 128 == 0 && NIO <= 4), "setmaxnreg works on warpgroups of 128 threads");
  static_assert(NB > NG, "the ring needs spare buffers for the rows in flight");
  constexpr bool SCHED = pfa_rows_sched(GATHER);  // gtab then is scv_pfa_tables_sched's
  static_assert(NB % NIO == 0, "a load/store warp owns fixed ring slots (it then meets a slot's barrier phases in order)");
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const bufs = sm + pfa_tab_total<PL>();
  // two barriers per slot and kind, used by alternate laps (use u of a slot ->
  // barrier u & 1, parity (u >> 1) & 1): an mbarrier parity wait cannot tell the
  // phase it wants from the one two phases earlier, and a transform group that
  // rotates over the slots can be one use ahead of a slot's producer
  unsigned long long* const full = (unsigned long long*)(bufs + (size_t)NB * K);
  unsigned long long* const done = full + 2 * NB;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2 * NB; ++b) {
      mbar_init(full + b, 32);
      mbar_init(done + b, 1);
    }
  }
  pfa_load_tables<PL, NT>(tab, gtab);  // ends with __syncthreads: the barriers are initialised for everyone
  // the CTA's row sequence: round q covers NG adjacent rows (adjacent rows of
  // the GATHER = 2 scratch share 128-byte lines), i -> (q = i / NG, slot i % NG)
  const long long G = gridDim.x;
  const long long rem = nrows - (long long)blockIdx.x * NG;
  if (rem <= 0) return;
  const long long qmax = (rem - 1) / (G * NG);
  const long long tail = rem - qmax * G * NG;
  const long long ni = qmax * NG + (tail < NG ? tail : NG);
  auto row_of = [&](long long i) { return (i / NG) * (G * NG) + (long long)blockIdx.x * NG + (i % NG); };
  if (threadIdx.x >= NG * NTG) {
    // ---- load / store warps
    if constexpr (SETREG != 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(SCV_ROWSP_SETREG_IO));
    const int w = (threadIdx.x - NG * NTG) >> 5, lane = threadIdx.x & 31;
    if (SETREG != 0 && w >= NIO) return;  // pad warp of the load/store warpgroup
    long long st[6] = {0, 0, 0, 0, 0, 0};
    PipeClk ck;
    if constexpr (GATHER == 5) {
      // Synthesis alpha pass into the TRANSPOSED chunk C[m][r] (r = the launch's flat row
      // index bb * K + g, row pitch RS even): the gamma+quadrature pass then streams a
      // column (m, bb) as 2047 contiguous elements instead of 16-byte pieces 32 KB apart
      // (half-used sectors, twice the L2 -> SM traffic).  A warp drains the two slots of
      // rows (r, r + 1), r even, together: lane pair (2i, 2i+1) writes C[k][r], C[k][r+1],
      // one full 32-byte sector.  Steps 2j and 2j + 1 of a CTA are such a row pair
      // (rounds of NG = 4 adjacent rows), in slots 2(j % (NB/2)) and + 1 of the same lap.
      static_assert(GATHER != 5 || (NG % 2 == 0 && NB % 2 == 0 && (NB / 2) % NIO == 0),
                    "row pairs share a round and a lap; a warp owns fixed slot pairs");
      const long long RS = (nrows + 1) & ~1LL;
      const int sub = lane & 1;
#pragma unroll 1
      for (long long i0 = 2 * w; i0 < ni + NB; i0 += 2 * NIO) {
        const int b = (int)(i0 % NB);
        const unsigned u = (unsigned)(i0 / NB);
        double2* const X0 = bufs + (size_t)b * K;
        ck.mark(st, 4);
        if (i0 >= NB) {
          const bool have1 = i0 - NB + 1 < ni;
          mbar_wait(done + ((u - 1) & 1) * NB + b, ((u - 1) >> 1) & 1);
          if (have1) mbar_wait(done + ((u - 1) & 1) * NB + b + 1, ((u - 1) >> 1) & 1);
          ck.mark(st, 2);
          const long long r = row_of(i0 - NB);
          double2* const dst = out + r + sub;
          const double2* const Xs = X0 + (size_t)sub * K;
          if (sub == 0 || have1) {
#pragma unroll 1
            for (int k0 = lane >> 1; k0 < K; k0 += 16 * RB) {
              int pos[RB];
              double2 v[RB];
#pragma unroll
              for (int j = 0; j < RB; ++j) {
                const int k = k0 + 16 * j;
                pos[j] = k < K ? pfa_pos_tab<PL>(tab, k) : 0;
              }
#pragma unroll
              for (int j = 0; j < RB; ++j) v[j] = Xs[pos[j]];
#pragma unroll
              for (int j = 0; j < RB; ++j) {
                const int k = k0 + 16 * j;
                if (k < K) dst[(long long)k * RS] = v[j];
              }
            }
          }
          __syncwarp();  // every lane has read its elements before any lane refills the buffers
          ck.mark(st, 3);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long long i = i0 + h;
          if (i < ni) {
            const long long r = row_of(i);
            const long long bb = r / K, g = r - bb * K;
            const double2* src = in + g * LK + (b0 + bb) * K;
            ring_fill<PL>(X0 + (size_t)h * K, tab, lane, 32, [&](int n) { return src + n; });
            cp_async_mbar_arrive(full + (u & 1) * NB + b + h);
          }
        }
      }
      ck.mark(st, 4);
      pipe_flush(st, 0, lane == 0);
      return;
    }
#pragma unroll 1
    for (long long i = w; i < ni + NB; i += NIO) {
      const int b = (int)(i % NB);
      const unsigned u = (unsigned)(i / NB);
      double2* const X = bufs + (size_t)b * K;
      ck.mark(st, 4);
      if (i >= NB) {
        // row i - NB was transformed in this buffer: write it out
        mbar_wait(done + ((u - 1) & 1) * NB + b, ((u - 1) >> 1) & 1);
        ck.mark(st, 2);
        const long long r = row_of(i - NB);
        double2* dst = out + r * K;
        if constexpr (GATHER == 2) {
          const long long bb = r / K, g = r - bb * K;
          dst = out + (g * LK + b0 + bb) * K;
        }
          if constexpr (SCHED) ring_drain_s<PL>(X, tab, lane, [&](int k) { return dst + k; });
        else ring_drain<PL, IORB>(X, tab, lane, 32, [&](int k) { return dst + k; });
        __syncwarp();  // every lane has read its elements before any lane refills the buffer
        ck.mark(st, 3);
      }
      if (i < ni) {
        const long long r = row_of(i);
        if constexpr (GATHER == 2) {
          constexpr int NPR = (K + 1) / 2;
          const long long bb = r / K, g = r - bb * K;
          const double2* src = in + (bb * NPR * K + g) * 2;  // + (m/2)*2K + (m&1)
          if constexpr (SCHED)
            ring_fill_s<PL>(X, tab, lane, [&](int n) { return src + (long long)(n >> 1) * (2 * K) + (n & 1); });
          else
            ring_fill<PL, IORB>(X, tab, lane, 32, [&](int n) { return src + (long long)(n >> 1) * (2 * K) + (n & 1); });
        } else {
          const double2* src = in + r * K;
          if constexpr (GATHER == 1 || GATHER == 5) {
            const long long bb = r / K, g = r - bb * K;
            src = in + g * LK + (b0 + bb) * K;
          }
          if constexpr (SCHED) ring_fill_s<PL>(X, tab, lane, [&](int n) { return src + n; });
          else ring_fill<PL, IORB>(X, tab, lane, 32, [&](int n) { return src + n; });
        }
        cp_async_mbar_arrive(full + (u & 1) * NB + b);
      }
    }
    ck.mark(st, 4);
    pipe_flush(st, 0, lane == 0);
    return;
  }
  // ---- transform groups
  if constexpr (SETREG != 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(SETREG));
  const int g = threadIdx.x / NTG, gtid = threadIdx.x - g * NTG, bar = 1 + g;
  long long st[6] = {0, 0, 0, 0, 0, 0};
  PipeClk ck;
#pragma unroll 1
  for (long long i = g; i < ni; i += NG) {
    const int b = (int)(i % NB);
    const unsigned u = (unsigned)(i / NB);
    mbar_wait(full + (u & 1) * NB + b, (u >> 1) & 1);
    ck.mark(st, 0);
    pfa_dft<PL, DIR, 1, NTG, K, PfaPipeCfg<K>::XW, PfaPipeCfg<K>::XS>(bufs + (size_t)b * K, tab, nullptr, gtid, bar);
    if (gtid == 0) mbar_arrive(done + (u & 1) * NB + b);
    ck.mark(st, 1);
  }
  pipe_flush(st, 0, gtid == 0);
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
  double2* X = scr + pfa_scratch<PL, PfaRD<K, false>::v, NT>();
  int4* rp = (int4*)(X + PfaNBuf<K, false>::v * R * K);  // per-row (gi, b, n, l)
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
      X[r * K + pfa_in_tab<PL>(tab, q)] = v;
    }
    __syncthreads();
    pfa_dft_rows<PL, +1, R, PfaRD<K, false>::v, NT>(X, tab, scr);
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int r = i / K, a = i - r * K;
      const int4 P = rp[r];
      if (P.x >= 0) out[((long long)P.x * L + P.y) * K + a] = X[r * K + pfa_pos_tab<PL>(tab, a)];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// analysis, gamma first (complex path): a task is R adjacent alpha-frequency
// columns m of one beta row b.  The column over the gamma frequency n is
// generated in closed form (nonzero for |m| <= |n|), inverse-transformed over
// n -> gamma, and stored at sig[g][b][m]: R*16-byte segments, written once,
// no reads (adjacent tasks run on adjacent CTAs, so L2 assembles full lines).
// The alpha IDFT then runs over contiguous rows in place (k_pfa_rows), so
// neither pass reads HBM with a stride.
// ---------------------------------------------------------------------------
template <int K> struct PfaGCfg { static constexpr int R = 8, NT = 128, MINB = 2; };
template <> struct PfaGCfg<255> { static constexpr int R = 8, NT = 256, MINB = 1; };
template <> struct PfaGCfg<511> { static constexpr int R = 4, NT = 256, MINB = 1; };
#ifndef SCV_GEN1023
#define SCV_GEN1023 4, 512, 1
#endif
#ifndef SCV_GEN2047
#define SCV_GEN2047 4, 384, 1
#endif
#define SCV_GCFG_(KK, ...)                                  \
  template <> struct PfaGCfg<KK> {                          \
    static constexpr int v_[3] = {__VA_ARGS__};             \
    static constexpr int R = v_[0], NT = v_[1], MINB = v_[2]; \
  };
SCV_GCFG_(1023, SCV_GEN1023)
SCV_GCFG_(2047, SCV_GEN2047)
// (re-swept with the 9 * 13 * 35 plan, r09: 512: 1318 ms; 640: 1282; 768: 1332; 1024: 1285)
#ifndef SCV_GEN4095_NT
#define SCV_GEN4095_NT 640
#endif
template <> struct PfaGCfg<4095> { static constexpr int R = 2, NT = SCV_GEN4095_NT, MINB = 1; };

#ifndef SCV_COLGEN_GU
#define SCV_COLGEN_GU 1
#endif
template <int K>
static constexpr size_t pfa_smem_g() {
  using PL = PfaPlan<K>;
  return ((size_t)PfaGCfg<K>::R * K + pfa_tab_total<PL>() + pfa_scratch<PL, PfaGCfg<K>::R, PfaGCfg<K>::NT>()) *
         sizeof(double2);
}

// TM = 1: beta-block scratch output T[bs][m0/R][g][r] (see k_ana_colgen_s)
template <int K, int TM = 0>
__global__ void __launch_bounds__(PfaGCfg<K>::NT, PfaGCfg<K>::MINB)
    k_ana_colgen(const double2* __restrict__ w, const double* __restrict__ hlb, const double* __restrict__ lsin,
                 const double* __restrict__ lcos, int b0, int nb, double2* __restrict__ out,
                 const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaGCfg<K>::R, NT = PfaGCfg<K>::NT;
  constexpr int L = (K + 1) / 2;
  constexpr int NGRP = (K + R - 1) / R;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const X = scr + pfa_scratch<PL, R, NT>();
  pfa_load_tables<PL, NT>(tab, gtab);
  const double fac0 = 1.0 / (8.0 * SCV_PI * SCV_PI);
  const int ntask = nb * NGRP;
#pragma unroll 1
  for (int task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int bs = task / NGRP;  // beta row within the slab
    const int b = b0 + bs;
    const int m0 = (task - bs * NGRP) * R;
    const double ls = lsin[b], lc = lcos[b];
    // generation: a thread owns one gamma frequency n (row gi of the R
    // columns), so the n-dependent index math is shared by the R columns and
    // the coefficient reads of consecutive m are contiguous (hlb row l,
    // w row (sheet, l)); batches of GU rows issue all gathers before use
    constexpr int NPT = (K + NT - 1) / NT, GU = K >= 2047 ? SCV_COLGEN_GU : 1;
#pragma unroll 1
    for (int i0 = 0; i0 < NPT; i0 += GU) {
      double hv[GU][R];
      double2 cv[GU][R];
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int gi = threadIdx.x + (i0 + u) * NT;
        const int n = gi <= L - 1 ? gi : gi - K;
        const int l = n < 0 ? -n : n;
        const double* hrow = hlb + l * (l + 1) / 2;
        const double2* wrow = w + ((n >= 0 ? 0 : 1) * L + l) * K + (L - 1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int m = m0 + r <= L - 1 ? m0 + r : m0 + r - K, am = m < 0 ? -m : m;
          hv[u][r] = 0.0;
          cv[u][r] = make_double2(0.0, 0.0);
          if (i0 + u < NPT && gi < K && m0 + r < K && am <= l) {
            hv[u][r] = hrow[am];
            cv[u][r] = wrow[m];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int gi = threadIdx.x + (i0 + u) * NT;
        if (i0 + u >= NPT || gi >= K) continue;
        const int n = gi <= L - 1 ? gi : gi - K;
        const int l = n < 0 ? -n : n;
        const double facl = (double)(2 * l + 1) * fac0;
        const int xi = pfa_in_tab<PL>(tab, gi);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int m = m0 + r <= L - 1 ? m0 + r : m0 + r - K, am = m < 0 ? -m : m;
          double2 v = make_double2(0.0, 0.0);
          if (m0 + r < K && am <= l) {
            const int es = n >= 0 ? l - m : l + m;  // power of sin(b/2)
            const int ec = n >= 0 ? l + m : l - m;  // power of cos(b/2)
            double lg = hv[u][r];
            if (es) lg += (double)es * ls;
            if (ec) lg += (double)ec * lc;
            double d = exp(lg);
            if (n < 0 && ((l - m) & 1)) d = -d;
            const double f = facl * d;
            v = make_double2(f * cv[u][r].x, f * cv[u][r].y);
          }
          X[r * K + xi] = v;
        }
      }
    }
    __syncthreads();
    pfa_dft<PL, +1, R, NT, K>(X, tab, scr);
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int g = i / R, r = i - g * R;
      const int mi = m0 + r;
#if SCV_EXP_COLGEN_CONTIG
      if (mi < K) out[(((long long)task * R + r) * K + g) % ((long long)nb * K * K)] = X[r * K + pfa_pos_tab<PL>(tab, g)];  // timing experiment only
#else
      if constexpr (TM) out[(((long long)bs * NGRP + m0 / R) * K + g) * R + r] = X[r * K + pfa_pos_tab<PL>(tab, g)];
      else if (mi < K) out[((long long)g * nb + bs) * K + mi] = X[r * K + pfa_pos_tab<PL>(tab, g)];
#endif
    }
    __syncthreads();
  }
}

// Variant with the generation coefficients staged in shared memory: a task
// is (beta block of BB rows, group of R adjacent m); the R columns'
// coefficients w[sheet][l][m] and hlb[l][|m|] are read from L2 once per task
// into shared memory and reused for the BB rows, so the per-row generation
// has no global loads.  (SCV_COLGEN_S=1 selects it for K = 2047.)
template <int K> struct PfaSCfg { static constexpr int R = 2, NT = 384, MINB = 1, BB = 16; };
#ifndef SCV_COLGEN_S
#define SCV_COLGEN_S 1
#endif
#ifndef SCV_COLGEN_S_BB
#define SCV_COLGEN_S_BB 128
#endif
#ifndef SCV_COLGEN_S_NT
#define SCV_COLGEN_S_NT 384
#endif
template <> struct PfaSCfg<2047> { static constexpr int R = 2, NT = SCV_COLGEN_S_NT, MINB = 1, BB = SCV_COLGEN_S_BB; };
// NGR > 1: the CTA runs NGR independent groups of NT/NGR threads, group g
// generating and transforming column m0 + g with its own named barrier, so
// one group's generation (exp, coefficient reads) overlaps the other's DMMA
// stages instead of the whole CTA alternating between the two phases.
#ifndef SCV_COLGEN_S_NGR
#define SCV_COLGEN_S_NGR 1
#endif
template <int K>
static constexpr size_t pfa_smem_s() {
  using PL = PfaPlan<K>;
  constexpr int R = PfaSCfg<K>::R;
  return ((size_t)R * K + pfa_tab_total<PL>() + pfa_scratch<PL, R, PfaSCfg<K>::NT>() + (size_t)R * K) *
             sizeof(double2) + (size_t)R * K * sizeof(double);
}

// TM = 1: write the beta-block scratch T[bs][m0/R][g][r] instead of the
// signal (R*K*16 contiguous bytes per task row; k_pfa_rows_g<K, +1, 2> then
// gathers the alpha rows from it and writes the signal).
template <int K, int TM = 0>
__global__ void __launch_bounds__(PfaSCfg<K>::NT, PfaSCfg<K>::MINB)
    k_ana_colgen_s(const double2* __restrict__ w, const double* __restrict__ hlb, const double* __restrict__ lsin,
                   const double* __restrict__ lcos, int b0, int nb, double2* __restrict__ out,
                   const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaSCfg<K>::R, NT = PfaSCfg<K>::NT, BB = PfaSCfg<K>::BB;
  constexpr int L = (K + 1) / 2;
  constexpr int NGRP = (K + R - 1) / R;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const X = scr + pfa_scratch<PL, R, NT>();
  double2* const CW = X + R * K;                 // [gi][r] W_{m,n} (0 where |m| > |n|)
  double* const CH = (double*)(CW + R * K);      // [gi][r] log sqrt C(2l, l+|m|)
  pfa_load_tables<PL, NT>(tab, gtab);
  const double fac0 = 1.0 / (8.0 * SCV_PI * SCV_PI);
  const int nbblk = (nb + BB - 1) / BB;
  const int ntask = nbblk * NGRP;
  constexpr int NPT = (K + NT - 1) / NT;
#pragma unroll 1
  for (int task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int bblk = task / NGRP;
    const int m0 = (task - bblk * NGRP) * R;
    // stage the R columns' coefficients
#pragma unroll
    for (int u = 0; u < NPT; ++u) {
      const int gi = threadIdx.x + u * NT;
      if (gi >= K) continue;
      const int n = gi <= L - 1 ? gi : gi - K;
      const int l = n < 0 ? -n : n;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int m = m0 + r <= L - 1 ? m0 + r : m0 + r - K, am = m < 0 ? -m : m;
        const bool nz = m0 + r < K && am <= l;
        CW[gi * R + r] = nz ? w[((n >= 0 ? 0 : 1) * L + l) * K + (L - 1) + m] : make_double2(0.0, 0.0);
        CH[gi * R + r] = nz ? hlb[l * (l + 1) / 2 + am] : 0.0;
      }
    }
    const int bs_end = min(nb, (bblk + 1) * BB);
    if constexpr (SCV_COLGEN_S_NGR > 1) {
      // group g owns column m0 + g (R == NGR): generation of one group
      // overlaps the other group's transform
      static_assert(R == SCV_COLGEN_S_NGR, "one column per group");
      constexpr int NTG = NT / SCV_COLGEN_S_NGR, NPG = (K + NTG - 1) / NTG;
      const int g = threadIdx.x / NTG, gtid = threadIdx.x - g * NTG, bar = 1 + g;
      double2* const Xg = X + g * K;
      const int mg = m0 + g <= L - 1 ? m0 + g : m0 + g - K, amg = mg < 0 ? -mg : mg;
      __syncthreads();  // coefficients staged
#pragma unroll 1
      for (int bs = bblk * BB; bs < bs_end; ++bs) {
        const int b = b0 + bs;
        const double ls = lsin[b], lc = lcos[b];
#pragma unroll 2
        for (int u = 0; u < NPG; ++u) {
          const int gi = gtid + u * NTG;
          if (gi >= K) continue;
          const int n = gi <= L - 1 ? gi : gi - K;
          const int l = n < 0 ? -n : n;
          double2 v = make_double2(0.0, 0.0);
          if (m0 + g < K && amg <= l) {
            const int es = n >= 0 ? l - mg : l + mg;
            const int ec = n >= 0 ? l + mg : l - mg;
            double lg = CH[gi * R + g];
            if (es) lg += (double)es * ls;
            if (ec) lg += (double)ec * lc;
            double d = exp(lg);
            if (n < 0 && ((l - mg) & 1)) d = -d;
            const double f = (double)(2 * l + 1) * fac0 * d;
            const double2 c = CW[gi * R + g];
            v = make_double2(f * c.x, f * c.y);
          }
          Xg[pfa_in_tab<PL>(tab, gi)] = v;
        }
        grp_sync(bar, NTG);
        pfa_dft<PL, +1, 1, NTG, K>(Xg, tab, scr, gtid, bar);
        if (m0 + g < K) {
#pragma unroll 4
          for (int gg = gtid; gg < K; gg += NTG) out[((long long)gg * nb + bs) * K + m0 + g] = Xg[pfa_pos_tab<PL>(tab, gg)];
        }
        grp_sync(bar, NTG);
      }
      __syncthreads();  // both groups done with CW / CH before restaging
      continue;
    }
#pragma unroll 1
    for (int bs = bblk * BB; bs < bs_end; ++bs) {
      const int b = b0 + bs;
      const double ls = lsin[b], lc = lcos[b];
      __syncthreads();  // coefficients staged / previous row's stores done
#pragma unroll 2
      for (int u = 0; u < NPT; ++u) {
        const int gi = threadIdx.x + u * NT;
        if (gi >= K) continue;
        const int n = gi <= L - 1 ? gi : gi - K;
        const int l = n < 0 ? -n : n;
        const double facl = (double)(2 * l + 1) * fac0;
        const int xi = pfa_in_tab<PL>(tab, gi);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int m = m0 + r <= L - 1 ? m0 + r : m0 + r - K, am = m < 0 ? -m : m;
          double2 v = make_double2(0.0, 0.0);
          if (m0 + r < K && am <= l) {
            const int es = n >= 0 ? l - m : l + m;  // power of sin(b/2)
            const int ec = n >= 0 ? l + m : l - m;  // power of cos(b/2)
            double lg = CH[gi * R + r];
            if (es) lg += (double)es * ls;
            if (ec) lg += (double)ec * lc;
            double d = exp(lg);
            if (n < 0 && ((l - m) & 1)) d = -d;
            const double f = facl * d;
            const double2 c = CW[gi * R + r];
            v = make_double2(f * c.x, f * c.y);
          }
          X[r * K + xi] = v;
        }
      }
      __syncthreads();
      pfa_dft<PL, +1, R, NT, K>(X, tab, scr);
#pragma unroll 4
      for (int i = threadIdx.x; i < R * K; i += NT) {
        const int g = i / R, r = i - g * R;
        const int mi = m0 + r;
        if constexpr (TM) {
          out[(((long long)bs * NGRP + m0 / R) * K + g) * R + r] = X[r * K + pfa_pos_tab<PL>(tab, g)];
        } else {
          if (mi < K) out[((long long)g * nb + bs) * K + mi] = X[r * K + pfa_pos_tab<PL>(tab, g)];
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Pipelined column generation (r02, K = 2047): the analysis gamma pass on the
// ring of k_pfa_rows_p.  A step is one column pair (m0, m0+1) of one beta row;
// its two columns sit in ring slots 2(i%3), 2(i%3)+1 and are transformed by the
// groups (2i + r) % 4.  Generator / store warp i % NIO first writes out the
// pair transformed in those slots three steps earlier (T[bs][m0/2][g][r], 512
// contiguous bytes per warp store), then generates pair i.
//
// Generation without a per-entry exp.  For a column m the entries of degree l
// (n = +l and n = -l) are C+-[l] D+-_b[l] with
//   C+[l] = (2l+1)/(8 pi^2) W_{m,+l},  C-[l] = (2l+1)/(8 pi^2) (-1)^{l-m} W_{m,-l}
//   D+_b[l] = d^l_{m,l}(beta_b) = exp(h[l,|m|] + (l-m) ls_b + (l+m) lc_b),  D- with m -> -m
// (wigner.py:304-322; h = log sqrt C(2l, l+|m|), ls/lc = log sin/cos(beta_b/2)).
// Along l at fixed (m, b), D+-[l+32] = D+-[l] * rho32[|m|][l] * sig32[b] with
//   rho32[a][l] = exp(h[l+32,a] - h[l,a]),  sig32[b] = (sin cos (beta_b/2))^32,
// both built on the host in long double.  Lane j owns the degrees l = j + 32 t:
// one exp per sign at its first degree >= |m|, then two multiplies per entry,
// with coalesced reads of the transposed coefficients CT[m][slot] (k_colgen_ct)
// and of rho32.  D is unimodal in l and |D| <= 1; where its peak matters the
// start value is >= e^-150 (cos^2(beta/2) = (1 + m/l*)/2 at the peak l*), so
// the multiplicative walk never has to recover from an underflow, and 31 steps
// add < 1e-14 of rounding.
// ---------------------------------------------------------------------------
#ifndef SCV_COLGENP
#define SCV_COLGENP 1
#endif
#ifndef SCV_CGP_NG
#define SCV_CGP_NG 4
#endif
#ifndef SCV_CGP_SETREG
#define SCV_CGP_SETREG 1
#endif
template <int K> struct PfaCgpCfg { static constexpr int NG = SCV_CGP_NG, NTG = 384 / SCV_CGP_NG, NIO = 4, NB = 6; };
template <int K>
static constexpr size_t pfa_smem_cgp() {
  using PL = PfaPlan<K>;
  return ((size_t)pfa_tab_total<PL>() + (size_t)PfaCgpCfg<K>::NB * K) * sizeof(double2) +
         4 * (size_t)PfaCgpCfg<K>::NB * sizeof(unsigned long long);
}

// CT[mc][gi] = C+-[l] F(l)/F(l*) of column mc (m = mc or mc - K) at gamma slot gi
// (n = gi or gi - K), 0 where |m| > l; F(l) = sqrt(C(2l, l+|m|)) / 2^l and l* is the
// first degree >= |m| in l's residue class mod 32 (the generator lane's start)
__global__ void k_colgen_ct(int L, const double2* __restrict__ w, const double* __restrict__ hlb,
                            double2* __restrict__ ct) {
  const int K = 2 * L - 1;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)K * K) return;
  const int mc = (int)(i / K), gi = (int)(i - (long long)mc * K);
  const int m = mc <= L - 1 ? mc : mc - K, am = m < 0 ? -m : m;
  const int n = gi <= L - 1 ? gi : gi - K, l = n < 0 ? -n : n;
  double2 v = make_double2(0.0, 0.0);
  if (am <= l) {
    const double2 c = w[((long long)(n >= 0 ? 0 : 1) * L + l) * K + (L - 1) + m];
    double f = (double)(2 * l + 1) * (1.0 / (8.0 * SCV_PI * SCV_PI));
    if (n < 0 && ((l - m) & 1)) f = -f;
    const int lst = am + ((l - am) & 31);
    if (l != lst) {
      // log F(l) - log F(l*), with ln 2 split so that (l - l*) ln2_hi is exact
      const double t = (double)(l - lst);
      double x = hlb[(long long)l * (l + 1) / 2 + am] - hlb[(long long)lst * (lst + 1) / 2 + am];
      x = fma(-t, 6.93147180369123816490e-01, x);
      x = fma(-t, 1.90821492927058770002e-10, x);
      f *= exp(x);
    }
    v = make_double2(f * c.x, f * c.y);
  }
  ct[i] = v;
}

template <int K>
__global__ void __launch_bounds__(PfaCgpCfg<K>::NG * PfaCgpCfg<K>::NTG + PfaCgpCfg<K>::NIO * 32, 1)
    k_ana_colgen_p(const double2* __restrict__ ct, const double* __restrict__ hlb, const double* __restrict__ lsin,
                   const double* __restrict__ lcos, const double* __restrict__ sig32, int b0, int nb,
                   double2* __restrict__ out, const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int NG = PfaCgpCfg<K>::NG, NTG = PfaCgpCfg<K>::NTG, NIO = PfaCgpCfg<K>::NIO, NB = PfaCgpCfg<K>::NB;
  constexpr int NT = NG * NTG + NIO * 32, NQT = NIO * 32;
  constexpr int L = (K + 1) / 2, NPR = (K + 1) / 2;
  static_assert((NG == 4 || NG == 2) && NB == 6 && NIO == 4,
                "pair steps use slots 2(i%3)+r and groups (2i+r)%NG; the team's warp s scales (column s>>1, sign s&1)");
  constexpr int GB = 16;  // degrees per batch of a generator lane
  static_assert(L % (32 * GB) == 0, "the generator walks l = lane + 32 t in batches of GB");
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const bufs = sm + pfa_tab_total<PL>();
  // barriers of alternate laps: see k_pfa_rows_p
  unsigned long long* const full = (unsigned long long*)(bufs + (size_t)NB * K);
  unsigned long long* const done = full + 2 * NB;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2 * NB; ++b) {
      mbar_init(full + b, 64);  // the two warps that scale a column
      mbar_init(done + b, 1);
    }
  }
  pfa_load_tables<PL, NT>(tab, gtab);
  // the CTA's contiguous range of (pair, beta row) steps, flat index = pair * nb + bs
  const long long S = (long long)NPR * nb;
  const long long lo = S * blockIdx.x / gridDim.x, hi = S * (blockIdx.x + 1) / gridDim.x;
  const long long ni = hi - lo;
  static_assert(!SCV_CGP_SETREG || (NG * NTG == 384 && NQT == 128), "setmaxnreg works on warpgroups of 128 threads");
  constexpr bool SETREG = SCV_CGP_SETREG && (K == 2047 || (K == 1023 && SCV_SETREG_1023));
  if (threadIdx.x >= NG * NTG) {
    if constexpr (SETREG) asm volatile("setmaxnreg.inc.sync.aligned.u32 152;\n");
    // ---- generator / store team: all NIO warps work on every step, in order
    // (a step's drain + fill latency sits on the ring's critical path: three slot
    // pairs, two of them under transform)
    const int t = threadIdx.x - NG * NTG, lane = t & 31, ws = t >> 5;
    const int tbar = 1 + NG;
    // Warp ws generates (column ws >> 1, sign ws & 1), lane j the degrees l = j + 32 k;
    // as a store thread t writes entry t & 1 of the pairs g = (t >> 1) + 64 j.  Both index
    // sets are constants of the thread, so their slot positions live in registers
    // (two 16-bit positions per register) instead of two map reads per element per step.
    constexpr int NL = L / 32;          // degrees per generator lane
    constexpr int ND = (K + 63) / 64;   // pairs per store thread
    static_assert(NL % GB == 0 && NL % 2 == 0 && ND % 2 == 0, "packed position registers");
    const int r_gen = ws >> 1, neg = ws & 1, r_st = t & 1;
    unsigned pg[NL / 2], pd[ND / 2];
#pragma unroll
    for (int k = 0; k < NL / 2; ++k) {
      const int l0 = lane + 32 * (2 * k), l1 = l0 + 32;
      pg[k] = (unsigned)pfa_in_tab<PL>(tab, neg ? (l0 ? K - l0 : 0) : l0) |
              ((unsigned)pfa_in_tab<PL>(tab, neg ? K - l1 : l1) << 16);
    }
#pragma unroll
    for (int j = 0; j < ND / 2; ++j) {
      const int g0 = (t >> 1) + 64 * (2 * j), g1 = g0 + 64;
      pd[j] = (unsigned)pfa_pos_tab<PL>(tab, g0 < K ? g0 : 0) | ((unsigned)pfa_pos_tab<PL>(tab, g1 < K ? g1 : 0) << 16);
    }
    long long st[6] = {0, 0, 0, 0, 0, 0}, st2[6] = {0, 0, 0, 0, 0, 0};
    PipeClk ck;
    // (pair, beta row) of the fill step and of the drain step, advanced incrementally
    int fpr = (int)(lo / nb), fbs = (int)(lo - (long long)fpr * nb);
    int dpr = fpr, dbs = fbs;
    // first batch of coefficients and the closed-form start value of a step: issued at
    // the end of the previous step, so the loads and the exp overlap the drain
    double2 c[GB];
    double d = 0.0, S32 = 0.0;
    int lst = 0;
    const double2* cp = ct;
    auto start_step = [&](int pr, int bs) {
      const int mc = 2 * pr + r_gen;
      d = 0.0;
      lst = L;
      if (mc >= K) return;  // the odd column past the end: zeros (transformed, never read)
      const int b = b0 + bs;
      const int m = mc <= L - 1 ? mc : mc - K, am = m < 0 ? -m : m;
      lst = am + ((lane - am) & 31);
      cp = ct + (long long)mc * K;
#pragma unroll
      for (int k = 0; k < GB; ++k) {
        const int l = lane + 32 * k;
        c[k] = cp[neg ? (l ? K - l : 0) : l];
      }
      if (lst < L) {
        // n >= 0: sin^(l-m) cos^(l+m); n < 0: sin^(l+m) cos^(l-m).  xlogy semantics at the
        // poles: a zero exponent drops its (possibly -inf) log
        const int es = neg ? lst + m : lst - m, ec = neg ? lst - m : lst + m;
        double lg = hlb[lst * (lst + 1) / 2 + am];
        if (es) lg += (double)es * lsin[b];
        if (ec) lg += (double)ec * lcos[b];
        d = exp(lg);
      }
      S32 = sig32[b] * 4294967296.0;  // sin(beta_b)^32 = (2 sin cos (beta_b/2))^32
    };
    if (ni > 0) start_step(fpr, fbs);
#pragma unroll 1
    for (int i = 0; i < (int)ni + 3; ++i) {
      const int s0 = 2 * (i % 3);
      const unsigned u = (unsigned)(i / 3);
      double2* const X0 = bufs + (size_t)s0 * K;
      double2* const X1 = X0 + K;
      ck.mark(st, 4);
      if (i >= 3) {
        // the pair of step i - 3 was transformed in these slots: write T[bs][pair][g][r]
        mbar_wait(done + ((u - 1) & 1) * NB + s0, ((u - 1) >> 1) & 1);
        mbar_wait(done + ((u - 1) & 1) * NB + s0 + 1, ((u - 1) >> 1) & 1);
        ck.mark(st, 2);
        double2* dst = out + (((long long)dbs * NPR + dpr) * K) * 2 + 2 * (t >> 1) + r_st;
        if (++dbs == nb) {
          dbs = 0;
          ++dpr;
        }
        const double2* Xr = r_st ? X1 : X0;
#pragma unroll
        for (int j0 = 0; j0 < ND / 2; j0 += RB / 2) {
          double2 v[RB];
#pragma unroll
          for (int j = 0; j < RB / 2; ++j) {
            v[2 * j] = Xr[pd[j0 + j] & 0xffffu];
            v[2 * j + 1] = Xr[pd[j0 + j] >> 16];
          }
#pragma unroll
          for (int j = 0; j < RB / 2; ++j) {
            const int g0 = (t >> 1) + 64 * (2 * (j0 + j));
            if (g0 < K) dst[2 * (64 * 2 * (j0 + j))] = v[2 * j];
            if (g0 + 64 < K) dst[2 * (64 * (2 * (j0 + j) + 1))] = v[2 * j + 1];
          }
        }
        grp_sync(tbar, NQT);  // the whole team has read the pair before anyone refills it
        ck.mark(st, 3);
      }
      if (i < (int)ni) {
        // entry l is CT[m][slot] * D_b[l*] sin(beta_b)^(l - l*), with D_b[l*] =
        // d^{l*}_{m,+-l*}(beta_b) in closed form at the lane's first degree l* >= |m|
        // (wigner.py:304-322) -- a geometric walk, no table reads.  Values go from
        // registers straight to their Ruritanian positions (one 16-byte store each;
        // CT's exact zeros below |m| overwrite the slot's previous contents).
        double2* const X = r_gen ? X1 : X0;
        PipeClk ck2;
        ck2.t = ck.t;
        if (2 * fpr + r_gen >= K) {
          for (int g = lane + 32 * neg; g < K; g += 64) X[g] = make_double2(0.0, 0.0);
        } else {
#pragma unroll
          for (int kb = 0; kb < NL; kb += GB) {
#pragma unroll
            for (int k = 0; k < GB; ++k) {
              const int l = lane + 32 * (kb + k);
              if (l > lst) d *= S32;
              c[k] = make_double2(d * c[k].x, d * c[k].y);  // d = 0 before l*, where CT is 0 too
            }
#pragma unroll
            for (int k = 0; k < GB; ++k) {
              const int l = lane + 32 * (kb + k);
              const unsigned pk = pg[(kb + k) >> 1];
              if (l > 0 || !neg) X[((kb + k) & 1) ? pk >> 16 : pk & 0xffffu] = c[k];
            }
            if (kb + GB < NL) {
#pragma unroll
              for (int k = 0; k < GB; ++k) {
                const int l = lane + 32 * (kb + GB + k);
                c[k] = cp[neg ? K - l : l];
              }
            }
          }
        }
        ck2.mark(st2, 3);  // generation
        mbar_arrive(full + (u & 1) * NB + s0 + r_gen);
        if (++fbs == nb) {
          fbs = 0;
          ++fpr;
        }
        if (i + 1 < (int)ni) start_step(fpr, fbs);
        ck2.mark(st2, 1);  // next step's loads issued + closed-form start
      }
    }
    ck.mark(st, 4);
    pipe_flush(st, 1, t == 0);
    pipe_flush(st2, 3, t == 0);
    return;
  }
  if constexpr (SETREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 120;\n");
  const int g = threadIdx.x / NTG, gtid = threadIdx.x - g * NTG, bar = 1 + g;
  const int r = g & 1;
  long long st[6] = {0, 0, 0, 0, 0, 0};
  PipeClk ck;
#pragma unroll 1
  for (long long i = g >> 1; i < ni; i += NG / 2) {
    const int slot = 2 * (int)(i % 3) + r;
    const unsigned u = (unsigned)(i / 3);
    mbar_wait(full + (u & 1) * NB + slot, (u >> 1) & 1);
    ck.mark(st, 0);
    pfa_dft<PL, +1, 1, NTG, K>(bufs + (size_t)slot * K, tab, nullptr, gtid, bar);
    if (gtid == 0) mbar_arrive(done + (u & 1) * NB + slot);
    ck.mark(st, 1);
  }
  pipe_flush(st, 1, gtid == 0);
}

// ---------------------------------------------------------------------------
// Staged column generation with TMA stores (SCV_COLGEN_TMA, K = 2047).
// k_ana_colgen_s spends ~30% of its stall samples in the store loop: every
// output element (g, b, m0..m0+1) is a 32-byte piece at stride nb*K*16 B, so
// each warp store instruction scatters over 16 lines while the DMMA pipe
// idles (profiles/r01v11_ncu_k_ana_colgen_s.txt).  Here the transformed
// column pair is permuted in place into the TMA box order [g][m0..m0+1] and
// written by 8 bulk tensor stores (box 4 doubles x 1 beta row x 256 gamma,
// out-of-range m / gamma clipped by the TMA unit); the CTA goes on to
// generate the next row into registers while the TMA engine streams the
// scattered pieces, and waits for the bulk READ of the buffer only before
// overwriting it.  Measured on B200 (r01v11): correct, but 170 vs 160 ms/map
// for the analysis gamma pass -- the scattered 32-byte pieces cost the same
// whether the LSU or the TMA unit issues them, and the in-place permutation
// adds two barriers per row -- so it is off by default.
// ---------------------------------------------------------------------------
#ifndef SCV_COLGEN_TMA
#define SCV_COLGEN_TMA 0
#endif
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* smem, int c0, int c1, int c2) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
               ::"l"(reinterpret_cast<unsigned long long>(map)), "r"(sa), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int K>
__global__ void __launch_bounds__(PfaSCfg<K>::NT, PfaSCfg<K>::MINB)
    k_ana_colgen_t(const double2* __restrict__ w, const double* __restrict__ hlb, const double* __restrict__ lsin,
                   const double* __restrict__ lcos, int b0, int nb, const __grid_constant__ CUtensorMap omap,
                   const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaSCfg<K>::R, NT = PfaSCfg<K>::NT, BB = PfaSCfg<K>::BB;
  constexpr int L = (K + 1) / 2;
  constexpr int NGRP = (K + R - 1) / R;
  constexpr int GB = 256;                         // gamma rows per TMA box
  constexpr int NBOX = (K + GB - 1) / GB;
  static_assert(R == 2, "box inner extent is one column pair (4 doubles)");
  extern __shared__ __align__(128) double2 sm[];
  double2* tab = sm;
  double2* const X = sm + pfa_tab_total<PL>();    // 128-byte aligned (tables are 2816 double2)
  double2* const CW = X + R * K;
  double* const CH = (double*)(CW + R * K);
  pfa_load_tables<PL, NT>(tab, gtab);
  const double fac0 = 1.0 / (8.0 * SCV_PI * SCV_PI);
  const int nbblk = (nb + BB - 1) / BB;
  const int ntask = nbblk * NGRP;
  constexpr int NPT = (K + NT - 1) / NT;
  constexpr int EPT = (R * K + NT - 1) / NT;
  bool pending = false;  // a bulk store still reads X (thread 0's bulk group)
#pragma unroll 1
  for (int task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int bblk = task / NGRP;
    const int m0 = (task - bblk * NGRP) * R;
#pragma unroll
    for (int u = 0; u < NPT; ++u) {
      const int gi = threadIdx.x + u * NT;
      if (gi >= K) continue;
      const int n = gi <= L - 1 ? gi : gi - K;
      const int l = n < 0 ? -n : n;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int m = m0 + r <= L - 1 ? m0 + r : m0 + r - K, am = m < 0 ? -m : m;
        const bool nz = m0 + r < K && am <= l;
        CW[gi * R + r] = nz ? w[((n >= 0 ? 0 : 1) * L + l) * K + (L - 1) + m] : make_double2(0.0, 0.0);
        CH[gi * R + r] = nz ? hlb[l * (l + 1) / 2 + am] : 0.0;
      }
    }
    __syncthreads();
    const int bs_end = min(nb, (bblk + 1) * BB);
#pragma unroll 1
    for (int bs = bblk * BB; bs < bs_end; ++bs) {
      const int b = b0 + bs;
      const double ls = lsin[b], lc = lcos[b];
      // generation into registers (X may still be read by the previous row's bulk stores)
      double2 gv[NPT][R];
#pragma unroll
      for (int u = 0; u < NPT; ++u) {
        const int gi = threadIdx.x + u * NT;
        const int n = gi <= L - 1 ? gi : gi - K;
        const int l = n < 0 ? -n : n;
        const double facl = (double)(2 * l + 1) * fac0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int m = m0 + r <= L - 1 ? m0 + r : m0 + r - K, am = m < 0 ? -m : m;
          double2 v = make_double2(0.0, 0.0);
          if (gi < K && m0 + r < K && am <= l) {
            const int es = n >= 0 ? l - m : l + m;
            const int ec = n >= 0 ? l + m : l - m;
            double lg = CH[gi * R + r];
            if (es) lg += (double)es * ls;
            if (ec) lg += (double)ec * lc;
            double d = exp(lg);
            if (n < 0 && ((l - m) & 1)) d = -d;
            const double f = facl * d;
            const double2 c = CW[gi * R + r];
            v = make_double2(f * c.x, f * c.y);
          }
          gv[u][r] = v;
        }
      }
      if (pending && threadIdx.x == 0) bulk_wait_read0();
      __syncthreads();
#pragma unroll
      for (int u = 0; u < NPT; ++u) {
        const int gi = threadIdx.x + u * NT;
        if (gi >= K) continue;
        const int xi = pfa_in_tab<PL>(tab, gi);
#pragma unroll
        for (int r = 0; r < R; ++r) X[r * K + xi] = gv[u][r];
      }
      __syncthreads();
      pfa_dft<PL, +1, R, NT, K>(X, tab, nullptr);
      // permute in place into the box order X'[g*R + r] (reads all, barrier, writes all)
      double2 ov[EPT];
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const int i = threadIdx.x + e * NT;
        if (i < R * K) {
          const int g = i / R, r = i - g * R;
          ov[e] = X[r * K + pfa_pos_tab<PL>(tab, g)];
        }
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const int i = threadIdx.x + e * NT;
        if (i < R * K) X[i] = ov[e];
      }
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
#pragma unroll 1
        for (int q = 0; q < NBOX; ++q) tma_store_3d(&omap, X + q * GB * R, 2 * m0, bs, q * GB);
        bulk_commit();
      }
      pending = true;
    }
    // CW / CH are re-staged next task: nothing of theirs is read by the bulk stores
    __syncthreads();
  }
  if (threadIdx.x == 0) bulk_wait0();
}

// ---------------------------------------------------------------------------
// analysis, real signal, gamma first.  For a real signal the gamma transform
// T_b[g, m] = sum_n F_b[n, m] e^{i n gamma_g} is Hermitian in m for every g, so
// only the columns m >= 0 are formed (half the columns of the complex path),
// with the n < 0 entries taken from the n > 0 half by the real-signal symmetry
// F[-n, -m] = conj(F[n, m]) and the n = 0 entry reduced to its real part --
// exactly the inputs the reference's real path reads (so3.py:386-417: the
// n >= 0 half spectrum, irfft semantics for the n = 0 bin).  Output T is
// (K, nb, L) complex; the alpha pass k_rows_c2r then forms two real rows per
// complex transform.
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(PfaGCfg<K>::NT, PfaGCfg<K>::MINB)
    k_ana_colgen_real(const double2* __restrict__ w, const double* __restrict__ hlb, const double* __restrict__ lsin,
                      const double* __restrict__ lcos, int b0, int nb, double2* __restrict__ T,
                      const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaGCfg<K>::R, NT = PfaGCfg<K>::NT;
  constexpr int L = (K + 1) / 2;
  constexpr int NGRP = (L + R - 1) / R;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const X = scr + pfa_scratch<PL, R, NT>();
  pfa_load_tables<PL, NT>(tab, gtab);
  const double fac0 = 1.0 / (8.0 * SCV_PI * SCV_PI);
  const int ntask = nb * NGRP;
  constexpr int NPT = (K + NT - 1) / NT;
#pragma unroll 1
  for (int task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int bs = task / NGRP;
    const int b = b0 + bs;
    const int m0 = (task - bs * NGRP) * R;
    const double ls = lsin[b], lc = lcos[b];
#pragma unroll 1
    for (int u = 0; u < NPT; ++u) {
      const int gi = threadIdx.x + u * NT;
      if (gi >= K) continue;
      const int n = gi <= L - 1 ? gi : gi - K;
      const int l = n < 0 ? -n : n;
      const double facl = (double)(2 * l + 1) * fac0;
      const int xi = pfa_in_tab<PL>(tab, gi);
      // n < 0 uses the n = +l sheet at -m, conjugated
      const double* hrow = hlb + l * (l + 1) / 2;
      const double2* wrow = w + (long long)l * K + (L - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int m = m0 + r;
        double2 v = make_double2(0.0, 0.0);
        if (m < L && m <= l) {
          const int ms = n >= 0 ? m : -m;   // the sheet-0 entry (n' = +l, m')
          const int es = l - ms, ec = l + ms;
          double lg = hrow[m];
          if (es) lg += (double)es * ls;
          if (ec) lg += (double)ec * lc;
          const double f = facl * exp(lg);
          const double2 cw = wrow[ms];
          v = n >= 0 ? make_double2(f * cw.x, f * cw.y) : make_double2(f * cw.x, -f * cw.y);
          if (n == 0) v.y = 0.0;  // l = 0: the real part (irfft semantics of the n = 0 bin)
        }
        X[r * K + xi] = v;
      }
    }
    __syncthreads();
    pfa_dft<PL, +1, R, NT, K>(X, tab, scr);
#pragma unroll 4
    for (int i = threadIdx.x; i < R * K; i += NT) {
      const int g = i / R, r = i - g * R;
      const int m = m0 + r;
      if (m < L) T[((long long)g * nb + bs) * L + m] = X[r * K + pfa_pos_tab<PL>(tab, g)];
    }
    __syncthreads();
  }
}

// alpha pass of the real analysis: rows ri = (g, bs) of T (L Hermitian-half
// bins each) -> real rows of sig (K, nb, K).  Two rows per complex transform:
// Z = T1 + i T2 extended by Z[-m] = conj(T1[m]) + i conj(T2[m]); the IDFT of Z
// is f1 + i f2.
template <int K>
__global__ void __launch_bounds__(PfaCfg<K, false>::NT, PfaCfg<K, false>::MINB)
    k_rows_c2r(long long nrows, const double2* __restrict__ T, double* __restrict__ out,
               const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, false>::R, NT = PfaCfg<K, false>::NT;
  constexpr int L = (K + 1) / 2;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const X = scr + pfa_scratch<PL, PfaRD<K, false>::v, NT>();
  pfa_load_tables<PL, NT>(tab, gtab);
  const long long nb = (nrows + 2 * R - 1) / (2 * R);
#pragma unroll 1
  for (long long bt = blockIdx.x; bt < nb; bt += gridDim.x) {
    const long long r0 = bt * 2 * R;
#pragma unroll 4
    for (int i = threadIdx.x; i < R * L; i += NT) {
      const int r = i / L, m = i - r * L;
      const long long ri1 = r0 + 2 * r, ri2 = ri1 + 1;
      double2 t1 = ri1 < nrows ? T[ri1 * L + m] : make_double2(0.0, 0.0);
      double2 t2 = ri2 < nrows ? T[ri2 * L + m] : make_double2(0.0, 0.0);
      if (m == 0) {
        t1.y = 0.0;
        t2.y = 0.0;
      }
      X[r * K + pfa_in_tab<PL>(tab, m)] = make_double2(t1.x - t2.y, t1.y + t2.x);
      if (m > 0) X[r * K + pfa_in_tab<PL>(tab, K - m)] = make_double2(t1.x + t2.y, -t1.y + t2.x);
    }
    __syncthreads();
    pfa_dft_rows<PL, +1, R, PfaRD<K, false>::v, NT>(X, tab, scr);
#pragma unroll 4
    for (int i = threadIdx.x; i < 2 * R * K; i += NT) {
      const int c = i / K, a = i - c * K;
      const long long ri = r0 + c;
      if (ri < nrows) {
        const double2 z = X[(c >> 1) * K + pfa_pos_tab<PL>(tab, a)];
        out[ri * K + a] = (c & 1) ? z.y : z.x;
      }
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
  double2* const buf0 = scr + pfa_scratch<PL, PfaRD<K, true>::v, NT>();  // buffer c at buf0 + c * R * K (stays a shared pointer)
  pfa_load_tables<PL, NT>(tab, gtab);
  const int cpb = real ? 2 * R : R;  // columns per batch
  const int ngrp = (K + cpb - 1) / cpb;
  const long long nb = (long long)L * ngrp;
  auto issue = [&](long long bt, double2* X) {
    const int b = (int)(bt / ngrp);
    const int a0 = (int)(bt - (long long)b * ngrp) * cpb;
    const int r = threadIdx.x % R, a = a0 + r;
    const double2* q = src + (long long)b * K + a + (long long)(threadIdx.x / R) * LK;
#pragma unroll 4
    for (int g = threadIdx.x / R; g < K; g += NT / R, q += (NT / R) * LK) {
      const int xi = r * K + pfa_in_tab<PL>(tab, g);
      if (a < K) cp_async16(X + xi, q);
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
        X[r * K + pfa_in_tab<PL>(tab, n)] = make_double2(t1.x - t2.y, t1.y + t2.x);
        if (n > 0) X[r * K + pfa_in_tab<PL>(tab, K - n)] = make_double2(t1.x + t2.y, -t1.y + t2.x);
      }
    }
    __syncthreads();
    pfa_dft_rows<PL, +1, R, PfaRD<K, true>::v, NT>(X, tab, scr);
    if (!real) {
      const int r = threadIdx.x % R, a = a0 + r;
      double2* q = src + (long long)b * K + a + (long long)(threadIdx.x / R) * LK;
      if (a < K) {
#pragma unroll 4
        for (int g = threadIdx.x / R; g < K; g += NT / R, q += (NT / R) * LK) *q = X[r * K + pfa_pos_tab<PL>(tab, g)];
      }
    } else {
#pragma unroll 4
      for (int i = threadIdx.x; i < 2 * R * K; i += NT) {
        const int g = i / (2 * R), c = i - g * (2 * R);
        const int r = c >> 1;
        const int a = a0 + c;
        if (a < K) {
          const double2 z = X[r * K + pfa_pos_tab<PL>(tab, g)];
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
    k_syn_alpha(int real, int tr, const void* __restrict__ in, int lsig, int b0, int nbb, double2* __restrict__ chunk,
                const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int R = PfaCfg<K, false>::R, NT = PfaCfg<K, false>::NT;
  constexpr int L = (K + 1) / 2;
  const long long LK = (long long)lsig * K;  // in: (K, lsig, K), rows b0.. of this launch
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const buf0 = scr + pfa_scratch<PL, PfaRD<K, false>::v, NT>();  // buffer c at buf0 + c * R * K (stays a shared pointer)
  pfa_load_tables<PL, NT>(tab, gtab);
  const int nrows = K * nbb;  // row index = bb*K + g
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
        cp_async16(X + r * K + pfa_in_tab<PL>(tab, a), F + (long long)g * LK + (long long)(b0 + bb) * K + a);
      } else {
        X[i] = make_double2(0.0, 0.0);
      }
    }
    cp_async_commit();
  };
  constexpr int NBUF = PfaNBuf<K, false>::v;
  long long bt = blockIdx.x;
  int cur = 0;
  if (NBUF == 2 && !real && bt < nb) issue(bt, buf0);
#pragma unroll 1
  for (; bt < nb; bt += gridDim.x) {
    const long long r0 = bt * rpb;
    double2* X = buf0 + cur * (R * K);
    if (!real && NBUF == 2) {
      const long long nx = bt + gridDim.x;
      if (nx < nb) issue(nx, buf0 + (cur ^ 1) * (R * K));
      else cp_async_commit();
      cp_async_wait<1>();
    } else if (!real) {
      issue(bt, buf0);
      cp_async_wait<0>();
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
        X[r * K + pfa_in_tab<PL>(tab, a)] = make_double2(v1, v2);
      }
    }
    __syncthreads();
    pfa_dft_rows<PL, -1, R, PfaRD<K, false>::v, NT>(X, tab, scr);
    if (!real && tr) {
      // transposed chunk [bb][m][g]: R consecutive g of one m are adjacent
#pragma unroll 4
      for (int i = threadIdx.x; i < R * K; i += NT) {
        const int m = i / R, r = i - m * R;
        const int ri = (int)r0 + r;
        if (ri < nrows) {
          const int bb = ri / K, g = ri - bb * K;
          chunk[((long long)bb * K + m) * K + g] = X[r * K + pfa_pos_tab<PL>(tab, m)];
        }
      }
    } else if (!real) {
#pragma unroll 4
      for (int i = threadIdx.x; i < R * K; i += NT) {
        const int r = i / K, m = i - r * K;
        const long long ri = r0 + r;
        if (ri < nrows) chunk[ri * K + m] = X[r * K + pfa_pos_tab<PL>(tab, m)];
      }
    } else if (tr) {
#pragma unroll 4
      for (int i = threadIdx.x; i < 2 * R * K; i += NT) {
        const int m = i / (2 * R), c = i - m * (2 * R);
        const int r = c >> 1;
        const int ri = (int)r0 + c;
        if (ri < nrows && (real != 2 || m < L)) {
          const double2 z = X[r * K + pfa_pos_tab<PL>(tab, m)];
          const double2 zc = X[r * K + pfa_pos_tab<PL>(tab, m == 0 ? 0 : K - m)];
          double2 v;
          if ((c & 1) == 0) v = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
          else v = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
          const int bb = ri / K, g = ri - bb * K;
          chunk[((long long)bb * K + m) * K + g] = v;
        }
      }
    } else {
      // Z = X1 + i X2 (X1, X2 Hermitian): X1[k] = (Z[k] + conj Z[-k])/2, X2[k] = (Z[k] - conj Z[-k])/(2i)
      // (real == 2: only the m >= 0 half the gamma+quadrature pass reads)
#pragma unroll 4
      for (int i = threadIdx.x; i < 2 * R * K; i += NT) {
        const int c = i / K, m = i - c * K;
        const int r = c >> 1;
        const long long ri = r0 + c;
        if (ri < nrows && (real != 2 || m < L)) {
          const double2 z = X[r * K + pfa_pos_tab<PL>(tab, m)];
          const double2 zc = X[r * K + pfa_pos_tab<PL>(tab, m == 0 ? 0 : K - m)];
          double2 v;
          if ((c & 1) == 0) v = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
          else v = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
          chunk[ri * K + m] = v;
        }
      }
    }
    __syncthreads();
    if (!real && NBUF == 2) cur ^= 1;
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
  double2* const buf0 = scr + pfa_scratch<PL, PfaRD<K, true>::v, NT>();  // buffer c at buf0 + c * R * K (stays a shared pointer)
  pfa_load_tables<PL, NT>(tab, gtab);
  const int ngrp = (K + R - 1) / R;
  const long long nb = (long long)nbb * ngrp;
  auto issue = [&](long long bt, double2* X) {
    const int bb = (int)(bt / ngrp);
    const int q0 = (int)(bt - (long long)bb * ngrp) * R;
    const int r = threadIdx.x % R, q = q0 + r;
    const double2* c = chunk + ((long long)bb * K + threadIdx.x / R) * K + q;
#pragma unroll 4
    for (int g = threadIdx.x / R; g < K; g += NT / R, c += (NT / R) * K) {
      const int xi = r * K + pfa_in_tab<PL>(tab, g);
      if (q < K) cp_async16(X + xi, c);
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
    pfa_dft_rows<PL, -1, R, PfaRD<K, true>::v, NT>(X, tab, scr);
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
      W1p[(w1p_colbase(n, real) + m + an) * (long long)L + b0 + bb] = X[r * K + pfa_pos_tab<PL>(tab, gn)];
    }
    __syncthreads();
    cur ^= 1;
  }
}

// ---------------------------------------------------------------------------
// synthesis gamma + beta quadrature (betaq.cu): a block owns alpha-frequency
// columns m; for each beta slab bb of the chunk it transforms the column over
// g -> n and accumulates S_{nm}(b) q_{nm}(b) for |n| >= |m| in shared memory;
// after the last slab it adds the partial sums into W[(sheet n), |n|, m].
// Replaces the W1p scatter, the per-column beta FFTs and the Delta contraction.
// Each (n, m) entry is owned by one block and chunks run in order, so the
// summation order is fixed (bit-reproducible).
// ---------------------------------------------------------------------------
template <int K> struct PfaQCfg { static constexpr int RQ = 1, NT = 256, MINB = 1; };
// threads of the K = 4095 gamma+quadrature block, re-swept with the 9 * 13 * 35 plan (r09, ms of this
// pass on the C5 streamed map): 256: 1384; 384: 1227; 448: 1274; 512: 1152; 576: 1225; 640: 1177; 768: 1183
#ifndef SCV_Q4095_NT
#define SCV_Q4095_NT 512
#endif
template <> struct PfaQCfg<4095> { static constexpr int RQ = 1, NT = SCV_Q4095_NT, MINB = 1; };
template <> struct PfaQCfg<255> { static constexpr int RQ = 1, NT = 128, MINB = 1; };
#ifndef SCV_Q1023
#define SCV_Q1023 1, 352, 1
#endif
#ifndef SCV_Q2047
#define SCV_Q2047 1, 192, 2
#endif
#define SCV_QCFG_(KK, ...)                                   \
  template <> struct PfaQCfg<KK> {                           \
    static constexpr int v_[3] = {__VA_ARGS__};              \
    static constexpr int RQ = v_[0], NT = v_[1], MINB = v_[2]; \
  };
SCV_QCFG_(1023, SCV_Q1023)
SCV_QCFG_(2047, SCV_Q2047)

template <int K>
static constexpr size_t pfa_smem_q() {
  using PL = PfaPlan<K>;
  return ((size_t)pfa_tab_total<PL>() + pfa_scratch<PL, PfaQCfg<K>::RQ, PfaQCfg<K>::NT>() +
          2 * (size_t)PfaQCfg<K>::RQ * K) * sizeof(double2);
}

#ifndef SCV_GQ_L2LINE
#define SCV_GQ_L2LINE 0
#endif
#ifndef SCV_GQ_RED
#define SCV_GQ_RED 1
#endif
// offset of the m block of the quadrature table (betaq.cu): QR * sum_{j=-(L-1)}^{m-1} (L - |j|),
// QR = the number of beta rows the table holds (L, or a rank's slab: scv_betaq_restrict)
__device__ __forceinline__ long long q_mbase(int m, int L, int QR) {
  const long long a = (long long)m + L - 1;  // number of terms
  if (m <= 0) return (long long)QR * (a * (a + 1) / 2);
  return (long long)QR * ((long long)L * (L + 1) / 2 + (long long)(m - 1) * L - (long long)m * (m - 1) / 2);
}

template <int K>
__global__ void __launch_bounds__(PfaQCfg<K>::NT, PfaQCfg<K>::MINB)
    k_syn_gamma_q(int real, int tr, const double2* __restrict__ chunk, int b0, int nbb, const double* __restrict__ qtab,
                  const long long* __restrict__ mbase, int qrows, double2* __restrict__ wout,
                  const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int NT = PfaQCfg<K>::NT, RQ = PfaQCfg<K>::RQ;
  constexpr int L = (K + 1) / 2;
  // real: only the columns m >= 0 are transformed (the chunk of a real
  // signal is Hermitian in (g, m) jointly: T(n, -m) = conj T(-n, m)), and the
  // n < 0 outputs of column m feed W(-n, -m) = sum_b q_{-n,-m}(b) conj T(n, m)
  const int NCG = real ? (L + RQ - 1) / RQ : (K + RQ - 1) / RQ;  // column groups of RQ adjacent m
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const scr = sm + pfa_tab_total<PL>();
  double2* const buf0 = scr + pfa_scratch<PL, RQ, NT>();  // two buffers of RQ K-point columns
  constexpr int NA = (K + NT - 1) / NT;                   // accumulators per column per thread: n slots tid + u*NT
  double2 acc[RQ][NA];
  pfa_load_tables<PL, NT>(tab, gtab);
  const int mine = blockIdx.x < NCG ? (NCG - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int ntask = mine * nbb;
  auto issue = [&](int task, double2* X) {
    const int col0 = (blockIdx.x + (task / nbb) * gridDim.x) * RQ;
    const int bb = task % nbb;
    if (tr) {  // transposed chunk [bb][m][g]: the column is contiguous
#pragma unroll
      for (int r = 0; r < RQ; ++r) {
        if (col0 + r >= K) continue;
        const double2* cp = chunk + ((long long)bb * K + col0 + r) * K;
#pragma unroll 4
        for (int g = threadIdx.x; g < K; g += NT) cp_async16(X + r * K + pfa_in_tab<PL>(tab, g), cp + g);
      }
    } else {   // chunk [bb][g][m]: RQ adjacent columns = RQ*16-byte segments at stride K
      const int r = threadIdx.x % RQ;
      const double2* cp = chunk + ((long long)bb * K + threadIdx.x / RQ) * K + col0 + r;
#pragma unroll 4
      for (int g = threadIdx.x / RQ; g < K; g += NT / RQ, cp += (long long)(NT / RQ) * K) {
        if (col0 + r < K) {
#if SCV_GQ_L2LINE
          cp_async16_l2line(X + r * K + pfa_in_tab<PL>(tab, g), cp);
#else
          cp_async16(X + r * K + pfa_in_tab<PL>(tab, g), cp);
#endif
        }
        else X[r * K + pfa_in_tab<PL>(tab, g)] = make_double2(0.0, 0.0);
      }
    }
    cp_async_commit();
  };
  if (ntask > 0) issue(0, buf0);
  int cur = 0;
#pragma unroll 1
  for (int task = 0; task < ntask; ++task) {
    if (task + 1 < ntask) issue(task + 1, buf0 + (cur ^ 1) * (RQ * K));
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double2* X = buf0 + cur * (RQ * K);
    const int col0 = (blockIdx.x + (task / nbb) * gridDim.x) * RQ;
    const int bb = task % nbb;
    if (bb == 0) {
#pragma unroll
      for (int r = 0; r < RQ; ++r)
#pragma unroll
        for (int u = 0; u < NA; ++u) acc[r][u] = make_double2(0.0, 0.0);
    }
    const long long b = b0 + bb;
    // quadrature weights of this task's (n, m) entries, loaded before the
    // transform so their latency hides behind it
    double qv[RQ][NA];
#pragma unroll
    for (int r = 0; r < RQ; ++r) {
      const int col = col0 + r;
      const int m = col <= L - 1 ? col : col - K;
      const int am = m < 0 ? -m : m;
      // table offsets in closed form (no dependent gather): mbase(m) = L * sum_{j<m} (L-|j|)
      const double* qp = qtab + q_mbase(min(m, L - 1), L, qrows) + b * (L - am) - am;    // + n       (n >= 0)
      const double* qn = qtab + q_mbase(max(-m, -(L - 1)), L, qrows) + b * (L - am) - am;  // + |n| (n < 0)
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        const int gn = threadIdx.x + u * NT;
        const int n = gn <= L - 1 ? gn : gn - K;
        const int an = n < 0 ? -n : n;
        qv[r][u] = 0.0;
        if (col >= (real ? L : K) || gn >= K || an < am || (real && n < 0 && m == 0)) continue;
        // raw load only; the sign q_{-l,m} = (-1)^{l+m} q_{l,-m} is applied at use
        // (real, n < 0: the weight of W(|n|, -m) is q_{|n|,-m} itself)
        qv[r][u] = __ldg(n >= 0 ? qp + n : qn + an);
      }
    }
    pfa_dft<PL, -1, RQ, NT, K>(X, tab, scr);
#pragma unroll
    for (int r = 0; r < RQ; ++r) {
      const int col = col0 + r;
      if (col >= K) continue;
      const int m = col <= L - 1 ? col : col - K;
      const int am = m < 0 ? -m : m;
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        const int gn = threadIdx.x + u * NT;
        const int n = gn <= L - 1 ? gn : gn - K;
        const int an = n < 0 ? -n : n;
        if (gn >= K || an < am || (real && n < 0 && m == 0)) continue;
        const double q = (!real && n < 0 && ((an + m) & 1)) ? -qv[r][u] : qv[r][u];
        double2 v = X[r * K + pfa_pos_tab<PL>(tab, gn)];
        if (real && n < 0) v.y = -v.y;
        acc[r][u].x = fma(v.x, q, acc[r][u].x);
        acc[r][u].y = fma(v.y, q, acc[r][u].y);
      }
      if (bb == nbb - 1) {
#pragma unroll
        for (int u = 0; u < NA; ++u) {
          const int gn = threadIdx.x + u * NT;
          const int n = gn <= L - 1 ? gn : gn - K;
          const int an = n < 0 ? -n : n;
          if (gn >= K || an < am || (real && n < 0 && m == 0)) continue;
          // complex: sheet by the sign of n; real: n < 0 slots hold W(|n|, -m) on sheet 0
          double2* o = real ? wout + (long long)an * K + ((n < 0 ? -m : m) + L - 1)
                            : wout + ((long long)(n >= 0 ? 0 : 1) * L + an) * K + (m + L - 1);
          const double2 a = acc[r][u];
#if SCV_GQ_RED
          // one add per entry per launch, launches stream-ordered: deterministic
          atomicAdd(&o->x, a.x);
          atomicAdd(&o->y, a.y);
#else
          double2 w = *o;
          w.x += a.x;
          w.y += a.y;
          *o = w;
#endif
        }
      }
    }
    __syncthreads();
    cur ^= 1;
  }
}

// ---------------------------------------------------------------------------
// Pipelined gamma pass + beta quadrature (r02, K = 2047, chunk [bb][g][m]).
// The ring and transform groups of k_pfa_rows_p; the load/store side is ONE team
// of NQW warps that walks the CTA's (column, beta row) steps in order.  At step
// i the team (1) prefetches the quadrature weights of the step whose transform
// finishes next, (2) waits for that transform (step i - NB, same ring slot),
// reads its outputs S_{nm}(b) through the position map and adds q_{nm}(b) S to
// the column's accumulators, which live in the team's registers (NA = K/(32 NQW)
// entries per thread) and are flushed into W after the chunk's last beta row,
// (3) streams the column of step i into the slot with cp.async.  The transform
// warps issue no global loads and hold no accumulators.  Columns are dealt
// x, x + G, ... so CTAs x and x + 1 read the two halves of each 32-byte sector
// at about the same time (the second is an L2 hit).
// ---------------------------------------------------------------------------
#ifndef SCV_GQP
#define SCV_GQP 1
#endif
// chunk between the pipelined synthesis passes transposed, C[m][bb * K + g] (k_pfa_rows_p
// GATHER = 5 writes it in row pairs), instead of [bb][g][m].  Measured (r02o): bit-identical
// results, but the alpha pass goes 82 -> 116 ms/map (its load/store warps become the
// bottleneck on the scattered sector writes) and the gamma+quadrature pass gains nothing
// (97.5 -> 96.0): its transform groups, not the column reads, bound it.  Off.
#ifndef SCV_SYN_PAIR
#define SCV_SYN_PAIR 0
#endif
#ifndef SCV_GQP_NQW
#define SCV_GQP_NQW 4
#endif
#ifndef SCV_GQP_NG
#define SCV_GQP_NG 4
#endif
// quadrature weights loaded one drain step ahead (1) or at the start of their step (0)
#ifndef SCV_GQP_WAHEAD
#define SCV_GQP_WAHEAD 0
#endif
#ifndef SCV_GQP_SETREG
#define SCV_GQP_SETREG 1
#endif
// Pacing of the team's refill: 64 warp copies to scattered slot positions issued back to back
// delay the transform warps' shared-memory traffic (the transforms run 31% slower next to the
// refill than alone, 12% in the row kernel whose copies are spread by its position-map reads).
// Sleeping SCV_GQP_PACE ns after every SCV_GQP_PACE_N copies spreads them; measured on the C4
// map (ms for this pass): off 97.1; 30 ns 92.1; 50 ns 87.6; 75 ns 103; 100 ns per 2 copies 90.
// Re-swept on the final kernels (r08q): 40 ns 83.6; 50 ns 83.9; 60 ns 84.5; 65 ns 101.9 (the
// team then bounds the pass); 100 ns per 2 copies 86.6.
#ifndef SCV_GQP_PACE
#define SCV_GQP_PACE 50
#endif
#ifndef SCV_GQP_PACE_N
#define SCV_GQP_PACE_N 1
#endif
// lengths whose column passes (k_ana_colgen_p, k_syn_gamma_qp) run as ring kernels
constexpr bool pfa_ring_cols(int K) { return K == 2047 || (K == 1023 && SCV_RING_1023); }
// lengths whose gamma+quadrature pass alone is a ring kernel
constexpr bool pfa_ring_gq(int K) { return pfa_ring_cols(K) || (K == 511 && SCV_RING_511); }
#ifndef SCV_GQP_PF
#define SCV_GQP_PF (2 + SCV_GQP_WAHEAD)
#endif
template <int K> struct PfaGqpCfg { static constexpr int NG = SCV_GQP_NG, NTG = 384 / SCV_GQP_NG, NQW = SCV_GQP_NQW, NB = 6; };
template <int K>
static constexpr size_t pfa_smem_gqp() {
  using PL = PfaPlan<K>;
  return ((size_t)pfa_tab_total<PL>() + (size_t)PfaGqpCfg<K>::NB * K) * sizeof(double2) +
         4 * (size_t)PfaGqpCfg<K>::NB * sizeof(unsigned long long);
}

template <int K>
__global__ void __launch_bounds__(PfaGqpCfg<K>::NG * PfaGqpCfg<K>::NTG + PfaGqpCfg<K>::NQW * 32, 1)
    k_syn_gamma_qp(int real, const double2* __restrict__ chunk, int b0, int nbb, const double* __restrict__ qtab,
                   int qrows, double2* __restrict__ wout, const double2* __restrict__ gtab) {
  using PL = PfaPlan<K>;
  constexpr int NG = PfaGqpCfg<K>::NG, NTG = PfaGqpCfg<K>::NTG, NQW = PfaGqpCfg<K>::NQW, NB = PfaGqpCfg<K>::NB;
  constexpr int NT = NG * NTG + NQW * 32, NQT = NQW * 32;
  constexpr int L = (K + 1) / 2;
  constexpr int NA = (K + NQT - 1) / NQT;
  extern __shared__ double2 sm[];
  double2* tab = sm;
  double2* const bufs = sm + pfa_tab_total<PL>();
  unsigned long long* const full = (unsigned long long*)(bufs + (size_t)NB * K);
  unsigned long long* const done = full + 2 * NB;  // barriers of alternate laps: see k_pfa_rows_p
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2 * NB; ++b) {
      mbar_init(full + b, NQT);
      mbar_init(done + b, 1);
    }
  }
  pfa_load_tables<PL, NT>(tab, gtab);
  // real: only the columns m >= 0 are transformed (see k_syn_gamma_q)
  const int NC = real ? L : K;
  const int mine = (int)blockIdx.x < NC ? (NC - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const long long ni = (long long)mine * nbb;
  if (ni == 0) return;
  // Register split between the roles (setmaxnreg moves registers between whole
  // warpgroups: threads 0..383 are the three transform warpgroups, 384..511 the
  // team): the transforms need 120 registers, the team holds 64 accumulator, 32
  // weight and 16 position registers per thread across steps.
  static_assert(!SCV_GQP_SETREG || (NG * NTG == 384 && NQT == 128), "setmaxnreg works on warpgroups of 128 threads");
  constexpr bool SETREG = SCV_GQP_SETREG && (K == 2047 || (K == 1023 && SCV_SETREG_1023));
  if (threadIdx.x >= NG * NTG) {
    if constexpr (SETREG) asm volatile("setmaxnreg.inc.sync.aligned.u32 152;\n");
    const int t = threadIdx.x - NG * NTG;
    constexpr int NH = NA / 2;
    static_assert(NQT == 128 && NA == 2 * NH && L == NH * NQT,
                  "entry u of thread t is frequency n = t + 128 u (u < NH) or -(K - t - 128 u) (u >= NH)");
    // Thread t owns the output frequencies gn = t + NQT u and the input samples
    // g = t + NQT u of every step, so their ring-slot positions are constants of
    // the thread: one packed register per u (low half = position of output gn,
    // high half = position of input sample g) instead of two position-map reads
    // per element per step.
    unsigned pp[NA];
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      const int gn = t + u * NQT;
      pp[u] = gn < K ? (unsigned)pfa_pos_tab<PL>(tab, gn) | ((unsigned)pfa_in_tab<PL>(tab, gn) << 16) : 0u;
    }
    const bool last_ok = t + (NA - 1) * NQT < K;  // gn = K does not exist (t = NQT - 1)
    double2 acc[NA];
    double qv[NA];
#pragma unroll
    for (int u = 0; u < NA; ++u) acc[u] = make_double2(0.0, 0.0);
    // quadrature weights of drain step e (column, beta row) into qv, and an L2
    // prefetch SCV_GQP_PF steps ahead (two runs of L - |m| doubles; the table is
    // streamed once per map, so the loads would otherwise wait on DRAM every step).
    // |n| of entry u is t + 128 u (n >= 0, u < NH) or K - t - 128 u (n < 0, u >= NH).
    // steps are (column index c, beta row bb) pairs, bb fastest; step (c, bb) exists iff c < mine
    auto load_weights = [&](int c, int bb) {
      const int col = (int)blockIdx.x + c * (int)gridDim.x;
      const long long b = b0 + bb;
      const int m = col <= L - 1 ? col : col - K;
      const int am = m < 0 ? -m : m;
      const double* qp = qtab + q_mbase(m, L, qrows) + b * (L - am) - am + t;            // + 128 u       (n >= 0)
      const double* qn = qtab + q_mbase(-m, L, qrows) + b * (L - am) - am + (K - t);     // - 128 u       (n < 0)
      const int lim = am - t;  // entry live iff |n| >= |m|
#pragma unroll
      for (int u = 0; u < NA / 2; ++u) qv[u] = NQT * u >= lim ? __ldg(qp + NQT * u) : 0.0;
#pragma unroll
      for (int u = NA / 2; u < NA; ++u) {
        const bool live = K - NQT * u - 2 * t >= lim && (u < NA - 1 || last_ok) && !(real && m == 0);
        qv[u] = live ? __ldg(qn - NQT * u) : 0.0;
      }
      int c2 = c, bb2 = bb + SCV_GQP_PF;
      while (bb2 >= nbb) {
        bb2 -= nbb;
        ++c2;
      }
      if (c2 < mine) {
        const int col2 = (int)blockIdx.x + c2 * (int)gridDim.x;
        const long long b2 = b0 + bb2;
        const int m2 = col2 <= L - 1 ? col2 : col2 - K;
        const int am2 = m2 < 0 ? -m2 : m2;
        const double* base = (t < 64 ? qtab + q_mbase(m2, L, qrows) : qtab + q_mbase(-m2, L, qrows)) + b2 * (L - am2);
        const int off = (t & 63) * 16;
        if (off < L - am2) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(base + off));
      }
    };
    long long st[6] = {0, 0, 0, 0, 0, 0}, st2[6] = {0, 0, 0, 0, 0, 0};
    PipeClk ck;
    const int nsteps = (int)ni;
    int slot = 0;
    unsigned uu = 0;             // use count of the current slot (lap of the ring)
    int dc = 0, db = 0;          // drain step (column index, beta row)
    int fc = 0, fb = 0;          // fill step
#pragma unroll 1
    for (int i = 0; i < nsteps + NB; ++i) {
      double2* const X = bufs + (size_t)slot * K;
      ck.mark(st, 4);
      PipeClk ck2;
      ck2.t = ck.t;
      if (SCV_GQP_WAHEAD && i == NB - 1) load_weights(0, 0);
      if (i >= NB) {
        if (!SCV_GQP_WAHEAD) {
          load_weights(dc, db);
          ck.mark(st, 3);
          ck2.mark(st2, 0);  // weight loads + prefetch issue
        }
        const int col = (int)blockIdx.x + dc * (int)gridDim.x;
        const int bb = db;
        const int m = col <= L - 1 ? col : col - K;
        mbar_wait(done + ((uu - 1) & 1) * NB + slot, ((uu - 1) >> 1) & 1);
        ck.mark(st, 2);
        ck2.mark(st2, 1);  // wait done
        // dead entries (|n| < |m|, gn = K, real n < 0 at m = 0) carry a zero weight; their
        // slot reads are valid positions
        {
          // q_{-l,m} = (-1)^{l+m} q_{l,-m}: for n < 0 the sign is (-1)^{|n|+m} = (-1)^{K-t+m} for every u >= NH
          // (128 u is even); real, n < 0: the weight of W(|n|, -m) is q_{|n|,-m} itself, applied to conj S
          const bool flip = !real && (((K - t) + m) & 1);
          double2 v[NA / 2];
#pragma unroll
          for (int u = 0; u < NA / 2; ++u) v[u] = X[pp[u] & 0xffffu];
#pragma unroll
          for (int u = 0; u < NA / 2; ++u) {
            acc[u].x = fma(v[u].x, qv[u], acc[u].x);
            acc[u].y = fma(v[u].y, qv[u], acc[u].y);
          }
#pragma unroll
          for (int u = 0; u < NA / 2; ++u) v[u] = X[pp[NA / 2 + u] & 0xffffu];
#pragma unroll
          for (int u = 0; u < NA / 2; ++u) {
            const double q = flip ? -qv[NA / 2 + u] : qv[NA / 2 + u];
            acc[NA / 2 + u].x = fma(v[u].x, q, acc[NA / 2 + u].x);
            acc[NA / 2 + u].y = fma(real ? -v[u].y : v[u].y, q, acc[NA / 2 + u].y);
          }
        }
        ck2.mark(st2, 2);  // accumulate
        if (bb == nbb - 1) {
          const int am = m < 0 ? -m : m;
#pragma unroll
          for (int u = 0; u < NA; ++u) {
            const int gn = t + u * NQT;
            const int n = gn <= L - 1 ? gn : gn - K;
            const int an = n < 0 ? -n : n;
            const double2 a = acc[u];
            acc[u] = make_double2(0.0, 0.0);
            if (gn >= K || an < am || (real && n < 0 && m == 0)) continue;
            double2* o = real ? wout + (long long)an * K + ((n < 0 ? -m : m) + L - 1)
                              : wout + ((long long)(n >= 0 ? 0 : 1) * L + an) * K + (m + L - 1);
            // one add per entry per launch, launches stream-ordered: deterministic
            atomicAdd(&o->x, a.x);
            atomicAdd(&o->y, a.y);
          }
        }
        grp_sync(1 + NG, NQT);  // the whole team has read the slot before anyone refills it
        ck.mark(st, 3);
        ck2.mark(st2, 3);  // flush + team barrier
        if (++db == nbb) {
          db = 0;
          ++dc;
        }
        if (SCV_GQP_WAHEAD && dc < mine) {
          load_weights(dc, db);
          ck.mark(st, 3);
          ck2.mark(st2, 0);  // weight loads + prefetch issue
        }
      }
      if (i < nsteps) {
        const int col = (int)blockIdx.x + fc * (int)gridDim.x;
        const int bb = fb;
        if (++fb == nbb) {
          fb = 0;
          ++fc;
        }
#if SCV_SYN_PAIR
        // transposed chunk C[m][r], r = bb * K + g, row pitch even (k_pfa_rows_p GATHER = 5)
        const double2* cp = chunk + (long long)col * (((long long)nbb * K + 1) & ~1LL) + (long long)bb * K + t;
        constexpr long long GS = NQT;
#else
        const double2* cp = chunk + (long long)bb * K * K + col + (long long)t * K;
        constexpr long long GS = (long long)NQT * K;
#endif
#pragma unroll
        for (int u = 0; u < NA; ++u) {
          if (u < NA - 1 || last_ok) cp_async16_m(X + (pp[u] >> 16), cp + GS * u);
#if SCV_GQP_PACE
          // spread the team's copies in time (a burst of 64 warp copies delays the transforms' shared loads)
          if ((u % SCV_GQP_PACE_N) == SCV_GQP_PACE_N - 1 && u < NA - 1) __nanosleep(SCV_GQP_PACE);
#endif
        }
        cp_async_mbar_arrive(full + (uu & 1) * NB + slot);
      }
      if (++slot == NB) {
        slot = 0;
        ++uu;
      }
    }
    ck.mark(st, 4);
    pipe_flush(st, 2, t == 0);
    pipe_flush(st2, 4, t == 0);
    return;
  }
  if constexpr (SETREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 120;\n");
  const int g = threadIdx.x / NTG, gtid = threadIdx.x - g * NTG, bar = 1 + g;
  long long st[6] = {0, 0, 0, 0, 0, 0};
  PipeClk ck;
#pragma unroll 1
  for (long long i = g; i < ni; i += NG) {
    const int slot = (int)(i % NB);
    const unsigned uu = (unsigned)(i / NB);
    mbar_wait(full + (uu & 1) * NB + slot, (uu >> 1) & 1);
    ck.mark(st, 0);
    pfa_dft<PL, -1, 1, NTG, K>(bufs + (size_t)slot * K, tab, nullptr, gtid, bar);
    if (gtid == 0) mbar_arrive(done + (uu & 1) * NB + slot);
    ck.mark(st, 1);
  }
  pipe_flush(st, 2, gtid == 0);
}

// real path: row(-n)[m] = (-1)^{m+n} conj(row(n)[-m]) for n > 0 (so3.py:379-382)
__global__ void k_wout_mirror(int L, double2* __restrict__ wout) {
  const int K = 2 * L - 1;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long tot = (long long)L * K;
  if (i >= tot) return;
  const int l = (int)(i / K), m = (int)(i - (long long)l * K) - (L - 1);
  if (l == 0) return;
  const int am = m < 0 ? -m : m;
  if (am > l) return;
  double2 v = wout[(long long)l * K + (L - 1) - m];
  v.y = -v.y;
  if ((m + l) & 1) v = make_double2(-v.x, -v.y);
  wout[((long long)L + l) * K + (L - 1) + m] = v;
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

// Position of output frequency k / input sample n in the D-dimensional
template <int K, int DIR, int GATHER>
static int launch_rows_p(scv_ctx* c, long long nrows, const double2* in, double2* out, const double2* tab, long long LK,
                         int b0, cudaStream_t s) {
  constexpr size_t smp = pfa_smem_pipe<K>();
  static_assert(smp <= 232448, "pipelined rows launch shape exceeds the 227 KB shared-memory limit");
  constexpr int NTB = pfa_pipe_threads<PfaPipeCfg<K>, K>();
  if constexpr (pfa_rows_sched(GATHER)) SCV_TRY(scv_pfa_tables_sched(c, K, &tab));  // same radix tables, scheduled maps
  int grid;
  SCV_TRY(persistent_grid(c, k_pfa_rows_p<K, DIR, GATHER>, NTB, smp, (nrows + PfaPipeCfg<K>::NG - 1) / PfaPipeCfg<K>::NG, &grid));
  k_pfa_rows_p<K, DIR, GATHER><<<grid, NTB, smp, s>>>(nrows, in, out, tab, LK, b0);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

// shared-memory layout (pfa.cuh, pfa_st): dimension s has stride st_s =
// p_{s+1}...p_{D-1}; output k sits at sum_s (k mod p_s) st_s, input n at
// sum_s (n * inv_s mod p_s) st_s with inv_s = (K/p_s)^{-1} mod p_s (Ruritanian map).
static void strides_of(const int f[4], int st[4]) {
  for (int s = 0; s < 4; ++s) {
    st[s] = 1;
    for (int t = s + 1; t < 4; ++t) st[s] *= f[t];
  }
}
int scv_pfa_pos_host(int K, int k) {
  int f[4], st[4];
  factors_of(K, f);
  strides_of(f, st);
  int a = 0;
  for (int s = 0; s < 4; ++s)
    if (f[s] > 1) a += (pfa_rader89(f[s]) ? r89_sigma(1, k % f[s]) : k % f[s]) * st[s];
  return a;
}
static int pfa_in_host(int K, int n) {
  int f[4], st[4];
  factors_of(K, f);
  strides_of(f, st);
  int a = 0;
  for (int s = 0; s < 4; ++s) {
    const int p = f[s];
    if (p == 1) continue;
    const int r = (K / p) % p;
    int inv = 1;
    while ((r * inv) % p != 1) ++inv;
    const int j = (int)(((long long)n * inv) % p);
    a += (pfa_rader89(p) ? r89_sigma(0, j) : j) * st[s];
  }
  return a;
}

// host-only view of the position maps (tests: the maps must reproduce the DFT
// under a plain emulation of the stages): out[k] and in[n], K entries each
extern "C" int scv_debug_pfa_maps(int K, int* out_pos, int* in_pos) {
  if (!scv_pfa_supported(K)) return SCV_EINVAL;
  for (int k = 0; k < K; ++k) {
    out_pos[k] = scv_pfa_pos_host(K, k);
    in_pos[k] = pfa_in_host(K, k);
  }
  return SCV_OK;
}
// sigma_in / sigma_out of the radix-89 storage order (89 entries each)
// lane schedule of the two maps (pfa_lane_schedule): entry [32 j + lane] = position | e << 11
extern "C" int scv_debug_pfa_sched(int K, int* out_sched, int* in_sched) {
  if (!scv_pfa_supported(K) || K > 2048) return SCV_EINVAL;
  std::vector<unsigned short> pos(2 * (size_t)K), sch(2 * (size_t)K);
  for (int k = 0; k < K; ++k) {
    pos[k] = (unsigned short)scv_pfa_pos_host(K, k);
    pos[K + k] = (unsigned short)pfa_in_host(K, k);
  }
  pfa_lane_schedule(pos.data(), K, sch.data());
  pfa_lane_schedule(pos.data() + K, K, sch.data() + K);
  for (int k = 0; k < K; ++k) {
    out_sched[k] = sch[k];
    in_sched[k] = sch[K + k];
  }
  return SCV_OK;
}
extern "C" int scv_debug_r89_sigma(int* sin, int* sout) {
  for (int j = 0; j < 89; ++j) {
    sin[j] = r89_sigma(0, j);
    sout[j] = r89_sigma(1, j);
  }
  return SCV_OK;
}

// TMA descriptor of a (K, nb, K) complex128 beta slab seen as doubles:
// dims (2K alpha-doubles, nb beta rows, K gamma), box (4, 1, 256) = one column
// pair of 256 gamma rows.  cuTensorMapEncodeTiled comes from the driver through
// the runtime's entry-point query (no libcuda link dependency).
static int scv_tma_map_slab(scv_ctx* c, const void* base, int K, int nb, CUtensorMap* map) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    SCV_CUDA(c, cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) return scv_fail(c, SCV_ECUDA, "cuTensorMapEncodeTiled unavailable");
    enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)2 * K, (cuuint64_t)nb, (cuuint64_t)K};
  const cuuint64_t strides[2] = {(cuuint64_t)K * 16, (cuuint64_t)nb * K * 16};
  const cuuint32_t box[3] = {4, 1, 256};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return scv_fail(c, SCV_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return SCV_OK;
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
  if constexpr (PfaPipeCfg<K>::NG > 0) return launch_rows_p<K, DIR, 0>(c, nrows, in, out, tab, 0, 0, s);
  if constexpr (PfaGrpCfg<K>::NG > 0) {
    constexpr size_t smg = pfa_smem_grp<K>();
    static_assert(smg <= 232448, "grouped rows launch shape exceeds the 227 KB shared-memory limit");
    constexpr int NTB = PfaGrpCfg<K>::NG * PfaGrpCfg<K>::NTG;
    int grid;
    SCV_TRY(persistent_grid(c, k_pfa_rows_g<K, DIR, 0>, NTB, smg, (nrows + PfaGrpCfg<K>::NG - 1) / PfaGrpCfg<K>::NG, &grid));
    k_pfa_rows_g<K, DIR, 0><<<grid, NTB, smg, s>>>(nrows, in, out, tab);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
    return SCV_OK;
  }
  constexpr size_t sm = pfa_smem<K, false>();
  static_assert(sm <= 232448, "prime-factor launch shape exceeds the 227 KB shared-memory limit");
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
  constexpr size_t sm = pfa_smem<K, false>();
  static_assert(sm <= 232448, "prime-factor launch shape exceeds the 227 KB shared-memory limit");
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
static int run_ana_colgen(scv_ctx* c, const double2* w, const double* hlb, const double* ls, const double* lc,
                          int b0, int nb, double2* out, cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  constexpr size_t sm = pfa_smem_g<K>();
  static_assert(sm <= 232448, "column-generation launch shape exceeds the 227 KB shared-memory limit");
  constexpr int L = (K + 1) / 2;
  const long long nt = (long long)nb * ((K + PfaGCfg<K>::R - 1) / PfaGCfg<K>::R);
  if constexpr (SCV_COLGEN_S && SCV_COLGEN_TMA && K == 2047) {
    constexpr size_t sms = pfa_smem_s<K>();
    static_assert(sms <= 232448, "staged column-generation launch shape exceeds the 227 KB shared-memory limit");
    static_assert((pfa_tab_total<PfaPlan<K>>() * sizeof(double2)) % 128 == 0, "TMA box source must be 128-byte aligned");
    CUtensorMap omap;
    SCV_TRY(scv_tma_map_slab(c, out, K, nb, &omap));
    const long long nts = (long long)((nb + PfaSCfg<K>::BB - 1) / PfaSCfg<K>::BB) * ((K + PfaSCfg<K>::R - 1) / PfaSCfg<K>::R);
    int grid;
    SCV_TRY(persistent_grid(c, k_ana_colgen_t<K>, PfaSCfg<K>::NT, sms, nts, &grid));
    k_ana_colgen_t<K><<<grid, PfaSCfg<K>::NT, sms, s>>>(w, hlb, ls, lc, b0, nb, omap, tab);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
    return SCV_OK;
  }
  if constexpr (SCV_COLGEN_S && K == 2047) {
    constexpr size_t sms = pfa_smem_s<K>();
    static_assert(sms <= 232448, "staged column-generation launch shape exceeds the 227 KB shared-memory limit");
    const long long nts = (long long)((nb + PfaSCfg<K>::BB - 1) / PfaSCfg<K>::BB) * ((K + PfaSCfg<K>::R - 1) / PfaSCfg<K>::R);
    int grid;
    SCV_TRY(persistent_grid(c, k_ana_colgen_s<K>, PfaSCfg<K>::NT, sms, nts, &grid));
    k_ana_colgen_s<K><<<grid, PfaSCfg<K>::NT, sms, s>>>(w, hlb, ls, lc, b0, nb, out, tab);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
    return SCV_OK;
  }
  int grid;
  SCV_TRY(persistent_grid(c, k_ana_colgen<K>, PfaGCfg<K>::NT, sm, nt, &grid));
  k_ana_colgen<K><<<grid, PfaGCfg<K>::NT, sm, s>>>(w, hlb, ls, lc, b0, nb, out, tab);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

template <int K>
static int run_ana_real_gf(scv_ctx* c, const double2* w, const double* hlb, const double* ls, const double* lc,
                           int b0, int nb, double2* T, double* out, cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  constexpr int L = (K + 1) / 2;
  {
    constexpr size_t sm = pfa_smem_g<K>();
    static_assert(sm <= 232448, "column-generation launch shape exceeds the 227 KB shared-memory limit");
    const long long nt = (long long)nb * ((L + PfaGCfg<K>::R - 1) / PfaGCfg<K>::R);
    int grid;
    SCV_TRY(persistent_grid(c, k_ana_colgen_real<K>, PfaGCfg<K>::NT, sm, nt, &grid));
    SCV_PROF(c, s, "so3inv_colgen");
    k_ana_colgen_real<K><<<grid, PfaGCfg<K>::NT, sm, s>>>(w, hlb, ls, lc, b0, nb, T, tab);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
  }
  if constexpr (PfaGrpCfg<K>::NG > 0) {
    constexpr size_t smg = pfa_smem_grp<K>();
    constexpr int NTB = PfaGrpCfg<K>::NG * PfaGrpCfg<K>::NTG;
    const long long nrows = (long long)K * nb;
    int grid;
    SCV_TRY(persistent_grid(c, k_pfa_rows_g<K, +1, 4>, NTB, smg, ((nrows + 1) / 2 + PfaGrpCfg<K>::NG - 1) / PfaGrpCfg<K>::NG, &grid));
    SCV_PROF(c, s, "so3inv_rows");
    k_pfa_rows_g<K, +1, 4><<<grid, NTB, smg, s>>>(nrows, T, (double2*)out, tab);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
    return SCV_OK;
  }
  {
    constexpr size_t sm = pfa_smem<K, false>();
    const long long nrows = (long long)K * nb;
    const long long nbt = (nrows + 2 * PfaCfg<K, false>::R - 1) / (2 * PfaCfg<K, false>::R);
    int grid;
    SCV_TRY(persistent_grid(c, k_rows_c2r<K>, PfaCfg<K, false>::NT, sm, nbt, &grid));
    SCV_PROF(c, s, "so3inv_rows");
    k_rows_c2r<K><<<grid, PfaCfg<K, false>::NT, sm, s>>>(nrows, T, out, tab);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
  }
  return SCV_OK;
}

template <int K>
static int run_ana_gamma(scv_ctx* c, int real, double2* src, double* dst, cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  constexpr size_t sm = pfa_smem<K, true>();
  static_assert(sm <= 232448, "prime-factor launch shape exceeds the 227 KB shared-memory limit");
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
static int run_syn_alpha(scv_ctx* c, int real, int tr, const void* in, int lsig, int b0, int nbb, double2* chunk,
                         cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  constexpr size_t sm = pfa_smem<K, false>();
  static_assert(sm <= 232448, "prime-factor launch shape exceeds the 227 KB shared-memory limit");
  // tr bit 2: the consumer is scv_pfa_syn_gamma_q (which may want its own chunk layout)
  const bool pair = (tr & 4) != 0;
  tr &= 3;
  (void)pair;
  if constexpr (PfaPipeCfg<K>::NG > 0) {
    if (!real && !tr) {
      const long long nrows = (long long)K * nbb;
      // the pipelined gamma+quadrature pass can read the chunk in column pairs
      if constexpr (pfa_ring_gq(K) && SCV_GQP && SCV_SYN_PAIR) {
        if (pair) return launch_rows_p<K, -1, 5>(c, nrows, (const double2*)in, chunk, tab, (long long)lsig * K, b0, s);
      }
      return launch_rows_p<K, -1, 1>(c, nrows, (const double2*)in, chunk, tab, (long long)lsig * K, b0, s);
    }
  }
  if constexpr (PfaGrpCfg<K>::NG > 0) {
    if (real == 2 && !tr) {
      constexpr size_t smg = pfa_smem_grp<K>();
      constexpr int NTB = PfaGrpCfg<K>::NG * PfaGrpCfg<K>::NTG;
      const long long nrows = (long long)K * nbb;
      int grid;
      SCV_TRY(persistent_grid(c, k_pfa_rows_g<K, -1, 3>, NTB, smg, ((nrows + 1) / 2 + PfaGrpCfg<K>::NG - 1) / PfaGrpCfg<K>::NG, &grid));
      k_pfa_rows_g<K, -1, 3><<<grid, NTB, smg, s>>>(nrows, (const double2*)in, chunk, tab, (long long)lsig * K, b0);
      c->launches++;
      SCV_CUDA(c, cudaGetLastError());
      return SCV_OK;
    }
    if (!real && !tr) {
      constexpr size_t smg = pfa_smem_grp<K>();
      constexpr int NTB = PfaGrpCfg<K>::NG * PfaGrpCfg<K>::NTG;
      const long long nrows = (long long)K * nbb;
      int grid;
      SCV_TRY(persistent_grid(c, k_pfa_rows_g<K, -1, 1>, NTB, smg, (nrows + PfaGrpCfg<K>::NG - 1) / PfaGrpCfg<K>::NG, &grid));
      k_pfa_rows_g<K, -1, 1><<<grid, NTB, smg, s>>>(nrows, (const double2*)in, chunk, tab, (long long)lsig * K, b0);
      c->launches++;
      SCV_CUDA(c, cudaGetLastError());
      return SCV_OK;
    }
  }
  const int rpb = real ? 2 * PfaCfg<K, false>::R : PfaCfg<K, false>::R;
  const long long nb = ((long long)K * nbb + rpb - 1) / rpb;
  int grid;
  SCV_TRY(persistent_grid(c, k_syn_alpha<K>, PfaCfg<K, false>::NT, sm, nb, &grid));
  k_syn_alpha<K><<<grid, PfaCfg<K, false>::NT, sm, s>>>(real, tr, in, lsig, b0, nbb, chunk, tab);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

template <int K>
static int run_syn_gamma(scv_ctx* c, int real, const double2* chunk, int b0, int nbb, double2* W1p, cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  constexpr size_t sm = pfa_smem<K, true>();
  static_assert(sm <= 232448, "prime-factor launch shape exceeds the 227 KB shared-memory limit");
  const long long nb = (long long)nbb * ((K + PfaCfg<K, true>::R - 1) / PfaCfg<K, true>::R);
  int grid;
  SCV_TRY(persistent_grid(c, k_syn_gamma<K>, PfaCfg<K, true>::NT, sm, nb, &grid));
  k_syn_gamma<K><<<grid, PfaCfg<K, true>::NT, sm, s>>>(real, chunk, b0, nbb, W1p, tab);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

template <int K>
static int run_syn_gamma_q(scv_ctx* c, int real, int tr, const double2* chunk, int b0, int nbb, const double* qtab,
                           const long long* mbase, int qrows, double2* wout, cudaStream_t s) {
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, K, &tab));
  if constexpr (pfa_ring_gq(K) && SCV_GQP) {
    if (!tr) {
      constexpr size_t smp = pfa_smem_gqp<K>();
      static_assert(smp <= 232448, "pipelined gamma+quadrature exceeds the 227 KB shared-memory limit");
      constexpr int NTP = PfaGqpCfg<K>::NG * PfaGqpCfg<K>::NTG + PfaGqpCfg<K>::NQW * 32;
      int grid;
      SCV_TRY(persistent_grid(c, k_syn_gamma_qp<K>, NTP, smp, real ? (K + 1) / 2 : K, &grid));
      k_syn_gamma_qp<K><<<grid, NTP, smp, s>>>(real, chunk, b0, nbb, qtab, qrows, wout, tab);
      c->launches++;
      SCV_CUDA(c, cudaGetLastError());
      return SCV_OK;
    }
  }
  constexpr size_t sm = pfa_smem_q<K>();
  static_assert(sm <= 232448, "gamma+quadrature launch shape exceeds the 227 KB shared-memory limit");
  int grid;
  SCV_TRY(persistent_grid(c, k_syn_gamma_q<K>, PfaQCfg<K>::NT, sm, (K + PfaQCfg<K>::RQ - 1) / PfaQCfg<K>::RQ, &grid));
  k_syn_gamma_q<K><<<grid, PfaQCfg<K>::NT, sm, s>>>(real, tr, chunk, b0, nbb, qtab, mbase, qrows, wout, tab);
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
// Blocked analysis (SCV_COLGEN_T = beta rows per block, 0 = off; env
// SCV_COLGEN_T overrides): per block of the slab [b0, b0+nb), k_ana_colgen_s
// writes the contiguous scratch T (65 KB per task row instead of 2047
// scattered 32-byte pieces) and k_pfa_rows_g<2047, +1, 2> gathers the alpha
// rows from T (async 32-byte pieces) into the signal.  Measured (r01v12):
// gamma pass 160 -> 144 ms/map, alpha pass 114 -> 118, map 563 -> 550 ms,
// +4.3 GB scratch at 64 rows per block.
// Returns 1 when not applicable (the caller runs colgen + rows in place).
#ifndef SCV_COLGEN_T
#define SCV_COLGEN_T 64
#endif
#ifndef SCV_COLGEN_T_4095
#define SCV_COLGEN_T_4095 16
#endif
static int ana_blocked_4095(scv_ctx* c, const double2* w, const double* hlb, const double* ls, const double* lc,
                            int b0, int nb, double2* sig, cudaStream_t s) {
  constexpr int KK = 4095, R = PfaGCfg<KK>::R, NPR = (KK + R - 1) / R;
  static_assert(R == 2, "the gather of k_pfa_rows<K, +1, 2> reads column pairs");
  const int blk = SCV_COLGEN_T_4095;
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, KK, &tab));
  void* T = nullptr;
  SCV_TRY(scv_scratch(c, 1, (size_t)blk * NPR * KK * R * 16, &T));
  constexpr size_t smc = pfa_smem_g<KK>();
  constexpr size_t smr = pfa_smem<KK, false>();
  constexpr int NTR = PfaCfg<KK, false>::NT, RR = PfaCfg<KK, false>::R;
  for (int bs0 = 0; bs0 < nb; bs0 += blk) {
    const int nbb = std::min(blk, nb - bs0);
    {
      SCV_PROF(c, s, "so3inv_colgen");
      int grid;
      SCV_TRY(persistent_grid(c, k_ana_colgen<KK, 1>, PfaGCfg<KK>::NT, smc, (long long)nbb * NPR, &grid));
      k_ana_colgen<KK, 1><<<grid, PfaGCfg<KK>::NT, smc, s>>>(w, hlb, ls, lc, b0 + bs0, nbb, (double2*)T, tab);
      c->launches++;
      SCV_CUDA(c, cudaGetLastError());
    }
    SCV_PROF(c, s, "so3inv_rows");
    const long long nrows = (long long)nbb * KK;
    if constexpr (PfaPipeCfg<KK>::NG > 0) {
      SCV_TRY((launch_rows_p<KK, +1, 2>(c, nrows, (const double2*)T, sig, tab, (long long)nb, bs0, s)));
    } else {
      int grid;
      SCV_TRY(persistent_grid(c, k_pfa_rows<KK, +1, 2>, NTR, smr, (nrows + RR - 1) / RR, &grid));
      k_pfa_rows<KK, +1, 2><<<grid, NTR, smr, s>>>(nrows, (const double2*)T, sig, tab, (long long)nb, bs0);
      c->launches++;
      SCV_CUDA(c, cudaGetLastError());
    }
  }
  return SCV_OK;
}

// rho32[a][l] = exp(h[l+32,a] - h[l,a]) (pitch L, l >= a, l + 32 < L) and
// sig32[b] = (sin(beta_b/2) cos(beta_b/2))^32 of k_ana_colgen_p, in long double
static int scv_colgen_tables(scv_ctx* c, int L, const double** rho, const double** sig) {
  const std::string kr = "rho32_" + std::to_string(L), ks = "sig32_" + std::to_string(L);
  auto it = c->aux.find(kr);
  if (it != c->aux.end()) {
    *rho = (const double*)it->second;
    *sig = (const double*)c->aux[ks];
    return SCV_OK;
  }
  const int K = 2 * L - 1;
  std::vector<ld> lf(2 * L + 2);
  lf[0] = 0.0L;
  for (int i = 1; i <= 2 * L + 1; ++i) lf[i] = lf[i - 1] + logl((ld)i);
  auto h = [&](int l, int a) { return 0.5L * (lf[2 * l] - lf[l + a] - lf[l - a]); };
  std::vector<double> r((size_t)L * L, 0.0), sg(L);
  for (int a = 0; a < L; ++a)
    for (int l = a; l + 32 < L; ++l) r[(size_t)a * L + l] = (double)expl(h(l + 32, a) - h(l, a));
  const ld pi = 3.141592653589793238462643383279502884L;
  for (int b = 0; b < L; ++b) {
    const int q = K - 2 * b - 1;  // cos(beta_b/2) = sin(pi q/(2K)), exactly 0 at beta = pi
    const ld sc = sinl(pi * (ld)(2 * b + 1) / (ld)(2 * K)) * (q == 0 ? 0.0L : sinl(pi * (ld)q / (ld)(2 * K)));
    sg[b] = (double)powl(sc, 32.0L);
  }
  double *dr = nullptr, *ds = nullptr;
  SCV_CUDA(c, cudaMalloc(&dr, r.size() * sizeof(double)));
  SCV_CUDA(c, cudaMalloc(&ds, sg.size() * sizeof(double)));
  SCV_CUDA(c, cudaMemcpy(dr, r.data(), r.size() * sizeof(double), cudaMemcpyHostToDevice));
  SCV_CUDA(c, cudaMemcpy(ds, sg.data(), sg.size() * sizeof(double), cudaMemcpyHostToDevice));
  c->aux[kr] = dr;
  c->aux[ks] = ds;
  const long long bytes = (long long)((r.size() + sg.size()) * sizeof(double));
  c->table_bytes += bytes;
  c->small_table_bytes += bytes;
  *rho = dr;
  *sig = ds;
  return SCV_OK;
}

template <int KK>
static int ana_blocked_ring(scv_ctx* c, int blk, const double2* w, const double* hlb, const double* ls, const double* lc,
                            int b0, int nb, double2* sig, cudaStream_t s) {
  constexpr int R = PfaSCfg<KK>::R, NPR = (KK + R - 1) / R;
  const double2* tab;
  SCV_TRY(scv_pfa_tables(c, KK, &tab));
  void* T = nullptr;
  const size_t tbytes = (size_t)blk * NPR * KK * R * 16;
  const size_t ctbytes = SCV_COLGENP ? (size_t)KK * KK * 16 : 0;
  SCV_TRY(scv_scratch(c, 1, tbytes + ctbytes, &T));
  const double *rho32 = nullptr, *sig32 = nullptr;
  double2* ct = (double2*)((char*)T + tbytes);
  if (SCV_COLGENP) {
    SCV_TRY(scv_colgen_tables(c, (KK + 1) / 2, &rho32, &sig32));
    SCV_PROF(c, s, "so3inv_colgen");
    const long long tot = (long long)KK * KK;
    k_colgen_ct<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>((KK + 1) / 2, w, hlb, ct);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
  }
  for (int bs0 = 0; bs0 < nb; bs0 += blk) {
    const int nbb = std::min(blk, nb - bs0);
    if constexpr (SCV_COLGENP) {
      SCV_PROF(c, s, "so3inv_colgen");
      constexpr size_t smp = pfa_smem_cgp<KK>();
      static_assert(smp <= 232448, "pipelined column generation exceeds the 227 KB shared-memory limit");
      constexpr int NTP = PfaCgpCfg<KK>::NG * PfaCgpCfg<KK>::NTG + PfaCgpCfg<KK>::NIO * 32;
      int grid;
      SCV_TRY(persistent_grid(c, k_ana_colgen_p<KK>, NTP, smp, (long long)NPR * nbb / 4 + 1, &grid));
      k_ana_colgen_p<KK><<<grid, NTP, smp, s>>>(ct, hlb, ls, lc, sig32, b0 + bs0, nbb, (double2*)T, tab);
      c->launches++;
      SCV_CUDA(c, cudaGetLastError());
    } else {
      SCV_PROF(c, s, "so3inv_colgen");
      constexpr size_t sms = pfa_smem_s<KK>();
      const long long nts = (long long)((nbb + PfaSCfg<KK>::BB - 1) / PfaSCfg<KK>::BB) * NPR;
      int grid;
      SCV_TRY(persistent_grid(c, k_ana_colgen_s<KK, 1>, PfaSCfg<KK>::NT, sms, nts, &grid));
      k_ana_colgen_s<KK, 1><<<grid, PfaSCfg<KK>::NT, sms, s>>>(w, hlb, ls, lc, b0 + bs0, nbb, (double2*)T, tab);
      c->launches++;
      SCV_CUDA(c, cudaGetLastError());
    }
    SCV_PROF(c, s, "so3inv_rows");
    const long long nrows = (long long)nbb * KK;
    if constexpr (PfaPipeCfg<KK>::NG > 0) {
      SCV_TRY((launch_rows_p<KK, +1, 2>(c, nrows, (const double2*)T, sig, tab, (long long)nb, bs0, s)));
    } else {
      static_assert(PfaGrpCfg<KK>::NG > 0, "the blocked analysis needs a row kernel with the pair gather");
      constexpr size_t smg = pfa_smem_grp<KK>();
      constexpr int NTB = PfaGrpCfg<KK>::NG * PfaGrpCfg<KK>::NTG;
      int grid;
      SCV_TRY(persistent_grid(c, k_pfa_rows_g<KK, +1, 2>, NTB, smg, (nrows + PfaGrpCfg<KK>::NG - 1) / PfaGrpCfg<KK>::NG, &grid));
      k_pfa_rows_g<KK, +1, 2><<<grid, NTB, smg, s>>>(nrows, (const double2*)T, sig, tab, (long long)nb, bs0);
      c->launches++;
      SCV_CUDA(c, cudaGetLastError());
    }
  }
  return SCV_OK;
}

int scv_pfa_ana_blocked(scv_ctx* c, int K, const double2* w, const double* hlb, const double* ls, const double* lc,
                        int b0, int nb, double2* sig, cudaStream_t s) {
  static const int blk = getenv("SCV_COLGEN_T") ? atoi(getenv("SCV_COLGEN_T")) : SCV_COLGEN_T;
  if (K == 4095 && SCV_COLGEN_T_4095 > 0) return ana_blocked_4095(c, w, hlb, ls, lc, b0, nb, sig, s);
  if (blk <= 0 || !SCV_COLGEN_S) return 1;
  if (K == 2047) return ana_blocked_ring<2047>(c, blk, w, hlb, ls, lc, b0, nb, sig, s);
  if constexpr (SCV_RING_1023 && SCV_COLGENP && PfaPipeCfg<1023>::NG > 0) {
    // four times the beta rows per block: the same scratch as at K = 2047
    if (K == 1023) return ana_blocked_ring<1023>(c, 4 * blk, w, hlb, ls, lc, b0, nb, sig, s);
  }
  return 1;
}

int scv_pfa_ana_colgen(scv_ctx* c, int K, const double2* w, const double* hlb, const double* ls, const double* lc,
                       int b0, int nb, double2* out, cudaStream_t s) {
#define CALL(KK) run_ana_colgen<KK>(c, w, hlb, ls, lc, b0, nb, out, s)
  PFA_SWITCH(K, CALL)
#undef CALL
}
int scv_pfa_ana_real_gf(scv_ctx* c, int K, const double2* w, const double* hlb, const double* ls, const double* lc,
                        int b0, int nb, double2* T, double* out, cudaStream_t s) {
#define CALL(KK) run_ana_real_gf<KK>(c, w, hlb, ls, lc, b0, nb, T, out, s)
  PFA_SWITCH(K, CALL)
#undef CALL
}
int scv_pfa_rows_inplace(scv_ctx* c, int K, int dir, long long nrows, double2* x, cudaStream_t s) {
  if (dir < 0) {
#define CALL(KK) run_rows<KK, -1>(c, nrows, x, x, s)
    PFA_SWITCH(K, CALL)
#undef CALL
  }
#define CALL(KK) run_rows<KK, +1>(c, nrows, x, x, s)
  PFA_SWITCH(K, CALL)
#undef CALL
}
int scv_pfa_ana_gamma(scv_ctx* c, int K, int real, double2* src, double* dst, cudaStream_t s) {
#define CALL(KK) run_ana_gamma<KK>(c, real, src, dst, s)
  PFA_SWITCH(K, CALL)
#undef CALL
}
int scv_pfa_syn_alpha(scv_ctx* c, int K, int real, int tr, const void* in, int lsig, int b0, int nbb,
                      double2* chunk, cudaStream_t s) {
#define CALL(KK) run_syn_alpha<KK>(c, real, tr, in, lsig, b0, nbb, chunk, s)
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

// b0 is relative to the first beta row of the table, which holds qrows rows
int scv_pfa_syn_gamma_q(scv_ctx* c, int K, int real, int tr, const double2* chunk, int b0, int nbb, const double* qtab,
                        const long long* mbase, int qrows, double2* wout, cudaStream_t s) {
  switch (K) {
    case 255: return run_syn_gamma_q<255>(c, real, tr, chunk, b0, nbb, qtab, mbase, qrows, wout, s);
    case 511: return run_syn_gamma_q<511>(c, real, tr, chunk, b0, nbb, qtab, mbase, qrows, wout, s);
    case 1023: return run_syn_gamma_q<1023>(c, real, tr, chunk, b0, nbb, qtab, mbase, qrows, wout, s);
    case 2047: return run_syn_gamma_q<2047>(c, real, tr, chunk, b0, nbb, qtab, mbase, qrows, wout, s);
    case 4095: return run_syn_gamma_q<4095>(c, real, tr, chunk, b0, nbb, qtab, mbase, qrows, wout, s);
    default: return scv_fail(c, SCV_EINVAL, "no gamma+quadrature kernel for length " + std::to_string(K));
  }
}

int scv_wout_mirror(scv_ctx* c, int L, double2* wout, cudaStream_t s) {
  const long long tot = (long long)L * (2 * L - 1);
  k_wout_mirror<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(L, wout);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}
