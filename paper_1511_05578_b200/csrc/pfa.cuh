// Prime-factor (Good-Thomas) DFT engine for the odd grid lengths K = 2^k - 1.
//
// Every sampling length of the lambda=2 tilings factors into coprime odd
// radices: 2047 = 23*89, 1023 = 31*33 (two DMMA stages; 3*11*31 until r08), 511 = 7*73, 255 = 3*5*17,
// 4095 = 9*13*35 (5*7*9*13 until r08), 63 = 7*9, 15 = 3*5; 3, 7, 31, 127 are prime.  Under the
// Ruritanian input map the K-point DFT is a p_1 x ... x p_d DFT with NO
// twiddle factors.  The rows stay in NATURAL order in shared memory for the
// whole transform:
//   * stage s (radix p) has K/p butterflies; butterfly b owns the positions
//     (b*p + j*(K/p)) mod K, j = 0..p-1, which are exactly the elements whose
//     dimension-s index is j and whose other indices are fixed (an element at
//     position n has dimension-s index (n * (K/p)^{-1}) mod p, so b*p has index
//     0 and adding K/p steps it by one).  Each stage transforms in place;
//   * after the last stage, output k sits at position
//     sum_s (k mod p_s) * (K/p_s) mod K  (the CRT map), read by pfa_pos().
// A stage butterfly is evaluated directly in the symmetric-pair form
//     y_k = A_k + DIR i B_k,  y_{p-k} = A_k - DIR i B_k,
//     A_k = x_0 + sum_j (x_j + x_{p-j}) cos(2 pi jk/p),
//     B_k =       sum_j (x_j - x_{p-j}) sin(2 pi jk/p),
// (p-1)^2 real FMAs per p points.  A work item is (row, butterfly, k-group of
// G output pairs); consecutive lanes take consecutive butterflies (odd
// position stride p -> bank-conflict-free 16-byte accesses) with a
// warp-uniform k-group, so the (cos, sin) pair of every (j, k) is ONE
// broadcast 16-byte shared load from a dense per-radix table.  All items of a
// stage are computed into registers before a barrier, then written back in
// place (no ping-pong buffer: 16 bytes of shared memory per element).
#pragma once
#include "scv_internal.cuh"

template <int K>
struct PfaPlan;  // D factors P0..P3 (1 = unused); NT/R tuned per length
#define SCV_PFA_PLAN(KK, DD, A, B, C, E)                                  \
  template <>                                                             \
  struct PfaPlan<KK> {                                                    \
    static constexpr int K = KK, D = DD, P0 = A, P1 = B, P2 = C, P3 = E;  \
  };
SCV_PFA_PLAN(3, 1, 3, 1, 1, 1)
SCV_PFA_PLAN(7, 1, 7, 1, 1, 1)
SCV_PFA_PLAN(15, 2, 3, 5, 1, 1)
SCV_PFA_PLAN(31, 1, 31, 1, 1, 1)
SCV_PFA_PLAN(63, 2, 7, 9, 1, 1)
SCV_PFA_PLAN(255, 3, 3, 5, 17, 1)
SCV_PFA_PLAN(511, 2, 7, 73, 1, 1)
// K = 1023: 0 = 3 * 11 * 31 (radices 3 and 11 on DFMA, 31 on DMMA); 1 = 33 * 31, 2 = 31 * 33 (two
// DMMA stages: the dense symmetric form only needs an odd radix, and 33 and 31 are coprime).
// A 1023-point transform took 11.6 k cycles in the ring kernels against 18.3 k for 2047 points
// (pipe counters, r08): three stages, two of them scalar, for a quarter of the FP64 work.
// Measured (r08, ms/map): C3 (L=512) 54.2 / 51.5 / 49.4 for plans 0 / 1 / 2, C4 334.0 / 331.8 /
// 331.8; round trips unchanged (4.1e-14, 9.4e-14).  Keeping the larger A fragments in registers
// (SCV_PFA_AREG_MAX 8 or 12) or the setmaxnreg split at K = 1023 (SCV_SETREG_1023): within noise.
#ifndef SCV_PLAN_1023
#define SCV_PLAN_1023 2
#endif
#if SCV_PLAN_1023 == 1
SCV_PFA_PLAN(1023, 2, 33, 31, 1, 1)
#elif SCV_PLAN_1023 == 2
SCV_PFA_PLAN(1023, 2, 31, 33, 1, 1)
#else
SCV_PFA_PLAN(1023, 3, 3, 11, 31, 1)
#endif
SCV_PFA_PLAN(2047, 2, 23, 89, 1, 1)
// K = 4095: 0 = 5 * 7 * 9 * 13 (5, 7 on DFMA; four stages, 484 bytes of spills in the row kernel);
// 1 = 35 * 9 * 13, 2 = 9 * 13 * 35, 4 = 13 * 9 * 35, 5 = 13 * 35 * 9 (three DMMA stages, no spills,
// 70 registers); 3 = 63 * 65 (does not fit the batched kernels' tables).  Measured on the C5
// streamed map (r08, ms/map): 5385 / 4216 / 4124 / 4189 / 4158 for plans 0 / 1 / 2 / 4 / 5, round
// trip 6.28e-13 throughout; ring shapes 128 / 256 / 384 threads per group with plan 2: 4255 / 4126 / 4119.
#ifndef SCV_PLAN_4095
#define SCV_PLAN_4095 2
#endif
#if SCV_PLAN_4095 == 1
SCV_PFA_PLAN(4095, 3, 35, 9, 13, 1)
#elif SCV_PLAN_4095 == 2
SCV_PFA_PLAN(4095, 3, 9, 13, 35, 1)
#elif SCV_PLAN_4095 == 3
SCV_PFA_PLAN(4095, 2, 63, 65, 1, 1)
#elif SCV_PLAN_4095 == 4
SCV_PFA_PLAN(4095, 3, 13, 9, 35, 1)
#elif SCV_PLAN_4095 == 5
SCV_PFA_PLAN(4095, 3, 13, 35, 9, 1)
#else
SCV_PFA_PLAN(4095, 4, 5, 7, 9, 13)
#endif

template <class PL, int S>
__host__ __device__ constexpr int pfa_p() {
  return S == 0 ? PL::P0 : S == 1 ? PL::P1 : S == 2 ? PL::P2 : PL::P3;
}
__host__ __device__ constexpr int pfa_h(int p) { return (p - 1) / 2; }
// output pairs per work item (k-group size) per radix
#ifndef SCV_PFA_G
#define SCV_PFA_G 6
#endif
__host__ __device__ constexpr int pfa_group(int p) { return pfa_h(p) < SCV_PFA_G ? pfa_h(p) : SCV_PFA_G; }
// padded number of output pairs (k-groups of G) for radix p
__host__ __device__ constexpr int pfa_gp(int p) { return p > 1 ? ((pfa_h(p) + pfa_group(p) - 1) / pfa_group(p)) * pfa_group(p) : 0; }
// Large radices (p >= 17) run on the FP64 tensor cores (DMMA m8n8k4, see
// pfa_stage_mma): their table is the pair of dense real matrices
// C[k][j] = cos(2 pi jk/p), S[k][j] = sin(2 pi jk/p), k = 0..M-1 (row 0 = the
// all-ones / all-zero row that produces y_0), j = 1..Kp, zero padded.
#ifndef SCV_MMA_MIN_RADIX
#define SCV_MMA_MIN_RADIX 17
#endif
// per length: K = 4095 = 5*7*9*13 runs its radices 9 and 13 on DMMA too
// (measured 48 vs 29 G points/s: the all-DFMA stages of 4095 spill), while
// 1023 keeps radix 11 on DFMA (66 vs 54 G points/s)
#ifndef SCV_MMA_MIN_RADIX_4095
#define SCV_MMA_MIN_RADIX_4095 9
#endif
__host__ __device__ constexpr bool pfa_use_mma(int p, int K) {
  return p >= (K == 4095 ? SCV_MMA_MIN_RADIX_4095 : SCV_MMA_MIN_RADIX);
}
// DMMA stage variant: 1 = warp-owned butterfly blocks (pfa_stage_mma_blk, no
// scratch), 0 = register-held 16x16 tiles / scratch-staged B (A/B builds)
#ifndef SCV_PFA_BLK
#define SCV_PFA_BLK 1
#endif
#ifndef SCV_PFA_KT_UNROLL
#define SCV_PFA_KT_UNROLL 11
#endif
constexpr int pfa_kt_unroll = SCV_PFA_KT_UNROLL;
#ifndef SCV_PFA_AREG
#define SCV_PFA_AREG 1
#endif
// largest A fragment (m8 tiles x k-steps, per matrix) a lane keeps in registers for a stage
#ifndef SCV_PFA_AREG_MAX
#define SCV_PFA_AREG_MAX 6
#endif
#ifndef SCV_PFA_SLOT_EVEN
#define SCV_PFA_SLOT_EVEN 1
#endif
#ifndef SCV_PFA_NBW_SMALL
#define SCV_PFA_NBW_SMALL 1
#endif
#ifndef SCV_PFA_NBW_BIG
#define SCV_PFA_NBW_BIG 1
#endif
__host__ __device__ constexpr int mma_M(int p) { return ((pfa_h(p) + 1 + 15) / 16) * 16; }   // output rows
__host__ __device__ constexpr int mma_Kp(int p) { return ((pfa_h(p) + 3) / 4) * 4; }         // reduction dim
__host__ __device__ constexpr int mma_pitch(int n) {  // row pitch (doubles) with pitch mod 16 in {4, 12}
  return (n % 16 == 4 || n % 16 == 12) ? n : (n % 16 < 4 ? n + (4 - n % 16) : n % 16 < 12 ? n + (12 - n % 16) : n + (20 - n % 16));
}
// A-operand layout of the DMMA stages.  SCV_PFA_A2 = 1 (experimental, with the
// warp-owned blocks; measured 1.5x SLOWER on B200 -- register pressure and
// spills in the 2047 kernels -- so off by default): the coefficients of k-steps 2q and 2q+1 of one A
// fragment are adjacent, C2[row][q][ac][kt & 1] (kt = 4-wide k-step, ac = lane
// & 3), so one 16-byte LDS feeds two k-steps; the row pitch is 8 mod 16
// doubles, which makes each 8-lane phase of the 16-byte loads cover all 32
// banks.  SCV_PFA_A2 = 0 (default): plain row-major [row][j], pitch 4|12 mod 16.
#ifndef SCV_PFA_A2
#define SCV_PFA_A2 0
#endif
// first operands of a warp's next block loaded under the current block's epilogue (block stage).
// Measured (r06q, C4): no spills, bit-identical, every K = 2047 pass 0.0-0.5 ms/map SLOWER
// (332.4 -> 333.9 ms/map): the start-of-block round trip is not what the warps wait on.  Off.
#ifndef SCV_PFA_PREFETCH
#define SCV_PFA_PREFETCH 0
#endif
#ifndef SCV_PFA_Q_UNROLL
#define SCV_PFA_Q_UNROLL 1
#endif
constexpr int pfa_q_unroll = SCV_PFA_Q_UNROLL;
static_assert(!SCV_PFA_A2 || SCV_PFA_BLK, "the paired A layout is implemented by the warp-owned block stage only");
__host__ __device__ constexpr int mma_pa(int p) {
  return SCV_PFA_A2 ? (((mma_Kp(p) + 7) / 8) * 8) % 16 == 0 ? ((mma_Kp(p) + 7) / 8) * 8 + 8 : ((mma_Kp(p) + 7) / 8) * 8
                    : mma_pitch(mma_Kp(p));
}
// offset (doubles) of coefficient (row, reduction index kk = j - 1) in a DMMA table
__host__ __device__ constexpr int mma_aoff(int p, int row, int kk) {
  return SCV_PFA_A2 ? row * mma_pa(p) + (kk / 8) * 8 + (kk % 4) * 2 + (kk / 4) % 2 : row * mma_pa(p) + kk;
}
// table size in double2 units: 1-D (cos, sin) table of p entries, or the two
// dense matrices (2 * M * pitch doubles = M * pitch double2)
// SCV_R89_PREPOS: the Rader stage reads its per-lane gather positions once per
// stage into registers instead of per block.  Measured (r01v25): column
// generation -0.7 ms/map, rows unchanged, gamma+quadrature +5.4 ms (the six
// extra registers spill there), so off by default.
#ifndef SCV_R89_PREPOS
#define SCV_R89_PREPOS 0
#endif
// Radix 89 by Rader + CRT (SCV_RADER89, see pfa_stage_rader89): the table is
// five small dense matrices (M0, M2: 16 x 12; Mc, RA, RB: 24 x 28 doubles)
// and the 44 Rader positions r_a = 3^a mod 89 as bytes.
#ifndef SCV_RADER89
#define SCV_RADER89 1
#endif
constexpr int R89_P12 = 12, R89_P28 = 28;
constexpr int R89_OFF_M2 = 16 * R89_P12, R89_OFF_MC = 2 * 16 * R89_P12, R89_OFF_RA = R89_OFF_MC + 24 * R89_P28,
              R89_OFF_RB = R89_OFF_RA + 24 * R89_P28, R89_OFF_RT = R89_OFF_RB + 24 * R89_P28;  // doubles
constexpr int R89_TAB = (R89_OFF_RT * 8 + 48 + 15) / 16;  // double2 units (+ 44 position bytes)
__host__ __device__ constexpr bool pfa_rader89(int p) { return SCV_RADER89 && p == 89; }
__host__ __device__ constexpr int pfa_tab(int p, int K) {
  return p <= 1 ? 0 : pfa_rader89(p) ? R89_TAB : pfa_use_mma(p, K) ? mma_M(p) * mma_pa(p) : p;
}
template <class PL>
__host__ __device__ constexpr int pfa_rtab_total() {
  return pfa_tab(PL::P0, PL::K) + pfa_tab(PL::P1, PL::K) + pfa_tab(PL::P2, PL::K) + pfa_tab(PL::P3, PL::K);
}
// followed by two 16-bit maps: out[k] = position of output frequency k,
// in[n] = position of input sample n (see pfa_st)
template <class PL>
__host__ __device__ constexpr int pfa_postab() { return (4 * PL::K + 15) / 16; }
template <class PL>
__host__ __device__ constexpr int pfa_tab_total() { return pfa_rtab_total<PL>() + pfa_postab<PL>(); }
// Shared-memory layout of a row during the transform: the D-dimensional array
// x[n_0][n_1]..[n_{D-1}] (row-major, n_s < p_s) of the Ruritanian input map,
// so dimension s has stride st_s = p_{s+1} * ... * p_{D-1} and stage s touches
// the elements base(c) + j * st_s of its K/p_s columns c (no modular index
// arithmetic inside the stages; the permutations live in two 16-bit tables).
template <class PL, int S>
__host__ __device__ constexpr int pfa_st() {
  return (S < 1 ? PL::P1 : 1) * (S < 2 ? PL::P2 : 1) * (S < 3 ? PL::P3 : 1);
}
template <class PL, int S>
__device__ __forceinline__ int pfa_base(int c) {
  constexpr int st = pfa_st<PL, S>(), p = pfa_p<PL, S>();
  if constexpr (st == 1) return c * p;
  else if constexpr (st * p == PL::K) return c;
  else return (c / st) * (st * p) + (c % st);
}
template <class PL, int S>
__host__ __device__ constexpr int pfa_tab_off() {
  return (S > 0 ? pfa_tab(PL::P0, PL::K) : 0) + (S > 1 ? pfa_tab(PL::P1, PL::K) : 0) + (S > 2 ? pfa_tab(PL::P2, PL::K) : 0);
}
// scratch (double2 units) for a DMMA stage over R rows: B matrices s and d
// (Kp x pitch(2*NBF padded to 16) doubles each) + x0 per butterfly
__host__ __device__ constexpr int mma_ncol(int K, int p, int R) { return ((2 * R * (K / p) + 15) / 16) * 16; }
// A DMMA stage keeps its accumulators in registers (pfa_stage_mma_reg, no
// scratch) when every warp of the NT-thread group owns at most
// SCV_PFA_TPW_MAX 16x16 output tiles; otherwise it stages B in scratch.
#ifndef SCV_PFA_TPW_MAX
#define SCV_PFA_TPW_MAX 2
#endif
__host__ __device__ constexpr int mma_tpw(int K, int p, int R, int NT) {
  return ((mma_M(p) / 16) * (mma_ncol(K, p, R) / 16) + NT / 32 - 1) / (NT / 32);
}
__host__ __device__ constexpr bool mma_reg(int K, int p, int R, int NT) { return mma_tpw(K, p, R, NT) <= SCV_PFA_TPW_MAX; }
__host__ __device__ constexpr int mma_scratch_p(int K, int p, int R, int NT) {
  return (p > 1 && pfa_use_mma(p, K) && !SCV_PFA_BLK && !mma_reg(K, p, R, NT)) ? mma_Kp(p) * mma_pitch(mma_ncol(K, p, R)) + R * (K / p) : 0;
}
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
template <class PL, int R, int NT>
__host__ __device__ constexpr int pfa_scratch() {
  return cmax(cmax(mma_scratch_p(PL::K, PL::P0, R, NT), mma_scratch_p(PL::K, PL::P1, R, NT)),
              cmax(mma_scratch_p(PL::K, PL::P2, R, NT), mma_scratch_p(PL::K, PL::P3, R, NT)));
}

// Coefficient tables (cos, sin)(2 pi i/p), i < p, per radix; staged once per
// CTA in shared memory (pfa_load_tables).  The butterfly walks j*k mod p
// incrementally (integer pipe) and reads each pair as a warp-broadcast
// 16-byte load.
// position of output k, from the shared table (one 2-byte load)
// (computed: sum_s (k mod p_s) st_s, constant divisors -> multiply-shift;
// SCV_PFA_POSTAB=1 reads the 16-bit table in shared memory instead)
#ifndef SCV_PFA_POSTAB
#define SCV_PFA_POSTAB 1
#endif
template <class PL>
__device__ __forceinline__ int pfa_pos_tab(const double2* tab, int k) {
  if constexpr (SCV_PFA_POSTAB) {
    return ((const unsigned short*)(tab + pfa_rtab_total<PL>()))[k];
  } else {
    int a = (k % PL::P0) * pfa_st<PL, 0>();
    if constexpr (PL::D > 1) a += (k % PL::P1) * pfa_st<PL, 1>();
    if constexpr (PL::D > 2) a += (k % PL::P2) * pfa_st<PL, 2>();
    if constexpr (PL::D > 3) a += (k % PL::P3) * pfa_st<PL, 3>();
    return a;
  }
}
// (K/p)^{-1} mod p
__host__ __device__ constexpr int pfa_inv(int K, int p) {
  int r = (K / p) % p, v = 1;
  while (p > 1 && (r * v) % p != 1) ++v;
  return v;
}
// position of input sample n (Ruritanian map), from the shared table
template <class PL>
__device__ __forceinline__ int pfa_in_tab(const double2* tab, int n) {
  if constexpr (SCV_PFA_POSTAB) {
    return ((const unsigned short*)(tab + pfa_rtab_total<PL>()))[PL::K + n];
  } else {
    constexpr int i0 = pfa_inv(PL::K, PL::P0), i1 = pfa_inv(PL::K, PL::P1);
    constexpr int i2 = pfa_inv(PL::K, PL::P2), i3 = pfa_inv(PL::K, PL::P3);
    int a = ((n * i0) % PL::P0) * pfa_st<PL, 0>();
    if constexpr (PL::D > 1) a += ((n * i1) % PL::P1) * pfa_st<PL, 1>();
    if constexpr (PL::D > 2) a += ((n * i2) % PL::P2) * pfa_st<PL, 2>();
    if constexpr (PL::D > 3) a += ((n * i3) % PL::P3) * pfa_st<PL, 3>();
    return a;
  }
}

// Stage the coefficient tables of this length into shared memory.
template <class PL, int NT>
__device__ __forceinline__ void pfa_load_tables(double2* tab, const double2* __restrict__ gtab) {
  for (int i = threadIdx.x; i < pfa_tab_total<PL>(); i += NT) tab[i] = gtab[i];
  __syncthreads();  // the load phase reads the position maps
}

// Accumulate k-group g (output pairs k = gG+1 .. gG+G) of one butterfly.
// Data loads are software-pipelined one j ahead; the G coefficient pairs of a
// j come from the shared table T (row stride GP) as broadcast loads.
template <int p, int G>
__device__ __forceinline__ void pfa_group_acc(const double2* __restrict__ T, const double2* __restrict__ Xr,
                                              int c0, double2 (&A)[G], double2 (&B)[G], double2& Z, int K,
                                              int step, int k0) {
  constexpr int h = (p - 1) / 2;
  const double2 x0 = Xr[c0];
  Z = x0;
#pragma unroll
  for (int t = 0; t < G; ++t) {
    A[t] = x0;
    B[t] = make_double2(0.0, 0.0);
  }
  int pa = c0 + step, pb = c0 + (p - 1) * step;
  double2 a = Xr[pa], bb = Xr[pb];
  // idx[t] = j*k_t mod p for k_t = gG+t+1 (zero-padded groups use k_t <= h guard at write time;
  // a k_t > h only produces unused accumulators)
  int idx[G];
#pragma unroll
  for (int t = 0; t < G; ++t) idx[t] = 0;
#pragma unroll 1
  for (int j = 1; j <= h; ++j) {
    pa += step;
    pb -= step;
    // prefetch the next j's data (software pipelining)
    double2 an = a, bn = bb;
    if (j < h) {
      an = Xr[pa];
      bn = Xr[pb];
    }
    const double2 s = make_double2(a.x + bb.x, a.y + bb.y);
    const double2 d = make_double2(a.x - bb.x, a.y - bb.y);
    Z.x += s.x;
    Z.y += s.y;
#pragma unroll
    for (int t = 0; t < G; ++t) {
      idx[t] += k0 + t;
      if (idx[t] >= p) idx[t] -= p;
      const double2 cs = T[idx[t]];
      A[t].x = fma(s.x, cs.x, A[t].x);
      A[t].y = fma(s.y, cs.x, A[t].y);
      B[t].x = fma(d.x, cs.y, B[t].x);
      B[t].y = fma(d.y, cs.y, B[t].y);
    }
    a = an;
    bb = bn;
  }
}

// cp.async 16-byte global -> shared copies (async prefetch of the next batch)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
// 8-byte variant (cp.async.ca: sizes below 16 go through L1)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
// same, with an L2 prefetch of the whole 128-byte line (strided column reads
// whose neighbouring columns are read by other CTAs at about the same time)
__device__ __forceinline__ void cp_async16_l2line(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

#ifdef SCV_PFA_NOINLINE
#define SCV_PFA_STAGE_INL __noinline__
#else
#define SCV_PFA_STAGE_INL __forceinline__
#endif
// Barrier over the NT threads of one work group (named barrier `bar`; bar 0 =
// __syncthreads when the group is the whole block).
__device__ __forceinline__ void grp_sync(int bar, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(nthreads) : "memory");
}

template <class PL, int S, int DIR, int R, int NT, int PITCH>
__device__ SCV_PFA_STAGE_INL void pfa_stage(double2* X, const double2* tab, int gtid = threadIdx.x, int bar = 0) {
  constexpr int p = pfa_p<PL, S>();
  constexpr int h = pfa_h(p);
  constexpr int K = PL::K;
  constexpr int step = pfa_st<PL, S>();
  constexpr int nbf = K / p;
  constexpr int G = pfa_group(p);
  constexpr int NG = (h + G - 1) / G;
  constexpr int items = R * nbf * NG;
  constexpr int IPT = (items + NT - 1) / NT;
  double2 A[IPT][G], B[IPT][G], Z[IPT];
  int pos[IPT], grp[IPT];
#pragma unroll
  for (int u = 0; u < IPT; ++u) {
    const int it = gtid + u * NT;
    grp[u] = -1;
    pos[u] = 0;
    if (IPT * NT > items && it >= items) continue;
    const int g = it / (R * nbf);
    const int rb = it - g * (R * nbf);
    const int r = rb / nbf, b = rb - r * nbf;
    const int c0 = pfa_base<PL, S>(b);
    grp[u] = g;
    pos[u] = r * PITCH + c0;
    pfa_group_acc<p, G>(tab + pfa_tab_off<PL, S>(), X + r * PITCH, c0, A[u], B[u], Z[u], K, step, g * G + 1);
  }
  grp_sync(bar, NT);
#pragma unroll
  for (int u = 0; u < IPT; ++u) {
    if (grp[u] < 0) continue;
    const int g = grp[u];
    const int rowoff = (pos[u] / PITCH) * PITCH;
    const int c0 = pos[u] - rowoff;
    double2* Xr = X + rowoff;
    if (g == 0) Xr[c0] = Z[u];
    int q1 = c0 + (g * G + 1) * step, q2 = c0 + (p - g * G - 1) * step;
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const int k = g * G + t + 1;
      if (k <= h) {
        const double2 iB = DIR < 0 ? make_double2(B[u][t].y, -B[u][t].x) : make_double2(-B[u][t].y, B[u][t].x);
        Xr[q1] = make_double2(A[u][t].x + iB.x, A[u][t].y + iB.y);
        Xr[q2] = make_double2(A[u][t].x - iB.x, A[u][t].y - iB.y);
      }
      q1 += step;
      q2 -= step;
    }
  }
  grp_sync(bar, NT);
}

// DMMA stage: batch of 2*R*K/p real columns (re/im of every butterfly).
//   prep : s_j = x_j + x_{p-j}, d_j = x_j - x_{p-j} into the B matrices Bs, Bd
//          [j-1][col] (col = 2*butterfly + {re, im}); x_0 saved per butterfly
//   GEMM : Acc_C = C . Bs,  Acc_S = S . Bd  with DMMA m8n8k4 (fp64 tensor core);
//          each warp owns 2x2 output tiles (16 k x 8 butterflies) for both
//   epil.: y_k = x0 + AccC + DIR i AccS,  y_{p-k} = x0 + AccC - DIR i AccS,
//          written in place (all of X was consumed by the prep).
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <class PL, int S, int DIR, int R, int NT, int PITCH>
__device__ __forceinline__ void pfa_stage_mma(double2* X, const double2* tab, double2* scr, int gtid, int bar) {
  constexpr int p = pfa_p<PL, S>();
  constexpr int h = pfa_h(p);
  constexpr int K = PL::K;
  constexpr int step = pfa_st<PL, S>();
  constexpr int nbf = K / p;
  constexpr int NBF = R * nbf;
  constexpr int M = mma_M(p), Kp = mma_Kp(p), PA = mma_pitch(Kp);
  constexpr int NCOL = mma_ncol(K, p, R), PB = mma_pitch(NCOL);
  const double* Cm = (const double*)(tab + pfa_tab_off<PL, S>());
  const double* Sm = Cm + M * PA;
  double* Bs = (double*)scr;
  double* Bd = Bs + Kp * PB;     // Bs, Bd: Kp*PB doubles each
  double2* x0s = scr + Kp * PB;  // NBF entries after Bs and Bd (2*Kp*PB doubles = Kp*PB double2)
  const int tid = gtid;
  // prep
  for (int i = tid; i < NBF * h; i += NT) {
    const int bf = i / h, j = i - bf * h + 1;
    const int r = bf / nbf, b = bf - r * nbf;
    const double2* Xr = X + r * PITCH;
    const int c0 = pfa_base<PL, S>(b);
    const int pa = c0 + j * step, pb = c0 + (p - j) * step;
    const double2 a = Xr[pa], bb = Xr[pb];
    Bs[(j - 1) * PB + 2 * bf] = a.x + bb.x;
    Bs[(j - 1) * PB + 2 * bf + 1] = a.y + bb.y;
    Bd[(j - 1) * PB + 2 * bf] = a.x - bb.x;
    Bd[(j - 1) * PB + 2 * bf + 1] = a.y - bb.y;
  }
  for (int bf = tid; bf < NBF; bf += NT) {
    const int r = bf / nbf, b = bf - r * nbf;
    x0s[bf] = X[r * PITCH + pfa_base<PL, S>(b)];
  }
  if constexpr (Kp > h) {
    for (int i = tid; i < (Kp - h) * PB; i += NT) {
      Bs[h * PB + i] = 0.0;
      Bd[h * PB + i] = 0.0;
    }
  }
  grp_sync(bar, NT);
  // GEMM + epilogue
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  constexpr int MB = M / 16, NB = NCOL / 16;
  const int ar = lane >> 2, ac = lane & 3;  // A fragment (row, col); B fragment (k = ac, n = ar)
  for (int blk = warp; blk < MB * NB; blk += NW) {
    const int mb = blk / NB, nb = blk - mb * NB;
    double acC[2][2][2], acS[2][2][2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        acC[u][v][0] = acC[u][v][1] = 0.0;
        acS[u][v][0] = acS[u][v][1] = 0.0;
      }
#pragma unroll 2
    for (int kt = 0; kt < Kp / 4; ++kt) {
      double aC[2], aS[2], bS[2], bD[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int row = mb * 16 + u * 8 + ar;
        aC[u] = Cm[row * PA + kt * 4 + ac];
        aS[u] = Sm[row * PA + kt * 4 + ac];
      }
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int col = nb * 16 + v * 8 + ar;
        bS[v] = Bs[(kt * 4 + ac) * PB + col];
        bD[v] = Bd[(kt * 4 + ac) * PB + col];
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          dmma(acC[u][v][0], acC[u][v][1], aC[u], bS[v]);
          dmma(acS[u][v][0], acS[u][v][1], aS[u], bD[v]);
        }
    }
    // epilogue: lane holds rows k = .. + ar, columns 2*ac, 2*ac+1 = (re, im) of butterfly nb*8+v*4+ac
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int k = mb * 16 + u * 8 + ar;
        const int bf = nb * 8 + v * 4 + ac;
        if (k > h || bf >= NBF) continue;
        const int r = bf / nbf, b = bf - r * nbf;
        double2* Xr = X + r * PITCH;
        const double2 x0 = x0s[bf];
        const double Ar = x0.x + acC[u][v][0], Ai = x0.y + acC[u][v][1];
        const int c0 = pfa_base<PL, S>(b);
        if (k == 0) {
          Xr[c0] = make_double2(Ar, Ai);
          continue;
        }
        const double Br = acS[u][v][0], Bi = acS[u][v][1];
        // DIR*i*B
        const double iBr = DIR < 0 ? Bi : -Bi, iBi = DIR < 0 ? -Br : Br;
        const int q1 = c0 + k * step, q2 = c0 + (p - k) * step;
        Xr[q1] = make_double2(Ar + iBr, Ai + iBi);
        Xr[q2] = make_double2(Ar - iBr, Ai - iBi);
      }
  }
  grp_sync(bar, NT);
}

// DMMA stage, register-held variant (default): the B fragments are formed
// directly from the row buffer (s_j, d_j of the lane's column computed from
// two 8-byte loads), every warp keeps the accumulators of its TPW tiles in
// registers across one barrier, then writes its outputs in place.  No scratch
// matrices, no prep pass; the A fragments (C, S) come from the shared table.
// Column col of the GEMM is (butterfly col/2, re|im col&1); butterfly b's
// element j sits at (b*p + j*K/p) mod K and element p-j at (b*p - j*K/p) mod K.
template <class PL, int S, int DIR, int R, int NT, int PITCH>
__device__ __forceinline__ void pfa_stage_mma_reg(double2* X, const double2* tab, int gtid, int bar) {
  constexpr int p = pfa_p<PL, S>();
  constexpr int h = pfa_h(p);
  constexpr int K = PL::K;
  constexpr int step = pfa_st<PL, S>();
  constexpr int nbf = K / p;
  constexpr int NBF = R * nbf;
  constexpr int M = mma_M(p), Kp = mma_Kp(p), PA = mma_pitch(Kp);
  constexpr int NCOL = mma_ncol(K, p, R);
  constexpr int MB = M / 16, NB = NCOL / 16, NTILE = MB * NB;
  constexpr int NW = NT / 32, TPW = (NTILE + NW - 1) / NW;
  const double* Cm = (const double*)(tab + pfa_tab_off<PL, S>());
  const double* Sm = Cm + M * PA;
  const double* Xd = (const double*)X;
  const int lane = gtid & 31, warp = gtid >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  double acC[TPW][2][2][2], acS[TPW][2][2][2];
  double2 x0[TPW][2];
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int blk = warp + t * NW;
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        acC[t][u][v][0] = acC[t][u][v][1] = 0.0;
        acS[t][u][v][0] = acS[t][u][v][1] = 0.0;
      }
    if (NTILE % NW != 0 && blk >= NTILE) continue;  // warp-uniform
    const int mb = blk / NB, nb = blk - mb * NB;
    // B-fragment columns of this lane: col = nb*16 + v*8 + ar
    int rowd[2], pa[2], pb[2];
    bool ok[2];
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int col = nb * 16 + v * 8 + ar;
      const int bf = col >> 1;
      ok[v] = bf < NBF;
      const int r = bf / nbf, b = bf - r * nbf;
      rowd[v] = 2 * r * PITCH + (col & 1);
      const int c0 = pfa_base<PL, S>(b);
      pa[v] = c0 + (ac + 1) * step;
      pb[v] = c0 + (p - ac - 1) * step;
      // x0 of the epilogue butterfly nb*8 + v*4 + ac
      const int bfe = nb * 8 + v * 4 + ac;
      const int re = bfe / nbf, be = bfe - re * nbf;
      x0[t][v] = bfe < NBF ? X[re * PITCH + pfa_base<PL, S>(be)] : make_double2(0.0, 0.0);
    }
#pragma unroll 2
    for (int kt = 0; kt < Kp / 4; ++kt) {
      const bool jin = (Kp == h) || (4 * kt + ac + 1 <= h);
      double bS[2], bD[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        double a = 0.0, bb = 0.0;
        if (ok[v] && jin) {
          a = Xd[rowd[v] + 2 * pa[v]];
          bb = Xd[rowd[v] + 2 * pb[v]];
        }
        bS[v] = a + bb;
        bD[v] = a - bb;
        pa[v] += 4 * step;
        pb[v] -= 4 * step;
      }
      double aC[2], aS[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int row = mb * 16 + u * 8 + ar;
        aC[u] = Cm[row * PA + kt * 4 + ac];
        aS[u] = Sm[row * PA + kt * 4 + ac];
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          dmma(acC[t][u][v][0], acC[t][u][v][1], aC[u], bS[v]);
          dmma(acS[t][u][v][0], acS[t][u][v][1], aS[u], bD[v]);
        }
    }
  }
  grp_sync(bar, NT);
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int blk = warp + t * NW;
    if (NTILE % NW != 0 && blk >= NTILE) continue;
    const int mb = blk / NB, nb = blk - mb * NB;
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int k = mb * 16 + u * 8 + ar;
        const int bf = nb * 8 + v * 4 + ac;
        if (k > h || bf >= NBF) continue;
        const int r = bf / nbf, b = bf - r * nbf;
        double2* Xr = X + r * PITCH;
        const double Ar = x0[t][v].x + acC[t][u][v][0], Ai = x0[t][v].y + acC[t][u][v][1];
        const int c0 = pfa_base<PL, S>(b);
        if (k == 0) {
          Xr[c0] = make_double2(Ar, Ai);
          continue;
        }
        const double Br = acS[t][u][v][0], Bi = acS[t][u][v][1];
        const double iBr = DIR < 0 ? Bi : -Bi, iBi = DIR < 0 ? -Br : Br;
        const int q1 = c0 + k * step, q2 = c0 + (p - k) * step;
        Xr[q1] = make_double2(Ar + iBr, Ai + iBi);
        Xr[q2] = make_double2(Ar - iBr, Ai - iBi);
      }
  }
  grp_sync(bar, NT);
}

// DMMA stage, warp-owned butterfly blocks (default).  A block is 4 butterflies
// (8 GEMM columns: re/im of each); ONE warp computes every output row k of its
// block (all ceil((h+1)/8) m8 tiles of C.s and S.d, accumulators in
// registers), then overwrites the block's own positions in place.  No other
// warp reads or writes those positions during the stage, so the only
// synchronisation is __syncwarp between the block's last read and first write
// and one barrier at the end of the stage (the next stage reads across
// blocks).  Warps stream through blocks with no block-wide barrier, so the
// DMMA chains of different warps (and CTAs) overlap freely.
// Block q covers butterflies {8g+o, 8g+o+4, 8g+o+2, 8g+o+6}, g = q/2, o = q&1 (see `slot`):
// butterfly positions 4 apart differ by 4 mod 8 doubles, so the two
// butterflies of each 16-lane phase of a B-fragment load hit disjoint banks.
template <class PL, int S, int DIR, int R, int NT, int PITCH, int XS = SCV_PFA_NBW_SMALL>
__device__ __forceinline__ void pfa_stage_mma_blk(double2* X, const double2* tab, int gtid, int bar) {
  constexpr int p = pfa_p<PL, S>();
  constexpr int h = pfa_h(p);
  constexpr int K = PL::K;
  constexpr int step = pfa_st<PL, S>();
  constexpr int nbf = K / p;
  constexpr int NBF = R * nbf;
  constexpr int M = mma_M(p), Kp = mma_Kp(p), PA = mma_pa(p);
  constexpr int M8 = (h + 1 + 7) / 8;          // m8 tiles covering k = 0..h
  constexpr int NBLK = 2 * ((NBF + 7) / 8);    // blocks of 4 (two per group of 8)
  constexpr int NW = NT / 32;
  const double* Cm = (const double*)(tab + pfa_tab_off<PL, S>());
  const double* Sm = Cm + M * PA;
  const double* Xd = (const double*)X;
  const int lane = gtid & 31, warp = gtid >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  // block-local butterfly slot i -> offset within the group of 8.  Butterfly bases are odd
  // multiples apart (step and p are odd), so offsets {0, 4} within a 16-lane phase keep the
  // 8-byte B-fragment loads on disjoint banks, and ALL-EVEN offsets {0, 4, 2, 6} (r02) also
  // make the eight lanes of a 16-byte epilogue store phase -- two output rows k x four
  // butterflies, bank group (offset + k) mod 8 -- conflict-free; the r01 offsets {0, 4, 1, 5}
  // collided two-way there (a twelfth of the row kernel's shared-memory wavefronts).
#if SCV_PFA_SLOT_EVEN
  auto slot = [](int i) { return 4 * (i & 1) + 2 * (i >> 1); };
#else
  auto slot = [](int i) { return (i >> 1) + 4 * (i & 1); };
#endif
  // small radices (<= 2 m8 tiles): NBW blocks per warp iteration, for more
  // independent DMMA chains per k-step
  constexpr int NBW = M8 <= 2 ? XS : SCV_PFA_NBW_BIG;
  // small radices: the lane's A fragments (M8 tiles x Kp/4 k-steps of C and S)
  // stay in registers for the whole stage; re-reading them per block is a
  // fifth of the transform's shared-memory traffic at K = 2047 (radix 23)
  constexpr bool AREG = SCV_PFA_AREG && !SCV_PFA_A2 && M8 * (Kp / 4) <= SCV_PFA_AREG_MAX;
  double aCr[AREG ? M8 : 1][AREG ? Kp / 4 : 1], aSr[AREG ? M8 : 1][AREG ? Kp / 4 : 1];
  if constexpr (AREG) {
#pragma unroll
    for (int t = 0; t < M8; ++t)
#pragma unroll
      for (int kt = 0; kt < Kp / 4; ++kt) {
        aCr[t][kt] = Cm[(t * 8 + ar) * PA + kt * 4 + ac];
        aSr[t][kt] = Sm[(t * 8 + ar) * PA + kt * 4 + ac];
      }
  }
  // B-fragment column of this lane in block q: butterfly slot ar>>1, component ar&1, and its
  // first two operands.  A slot past the last butterfly re-reads the last one (GEMM columns
  // are independent and that column is never stored), and the reduction indices
  // j = h+1..Kp of the zero-padded coefficient columns read the butterfly's own elements
  // j <= p-1 (finite data times exact zeros), so the operand loads need no predicates.
  auto first_operands = [&](int q, int& rowd_, int& pa_, int& pb_, double& an_, double& bn_) {
    const int gb = (q >> 1) * 8 + (SCV_PFA_SLOT_EVEN ? 1 : 2) * (q & 1);
    const int bfB = min(gb + slot(ar >> 1), NBF - 1);
    const int r = R == 1 ? 0 : bfB / nbf, b = bfB - r * nbf;
    const int c0 = pfa_base<PL, S>(b);
    rowd_ = 2 * r * PITCH + (ar & 1);
    pa_ = c0 + (ac + 1) * step;
    pb_ = c0 + (p - ac - 1) * step;
    // B operands software-pipelined one k-step ahead (the s/d formation of
    // step kt must not wait on its own shared loads)
    an_ = Xd[rowd_ + 2 * pa_];
    bn_ = Xd[rowd_ + 2 * pb_];
  };
  // SCV_PFA_PREFETCH: the first operands of the warp's NEXT block are loaded before the
  // epilogue stores of the current one (disjoint butterflies), so the next iteration does
  // not start with a shared-memory round trip
  int rowd[NBW], pa[NBW], pb[NBW];
  double an[NBW], bn[NBW];
  if constexpr (SCV_PFA_PREFETCH != 0) {
#pragma unroll
    for (int w = 0; w < NBW; ++w) first_operands(warp + w * NW, rowd[w], pa[w], pb[w], an[w], bn[w]);
  }
#pragma unroll 1
  for (int q0 = warp; q0 < NBLK; q0 += NW * NBW) {
    int eoff[NBW];
    bool okB[NBW], okE[NBW];
    double2 x0[NBW];
    double accC[NBW][M8][2], accS[NBW][M8][2];
#pragma unroll
    for (int w = 0; w < NBW; ++w) {
      const int q = q0 + w * NW;
      const int gb = (q >> 1) * 8 + (SCV_PFA_SLOT_EVEN ? 1 : 2) * (q & 1);
      okB[w] = true;
      if constexpr (SCV_PFA_PREFETCH == 0) first_operands(q, rowd[w], pa[w], pb[w], an[w], bn[w]);
      // epilogue butterfly of this lane: slot ac (accumulator columns 2ac, 2ac+1)
      const int bfE = gb + slot(ac);
      okE[w] = q < NBLK && bfE < NBF;
      eoff[w] = 0;
      x0[w] = make_double2(0.0, 0.0);
      if (okE[w]) {
        const int r = R == 1 ? 0 : bfE / nbf, b = bfE - r * nbf;
        eoff[w] = r * PITCH + pfa_base<PL, S>(b);
        x0[w] = X[eoff[w]];
      }
#pragma unroll
      for (int t = 0; t < M8; ++t) accC[w][t][0] = accC[w][t][1] = accS[w][t][0] = accS[w][t][1] = 0.0;
    }
#if SCV_PFA_A2
    // k-steps in pairs: one 16-byte A load per (tile, C|S) feeds steps 2q, 2q+1
    constexpr int KT = Kp / 4, KQ = (KT + 1) / 2;
#pragma unroll pfa_q_unroll
    for (int q = 0; q < KQ; ++q) {
      double2 aC2[M8], aS2[M8];
#pragma unroll
      for (int t = 0; t < M8; ++t) {
        const int off = (t * 8 + ar) * PA + q * 8 + ac * 2;
        aC2[t] = *(const double2*)(Cm + off);
        aS2[t] = *(const double2*)(Sm + off);
      }
#pragma unroll
      for (int two = 0; two < 2; ++two) {
        const int kt = 2 * q + two;
        if (KT % 2 == 1 && kt >= KT) break;
        double bS[NBW], bD[NBW];
#pragma unroll
        for (int w = 0; w < NBW; ++w) {
          const double a = an[w], bb = bn[w];
          pa[w] += 4 * step;
          pb[w] -= 4 * step;
          an[w] = 0.0;
          bn[w] = 0.0;
          if (kt + 1 < KT && okB[w] && ((Kp == h) || (4 * kt + 4 + ac + 1 <= h))) {
            an[w] = Xd[rowd[w] + 2 * pa[w]];
            bn[w] = Xd[rowd[w] + 2 * pb[w]];
          }
          bS[w] = a + bb;
          bD[w] = a - bb;
        }
#pragma unroll
        for (int t = 0; t < M8; ++t) {
          const double aC = two ? aC2[t].y : aC2[t].x;
          const double aS = two ? aS2[t].y : aS2[t].x;
#pragma unroll
          for (int w = 0; w < NBW; ++w) {
            dmma(accC[w][t][0], accC[w][t][1], aC, bS[w]);
            dmma(accS[w][t][0], accS[w][t][1], aS, bD[w]);
          }
        }
      }
    }
#else
#pragma unroll pfa_kt_unroll
    for (int kt = 0; kt < Kp / 4; ++kt) {
      double bS[NBW], bD[NBW];
#pragma unroll
      for (int w = 0; w < NBW; ++w) {
        const double a = an[w], bb = bn[w];
        pa[w] += 4 * step;
        pb[w] -= 4 * step;
        if (kt + 1 < Kp / 4) {
          an[w] = Xd[rowd[w] + 2 * pa[w]];
          bn[w] = Xd[rowd[w] + 2 * pb[w]];
        }
        bS[w] = a + bb;
        bD[w] = a - bb;
      }
#pragma unroll
      for (int t = 0; t < M8; ++t) {
        const int row = t * 8 + ar;
        double aC, aS;
        if constexpr (AREG) {
          aC = aCr[t][kt];
          aS = aSr[t][kt];
        } else {
          aC = Cm[row * PA + kt * 4 + ac];
          aS = Sm[row * PA + kt * 4 + ac];
        }
#pragma unroll
        for (int w = 0; w < NBW; ++w) {
          dmma(accC[w][t][0], accC[w][t][1], aC, bS[w]);
          dmma(accS[w][t][0], accS[w][t][1], aS, bD[w]);
        }
      }
    }
#endif
    __syncwarp();
    if constexpr (SCV_PFA_PREFETCH != 0) {
      if (q0 + NW * NBW < NBLK) {
#pragma unroll
        for (int w = 0; w < NBW; ++w)
          first_operands(q0 + NW * NBW + w * NW, rowd[w], pa[w], pb[w], an[w], bn[w]);
      }
    }
#pragma unroll
    for (int w = 0; w < NBW; ++w) {
      if (!okE[w]) continue;
      double2* Xr = X + eoff[w];
#pragma unroll
      for (int t = 0; t < M8; ++t) {
        const int k = t * 8 + ar;
        if (k > h) continue;
        const double Ar = x0[w].x + accC[w][t][0], Ai = x0[w].y + accC[w][t][1];
        if (k == 0) {
          Xr[0] = make_double2(Ar, Ai);
          continue;
        }
        const double Br = accS[w][t][0], Bi = accS[w][t][1];
        const double iBr = DIR < 0 ? Bi : -Bi, iBi = DIR < 0 ? -Br : Br;
        Xr[k * step] = make_double2(Ar + iBr, Ai + iBi);
        Xr[(p - k) * step] = make_double2(Ar - iBr, Ai - iBi);
      }
    }
    __syncwarp();
  }
  grp_sync(bar, NT);
}

// Radix-89 stage by Rader's algorithm with a 4 x 11 CRT split, on the FP64
// tensor cores.  With r_a = 3^a mod 89 (3 is a primitive root; a < 44 picks one
// of each pair {j, 89-j}), s'_a = x_{r_a} + x_{89-r_a}, d'_a = x_{r_a} - x_{89-r_a}:
//   A'_b = sum_a cos(2 pi r_a r_b / 89) s'_a   (44-point cyclic correlation),
//   B'_b = sum_a sin(2 pi r_a r_b / 89) d'_a   (44-point negacyclic correlation),
//   y_{r_b} = x0 + A'_b + DIR i B'_b,  y_{89-r_b} = x0 + A'_b - DIR i B'_b,  y_0 = x0 + sum s'.
// a <-> (a mod 4, a mod 11) turns each correlation into a 2-D one; a 4-point
// transform along a mod 4 (cyclic DFT for A', sign-twisted odd DFT for B', done
// in-lane: each lane holds all four a mod 4 of its a mod 11 values) leaves
// dense 11 x 11 (real) / 22 x 22 (complex as real) products on the tensor
// cores: 66 DMMA per 4 butterflies instead of the 132 of the dense symmetric
// form (pfa_stage_mma_blk).  The matrices are built on the host in long double
// (pfa.cu) and checked end to end against torch.fft (tools/fftbench.py).
// Warp-owned blocks of 4 butterflies as in pfa_stage_mma_blk.  Lane (ar, ac):
// B-fragment column ar (butterfly slot(ar>>1), component ar&1) holding the
// a mod 11 = ac + 4 kt values; epilogue butterfly slot(ac), output rows ar.
//
// Storage order of the 89 elements of a butterfly (r02).  Radix 89 is the
// innermost dimension (stride 1), and every other reader / writer of the row
// buffer goes through the 16-bit position maps, so the order of a butterfly's
// 89 elements in shared memory is free.  It is chosen so that this stage needs
// no permutation at run time:
//   * INPUT element j sits at r89_sigma_in(j): 0 for j = 0; for the pair
//     a = (33 a1 + 12 a2) mod 44 the two elements (u_a, v_a) sit at
//     1 + (11 a1 + a2) and 45 + (11 a1 + a2), where (u_a, v_a) = (r_a, 89 - r_a)
//     if the negacyclic wrap sign of a is + and (89 - r_a, r_a) if it is -, so
//     the twisted difference is always x_u - x_v.  A lane's 4 x 2 gather of a
//     k-step is eight 8-byte loads at compile-time offsets from one base, and
//     the 16 lanes of a shared-memory phase cover 128 contiguous bytes.
//   * OUTPUT y_k sits at r89_sigma_out(k): 0 for k = 0; for b = (33 b1 +
//     12 b2) mod 44 the outputs x0 + A'_b + DIR i B and x0 + A'_b - DIR i B go
//     to 1 + t and 45 + t, t = 2 b2 + (b1 & 1) + 22 (b1 >> 1) (B without the
//     wrap sign: the + output is y_{r_b} if the sign of b is +, y_{89-r_b}
//     otherwise).  The eight lanes of a 16-byte store phase hit eight different
//     16-byte bank groups.
// The host builds the position maps with the same two functions (pfa.cu).
// y_0 = x0 + sum_a s'_a comes out of the tensor core as well: row 11 of the
// first 11 x 11 matrix (padding until r02) is all ones.
__host__ __device__ constexpr int r89_in_slot(int a1, int a2) { return 11 * a1 + a2; }
__host__ __device__ constexpr int r89_out_slot(int b1, int b2) { return 2 * b2 + (b1 & 1) + 22 * (b1 >> 1); }
// SCV_R89_NBW blocks of 4 butterflies per warp iteration: the lane's A fragments of the five
// Rader matrices (66 eight-byte loads per block, more than half of the stage's shared-memory
// wavefronts) are loaded once per iteration and feed every block of it.  Costs 26 accumulator
// and 8 operand doubles per extra block, so it needs a launch shape that leaves the transform
// threads the registers (see PfaPipeCfg).
#ifndef SCV_R89_NBW
#define SCV_R89_NBW 1
#endif
template <class PL, int S, int DIR, int R, int NT, int PITCH, int XW = SCV_R89_NBW>
__device__ __forceinline__ void pfa_stage_rader89(double2* X, const double2* tab, int gtid, int bar) {
  constexpr int p = 89;
  constexpr int K = PL::K;
  static_assert(pfa_st<PL, S>() == 1, "the Rader storage order needs radix 89 as the innermost dimension");
  static_assert(SCV_PFA_POSTAB == 1, "the Rader storage order lives in the position tables");
  constexpr int nbf = K / p;
  constexpr int NBF = R * nbf;
  constexpr int NBLK = 2 * ((NBF + 7) / 8);
  constexpr int NW = NT / 32;
  constexpr int NBW = XW;
  const double* T0 = (const double*)(tab + pfa_tab_off<PL, S>());
  const double* Xd = (const double*)X;
  const int lane = gtid & 31, warp = gtid >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  constexpr double s2 = 0.70710678118654752440;
  auto slot = [](int i) { return (i >> 1) + 4 * (i & 1); };
  const bool a2ok = ac < 3;  // a mod 11 = ac + 8 exists in the third k-step
#pragma unroll 1
  for (int q0 = warp; q0 < NBLK; q0 += NW * NBW) {
    const double* xg[NBW];
    bool okE[NBW];
    int eoff[NBW];
    double2 x0[NBW];
    // ---- per k-step kt (a2 = ac + 4 kt): gather, in-lane 4-point transforms,
    // and the tensor-core products of that k-step (the Im halves of the 22 x 22
    // products are k-step kt + 3), so only one k-step of B operands is live
    double y0[NBW][2][2], y2[NBW][2][2], yu[NBW][3][2], za[NBW][3][2], zb[NBW][3][2];
#pragma unroll
    for (int w = 0; w < NBW; ++w) {
      const int q = q0 + w * NW;
      const int gb = (q >> 1) * 8 + 2 * (q & 1);
      // B-fragment butterfly of this lane; a block past the end re-reads the last
      // butterfly (its GEMM columns are independent and never stored)
      const int bfB = min(gb + slot(ar >> 1), NBF - 1);
      {
        const int rr = R == 1 ? 0 : bfB / nbf, b = bfB - rr * nbf;
        xg[w] = Xd + 2 * (rr * PITCH + b * p + 1 + ac) + (ar & 1);
      }
      const int bfE = gb + slot(ac);
      okE[w] = q < NBLK && bfE < NBF;
      eoff[w] = 0;
      x0[w] = make_double2(0.0, 0.0);
      if (okE[w]) {
        const int rr = R == 1 ? 0 : bfE / nbf, b = bfE - rr * nbf;
        eoff[w] = rr * PITCH + b * p;
        x0[w] = X[eoff[w]];
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) y0[w][t][0] = y0[w][t][1] = y2[w][t][0] = y2[w][t][1] = 0.0;
#pragma unroll
      for (int t = 0; t < 3; ++t)
        yu[w][t][0] = yu[w][t][1] = za[w][t][0] = za[w][t][1] = zb[w][t][0] = zb[w][t][1] = 0.0;
    }
#pragma unroll
    for (int kt = 0; kt < 3; ++kt) {
      double bV0[NBW], bV2[NBW], bUr[NBW], bUi[NBW], bAr[NBW], bAi[NBW], bBr[NBW], bBi[NBW];
#pragma unroll
      for (int w = 0; w < NBW; ++w) {
        double sv[4], dv[4];
#pragma unroll
        for (int a1 = 0; a1 < 4; ++a1) {
          double xu = 0.0, xv = 0.0;
          if (kt < 2 || a2ok) {
            xu = xg[w][2 * (r89_in_slot(a1, 4 * kt))];
            xv = xg[w][2 * (r89_in_slot(a1, 4 * kt) + 44)];
          }
          sv[a1] = xu + xv;
          dv[a1] = xu - xv;
        }
        bV0[w] = (sv[0] + sv[2]) + (sv[1] + sv[3]);
        bV2[w] = (sv[0] + sv[2]) - (sv[1] + sv[3]);
        bUr[w] = sv[0] - sv[2];
        bUi[w] = sv[1] - sv[3];
        const double P = (dv[1] - dv[3]) * s2, Q = (dv[1] + dv[3]) * s2;
        bAr[w] = dv[0] + P;
        bAi[w] = -dv[2] - Q;
        bBr[w] = dv[0] - P;
        bBi[w] = dv[2] - Q;
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int o = (t * 8 + ar) * R89_P12 + kt * 4 + ac;
        const double a0 = T0[o], a2 = T0[R89_OFF_M2 + o];
#pragma unroll
        for (int w = 0; w < NBW; ++w) {
          dmma(y0[w][t][0], y0[w][t][1], a0, bV0[w]);
          dmma(y2[w][t][0], y2[w][t][1], a2, bV2[w]);
        }
      }
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int o = (t * 8 + ar) * R89_P28 + kt * 4 + ac;
        const double c0 = T0[R89_OFF_MC + o], c1 = T0[R89_OFF_MC + o + 12];
        const double ra0 = T0[R89_OFF_RA + o], ra1 = T0[R89_OFF_RA + o + 12];
        const double rb0 = T0[R89_OFF_RB + o], rb1 = T0[R89_OFF_RB + o + 12];
#pragma unroll
        for (int w = 0; w < NBW; ++w) {
          dmma(yu[w][t][0], yu[w][t][1], c0, bUr[w]);
          dmma(yu[w][t][0], yu[w][t][1], c1, bUi[w]);
          dmma(za[w][t][0], za[w][t][1], ra0, bAr[w]);
          dmma(za[w][t][0], za[w][t][1], ra1, bAi[w]);
          dmma(zb[w][t][0], zb[w][t][1], rb0, bBr[w]);
          dmma(zb[w][t][0], zb[w][t][1], rb1, bBi[w]);
        }
      }
    }
    // rows 3..5 of the third product tile hold the Im parts of b2 = 8..10
    double uhi[NBW][2], ahi[NBW][2], bhi[NBW][2];
#pragma unroll
    for (int w = 0; w < NBW; ++w)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uhi[w][c] = __shfl_down_sync(0xffffffffu, yu[w][2][c], 12);
        ahi[w][c] = __shfl_down_sync(0xffffffffu, za[w][2][c], 12);
        bhi[w][c] = __shfl_down_sync(0xffffffffu, zb[w][2][c], 12);
      }
    __syncwarp();
#pragma unroll
    for (int w = 0; w < NBW; ++w) {
      if (!okE[w]) continue;
      double2* Xr = X + eoff[w];
      // y_0: row 11 of the first product (the all-ones row) is sum_a s'_a
      if (ar == 3) Xr[0] = make_double2(x0[w].x + y0[w][1][0], x0[w].y + y0[w][1][1]);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if (hh == 1 && ar >= 3) continue;
        // per component c (0 = re, 1 = im of the butterfly); x0 rides on Y0
        double Aq[4][2], Bq[4][2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const double Y0 = y0[w][hh][c] + (c ? x0[w].y : x0[w].x), Y2 = y2[w][hh][c];
          const double Yr = hh ? yu[w][2][c] : yu[w][0][c], Yi = hh ? uhi[w][c] : yu[w][1][c];
          const double ZAr = hh ? za[w][2][c] : za[w][0][c], ZAi = hh ? ahi[w][c] : za[w][1][c];
          const double ZBr = hh ? zb[w][2][c] : zb[w][0][c], ZBi = hh ? bhi[w][c] : zb[w][1][c];
          Aq[0][c] = (Y0 + Y2) + Yr;
          Aq[1][c] = (Y0 - Y2) + Yi;
          Aq[2][c] = (Y0 + Y2) - Yr;
          Aq[3][c] = (Y0 - Y2) - Yi;
          Bq[0][c] = ZAr + ZBr;
          Bq[1][c] = ((ZAr + ZAi) + (ZBi - ZBr)) * s2;
          Bq[2][c] = ZAi - ZBi;
          Bq[3][c] = ((ZAi - ZAr) + (ZBr + ZBi)) * s2;
        }
        double2* Xo = Xr + 1 + 2 * (hh * 8 + ar);
#pragma unroll
        for (int b1 = 0; b1 < 4; ++b1) {
          const int t = r89_out_slot(b1, 0);
          // DIR i B
          const double iBr = DIR < 0 ? Bq[b1][1] : -Bq[b1][1], iBi = DIR < 0 ? -Bq[b1][0] : Bq[b1][0];
          Xo[t] = make_double2(Aq[b1][0] + iBr, Aq[b1][1] + iBi);
          Xo[t + 44] = make_double2(Aq[b1][0] - iBr, Aq[b1][1] - iBi);
        }
      }
    }
    __syncwarp();
  }
  grp_sync(bar, NT);
}

// In-place K-point DFT (sign DIR) of R rows at X[r*PITCH + n] (natural order
// in; CRT order out, read through pfa_pos).  Caller syncs before (data ready).
// scr: pfa_scratch<PL,R,NT>() double2 of shared scratch (DMMA stages).
// XW, XS: blocks per warp iteration of the Rader-89 stage and of the small-radix block stage
// (kernels whose transform threads have the registers raise them, see PfaPipeCfg)
template <class PL, int S, int DIR, int R, int NT, int PITCH, int XW = SCV_R89_NBW, int XS = SCV_PFA_NBW_SMALL>
__device__ __forceinline__ void pfa_stage_any(double2* X, const double2* tab, double2* scr, int gtid, int bar) {
  constexpr int p = pfa_p<PL, S>();
  if constexpr (pfa_rader89(p)) pfa_stage_rader89<PL, S, DIR, R, NT, PITCH, XW>(X, tab, gtid, bar);
  else if constexpr (pfa_use_mma(p, PL::K) && SCV_PFA_BLK) pfa_stage_mma_blk<PL, S, DIR, R, NT, PITCH, XS>(X, tab, gtid, bar);
  else if constexpr (pfa_use_mma(p, PL::K) && mma_reg(PL::K, p, R, NT)) pfa_stage_mma_reg<PL, S, DIR, R, NT, PITCH>(X, tab, gtid, bar);
  else if constexpr (pfa_use_mma(p, PL::K)) pfa_stage_mma<PL, S, DIR, R, NT, PITCH>(X, tab, scr, gtid, bar);
  else pfa_stage<PL, S, DIR, R, NT, PITCH>(X, tab, gtid, bar);
}

// gtid/bar: thread index within the work group of NT threads and its named
// barrier (defaults: the whole block, barrier 0).
#ifndef SCV_EXP_SKIP_STAGES
#define SCV_EXP_SKIP_STAGES 0
#endif
template <class PL, int DIR, int R, int NT, int PITCH, int XW = SCV_R89_NBW, int XS = SCV_PFA_NBW_SMALL>
__device__ __forceinline__ void pfa_dft(double2* X, const double2* tab, double2* scr, int gtid = threadIdx.x,
                                        int bar = 0) {
  // SCV_EXP_SKIP_STAGES (timing experiments only, wrong results): bit s skips stage s
  if constexpr (!(SCV_EXP_SKIP_STAGES & 1)) pfa_stage_any<PL, 0, DIR, R, NT, PITCH, XW, XS>(X, tab, scr, gtid, bar);
  if constexpr (PL::D > 1 && !(SCV_EXP_SKIP_STAGES & 2)) pfa_stage_any<PL, 1, DIR, R, NT, PITCH, XW, XS>(X, tab, scr, gtid, bar);
  if constexpr (PL::D > 2 && !(SCV_EXP_SKIP_STAGES & 4)) pfa_stage_any<PL, 2, DIR, R, NT, PITCH, XW, XS>(X, tab, scr, gtid, bar);
  if constexpr (PL::D > 3 && !(SCV_EXP_SKIP_STAGES & 8)) pfa_stage_any<PL, 3, DIR, R, NT, PITCH, XW, XS>(X, tab, scr, gtid, bar);
}

// Out-of-line variant: isolates the transform's register allocation from a
// large calling kernel (used by the fused beta stage).
template <class PL, int DIR, int R, int NT, int PITCH>
__device__ __noinline__ void pfa_dft_ool(double2* X, const double2* tab, double2* scr) {
  pfa_dft<PL, DIR, R, NT, PITCH>(X, tab, scr, threadIdx.x, 0);
}

// host side (pfa.cu)
int scv_pfa_tables(scv_ctx* c, int K, const double2** out);  // device copy of the tables
bool scv_pfa_supported(int K);
