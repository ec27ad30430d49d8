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


// ---------------------------------------------------------------------------
// The same table as two dense matrix products on the FP64 tensor cores (r02;
// k_betaq_build above stays as the cross-check, SCV_BETAQ_BUILD=0).
//
// Columns are the pairs (m, l) of one parity par = (-1)^{l+m}; c(-m') = par c(m'),
// so only m' >= 0 is kept:
//   U_e(m'') = sum_{m' >= 0, m' == m'' (2)} T_par[m''][m'] c(m'),
//              T_par[m''][m'] = w(m''-m') + par w(m''+m')  (m' > 0),  w(m'')  (m' = 0),
//              w(d) = 2 / (1 - d^2)                                   -> GEMM 1 (two parity blocks)
//   Q(b)     = sum_{m'' >= 0} G_par[b][m''] U_e(m''),
//              even: G = (2 - [m''=0]) cos(m'' beta_b), row L-1 = (1 - [m''=0]/2) (-1)^{m''};
//              odd : G = sin(m'' beta_b), row L-1 = 0                 -> GEMM 2
//   q(b)     = (2f, 4f) (+-1) Q(b) per column (k_bq_scatter), and for odd parity
//              q(L-1) from sum_{m''} (-1)^{m''} (c(m''-1) - c(m''+1)), which telescopes to
//              2 (-1)^{L-1} c(L-1) (non-zero for l = L-1 only).
// 3 L^4 flops in all (3.3e12 at L = 1024) instead of L^4 dependent shared-memory
// multiply-adds with a division each.  Work is batched over LB consecutive
// degrees l; within a batch the columns are ordered m-major, l fastest.
// Matrices are stored with the even indices first, then the odd ones, each block
// padded to a multiple of 64.
// ---------------------------------------------------------------------------
constexpr int GT_J = 64, GT_I = 128, GT_K = 16, GT_NT = 256, GT_ST = 3;
constexpr int GT_PW = GT_K + 4, GT_PX = GT_I + 4;  // row pitches (doubles), 4 mod 16: conflict-free fragments
constexpr size_t GT_SMEM = (size_t)GT_ST * (GT_J * GT_PW + GT_K * GT_PX) * sizeof(double);

__device__ __forceinline__ void bq_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void bq_cp16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem));
}

// D[j][i] = sum_k W[j][k] X[k][i]; W (J x Kd, pitch ldw), X (Kd x I, pitch ldx), D (J x I, pitch ldd), all
// row-major doubles; J % 64 == I % 128 == Kd % 16 == 0, pitches even.  CTA tile 64 x 128, 8 warps of 32 x 32
// (4 x 4 DMMA m8n8k4 tiles), 3-stage cp.async pipeline over k.
__global__ void __launch_bounds__(GT_NT, 2) k_bq_gemm(int Kd, const double* __restrict__ W, int ldw,
                                                     const double* __restrict__ X, long long ldx,
                                                     double* __restrict__ D, long long ldd) {
  extern __shared__ double smg[];
  double* Ws = smg;                             // [ST][64][PW]
  double* Xs = smg + GT_ST * GT_J * GT_PW;      // [ST][16][PX]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const int wj = warp >> 2, wi = warp & 3;
  const long long i0 = (long long)blockIdx.x * GT_I;
  const int j0 = blockIdx.y * GT_J;
  const int nk = Kd / GT_K;
  auto load = [&](int kt, int st) {
    const int k0 = kt * GT_K;
    // W tile: 64 rows x 16 doubles = 512 chunks of 16 bytes
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int ch = t + q * GT_NT, row = ch >> 3, c2 = (ch & 7) * 2;
      bq_cp16(Ws + (st * GT_J + row) * GT_PW + c2, W + (long long)(j0 + row) * ldw + k0 + c2);
    }
    // X tile: 16 rows x 128 doubles = 1024 chunks
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ch = t + q * GT_NT, row = ch >> 6, c2 = (ch & 63) * 2;
      bq_cp16(Xs + (st * GT_K + row) * GT_PX + c2, X + (long long)(k0 + row) * ldx + i0 + c2);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int s = 0; s < GT_ST - 1; ++s) {
    if (s < nk) load(s, s);
    else asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GT_ST - 2));
    __syncthreads();  // tile kt has landed; everyone is done with the stage refilled next
    if (kt + GT_ST - 1 < nk) load(kt + GT_ST - 1, (kt + GT_ST - 1) % GT_ST);
    else asm volatile("cp.async.commit_group;\n" ::);
    const double* ws = Ws + ((kt % GT_ST) * GT_J + wj * 32) * GT_PW;
    const double* xs = Xs + (kt % GT_ST) * GT_K * GT_PX + wi * 32;
#pragma unroll
    for (int kk = 0; kk < GT_K; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = ws[(mt * 8 + ar) * GT_PW + kk + ac];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) b[nt] = xs[(kk + ac) * GT_PX + nt * 8 + ar];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) bq_dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
    }
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      double* o = D + (long long)(j0 + wj * 32 + mt * 8 + ar) * ldd + i0 + wi * 32 + nt * 8 + 2 * ac;
      *(double2*)o = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
    }
}

// row index of m'' (or m') in the even-first storage
__host__ __device__ __forceinline__ int bq_row(int mi, int LeP) { return (mi & 1) ? LeP + (mi >> 1) : (mi >> 1); }

// T_par blocks: T[row(m'')][j] for m' = 2 j + sub, same parity sub as m''; pitch LP
__global__ void k_bq_build_T(int L, int LeP, int LP, int par, double* __restrict__ T) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)LP * LP) return;
  const int row = (int)(idx / LP), j = (int)(idx - (long long)row * LP);
  const int sub = row >= LeP;
  const int mpp = sub ? 2 * (row - LeP) + 1 : 2 * row;
  const int mp = 2 * j + sub;
  double v = 0.0;
  if (mpp < L && mp < L) {
    const double d1 = (double)(mpp - mp), d2 = (double)(mpp + mp);
    v = mp == 0 ? 2.0 / (1.0 - d1 * d1) : 2.0 / (1.0 - d1 * d1) + (double)par * (2.0 / (1.0 - d2 * d2));
  }
  T[idx] = v;
}
// G_par[b][row(m'')], pitch LP, JP rows
__global__ void k_bq_build_G(int L, int LeP, int LP, int JP, int par, int qb0, int qnb, const double* __restrict__ trig,
                             double* __restrict__ G) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)JP * LP) return;
  const int K = 2 * L - 1;
  const int row = (int)(idx / LP), col = (int)(idx - (long long)row * LP);
  const int b = row < qnb ? qb0 + row : L;  // rows past the range are zero
  const int sub = col >= LeP;
  const int mpp = sub ? 2 * (col - LeP) + 1 : 2 * col;
  double v = 0.0;
  if (mpp < L && b < L) {
    if (b < L - 1) {
      const int j = (int)(((long long)(2 * b + 1) * mpp) % (2 * K));
      v = par > 0 ? (mpp == 0 ? 1.0 : 2.0) * trig[2 * j] : trig[2 * j + 1];
    } else {
      v = par > 0 ? (mpp == 0 ? 0.5 : 1.0) * ((mpp & 1) ? -1.0 : 1.0) : 0.0;
    }
  }
  G[idx] = v;
}
// C[row(m')][i] = Delta^l_{m'm} Delta^l_{m'l} of column i = (m, l); zero for m' > l and for padding
__global__ void k_bq_cmat(int L, int LeP, int LP, const double* __restrict__ delta, const int2* __restrict__ cols, int NC,
                          long long NCP, double* __restrict__ C) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = blockIdx.y;
  if (i >= NCP) return;
  const int sub = row >= LeP;
  const int mp = sub ? 2 * (row - LeP) + 1 : 2 * row;
  double v = 0.0;
  if (i < NC && mp < L) {
    const int2 ml = cols[i];
    if (mp <= ml.y) v = wedge_get(delta, ml.y, mp, ml.x) * wedge_get(delta, ml.y, mp, ml.y);
  }
  C[(long long)row * NCP + i] = v;
}
// q[mbase(m) + b (L-|m|) + (l-|m|)] from Q[b][i]
__global__ void k_bq_scatter(int L, double pref, int par, int qb0, const double* __restrict__ delta,
                             const int2* __restrict__ cols, int NC, long long NCP, const double* __restrict__ Qm,
                             const long long* __restrict__ mbase, double* __restrict__ q) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = qb0 + blockIdx.y;
  const double* Q = Qm - (long long)qb0 * NCP;  // Q[b][i] with b the absolute beta row
  if (i >= NC) return;
  const int K = 2 * L - 1;
  const int m = cols[i].x, l = cols[i].y;
  const int am = m < 0 ? -m : m;
  const int mn = m - l;
  const double f = pref / (double)K;
  double v;
  if (par > 0) {
    v = 2.0 * f * (((mn / 2) & 1) ? -Q[(long long)b * NCP + i] : Q[(long long)b * NCP + i]);
  } else if (b < L - 1) {
    const int e = (mn - 1) / 2;
    v = 4.0 * f * ((e & 1) ? -Q[(long long)b * NCP + i] : Q[(long long)b * NCP + i]);
  } else {
    double to = 0.0;
    if (l == L - 1) {
      to = 2.0 * wedge_get(delta, l, L - 1, m) * wedge_get(delta, l, L - 1, l);
      if ((L - 1) & 1) to = -to;
    }
    const int e = (mn + 1) / 2;
    v = f * 0.5 * SCV_PI * ((((e % 2) + 2) % 2) ? -to : to);
  }
  q[mbase[m + L - 1] + (long long)(b - qb0) * (L - am) + (l - am)] = v;
}

static int bq_round(int x, int m) { return (x + m - 1) / m * m; }

}  // namespace

bool scv_betaq_enabled(int L) {
  static const char* e = getenv("SCV_BETAQ");
  if (e && e[0] == '0') return false;
  return L >= 2;
}

// GEMM formulation of the build (see above): fills dq (L^3 doubles, bases dmb).
static int betaq_fill_gemm(scv_ctx* c, int L, int qb0, int qnb, cudaStream_t s, double* dq, const long long* dmb,
                           const double* dtrig) {
  const int K = 2 * L - 1;
  const int Le = (L + 1) / 2, Lo = L / 2;
  const int LeP = bq_round(Le, 64), LoP = bq_round(std::max(Lo, 1), 64), LP = LeP + LoP, JP = bq_round(qnb, 64);
  const int LB = L <= 1024 ? 32 : 16;  // degrees per batch (scratch: 3 x LP x NCP doubles)
  // column lists of every (batch, parity), m-major with l fastest
  struct Batch { int la, lb, par; size_t off; int nc; };
  std::vector<Batch> batches;
  std::vector<int2> cols;
  int ncmax = 0;
  for (int la = 0; la < L; la += LB) {
    const int lb = std::min(L, la + LB);
    for (int par = 1; par >= -1; par -= 2) {
      Batch b{la, lb, par, cols.size(), 0};
      for (int m = -(lb - 1); m <= lb - 1; ++m)
        for (int l = std::max(std::abs(m), la); l < lb; ++l)
          if ((((l + m) & 1) != 0) == (par < 0)) cols.push_back(make_int2(m, l));
      b.nc = (int)(cols.size() - b.off);
      ncmax = std::max(ncmax, b.nc);
      if (b.nc) batches.push_back(b);
    }
  }
  const long long NCPmax = bq_round(ncmax, GT_I);
  double *T[2] = {nullptr, nullptr}, *G[2] = {nullptr, nullptr}, *C = nullptr, *U = nullptr, *Q = nullptr;
  int2* dcols = nullptr;
  auto cleanup = [&]() {
    for (int i = 0; i < 2; ++i) {
      cudaFree(T[i]);
      cudaFree(G[i]);
    }
    cudaFree(C);
    cudaFree(U);
    cudaFree(Q);
    cudaFree(dcols);
  };
#define BQ_CUDA(x)                     \
  do {                                 \
    cudaError_t bqe_ = (x);            \
    if (bqe_ != cudaSuccess) {         \
      cleanup();                       \
      SCV_CUDA(c, bqe_);               \
    }                                  \
  } while (0)
  for (int i = 0; i < 2; ++i) {
    BQ_CUDA(cudaMalloc(&T[i], (size_t)LP * LP * sizeof(double)));
    BQ_CUDA(cudaMalloc(&G[i], (size_t)JP * LP * sizeof(double)));
  }
  BQ_CUDA(cudaMalloc(&C, (size_t)LP * NCPmax * sizeof(double)));
  BQ_CUDA(cudaMalloc(&U, (size_t)LP * NCPmax * sizeof(double)));
  BQ_CUDA(cudaMalloc(&Q, (size_t)JP * NCPmax * sizeof(double)));
  BQ_CUDA(cudaMalloc(&dcols, cols.size() * sizeof(int2)));
  BQ_CUDA(cudaMemcpyAsync(dcols, cols.data(), cols.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
  BQ_CUDA(cudaFuncSetAttribute(k_bq_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GT_SMEM));
  for (int i = 0; i < 2; ++i) {
    const int par = i == 0 ? 1 : -1;
    k_bq_build_T<<<(unsigned)(((long long)LP * LP + 255) / 256), 256, 0, s>>>(L, LeP, LP, par, T[i]);
    k_bq_build_G<<<(unsigned)(((long long)JP * LP + 255) / 256), 256, 0, s>>>(L, LeP, LP, JP, par, qb0, qnb, dtrig, G[i]);
    c->launches += 2;
  }
  BQ_CUDA(cudaGetLastError());
  const double pref = 4.0 * SCV_PI * SCV_PI / ((double)K * (double)K);
  for (const Batch& b : batches) {
    const int pi = b.par > 0 ? 0 : 1;
    const long long NCP = bq_round(b.nc, GT_I);
    const int2* bc = dcols + b.off;
    k_bq_cmat<<<dim3((unsigned)((NCP + 255) / 256), LP), 256, 0, s>>>(L, LeP, LP, c->delta, bc, b.nc, NCP, C);
    // GEMM 1, even and odd m'' blocks; the reduction stops at the batch's largest degree
    const int kde = bq_round((b.lb - 1) / 2 + 1, GT_K), kdo = bq_round(b.lb / 2, GT_K);
    k_bq_gemm<<<dim3((unsigned)(NCP / GT_I), LeP / GT_J), GT_NT, GT_SMEM, s>>>(kde, T[pi], LP, C, NCP, U, NCP);
    if (kdo > 0)
      k_bq_gemm<<<dim3((unsigned)(NCP / GT_I), LoP / GT_J), GT_NT, GT_SMEM, s>>>(
          kdo, T[pi] + (size_t)LeP * LP, LP, C + (size_t)LeP * NCP, NCP, U + (size_t)LeP * NCP, NCP);
    else
      BQ_CUDA(cudaMemsetAsync(U + (size_t)LeP * NCP, 0, (size_t)LoP * NCP * sizeof(double), s));
    // GEMM 2
    k_bq_gemm<<<dim3((unsigned)(NCP / GT_I), JP / GT_J), GT_NT, GT_SMEM, s>>>(LP, G[pi], LP, U, NCP, Q, NCP);
    k_bq_scatter<<<dim3((unsigned)((b.nc + 255) / 256), qnb), 256, 0, s>>>(L, pref, b.par, qb0, c->delta, bc, b.nc, NCP,
                                                                         Q, dmb, dq);
    c->launches += 5;
    BQ_CUDA(cudaGetLastError());
  }
  BQ_CUDA(cudaStreamSynchronize(s));
#undef BQ_CUDA
  cleanup();
  return SCV_OK;
}

// The direct build: one CTA per (m, 8 consecutive l), k_betaq_build.
static int betaq_fill_direct(scv_ctx* c, int L, cudaStream_t s, double* dq, const long long* dmb, const double* dtrig) {
  const int K = 2 * L - 1;
  // degrees per task: as many as fit next to the trig tables in shared memory
  // (8 up to L = 1024, fewer at L = 2048)
  const size_t fixed = (size_t)4 * K + 2 * L + 2 + L + 32;
  const int QG = (int)std::max<long long>(1, std::min<long long>(QG_MAX, ((long long)(232448 / sizeof(double)) - (long long)fixed) / L));
  std::vector<int2> tasks;
  for (int m = -(L - 1); m <= L - 1; ++m)
    for (int l0 = std::abs(m); l0 < L; l0 += QG) tasks.push_back(make_int2(m, l0));
  void* dtask = nullptr;
  SCV_CUDA(c, cudaMalloc(&dtask, tasks.size() * sizeof(int2)));
  SCV_CUDA(c, cudaMemcpyAsync(dtask, tasks.data(), tasks.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
  const size_t sm = (fixed + (size_t)QG * L) * sizeof(double);
  SCV_CUDA(c, cudaFuncSetAttribute(k_betaq_build, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per = 0, sms = 0;
  SCV_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_betaq_build, QNT, sm));
  SCV_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  const int grid = std::max(1, std::min((int)tasks.size(), std::max(per, 1) * sms));
  const double pref = 4.0 * SCV_PI * SCV_PI / ((double)K * (double)K);
  k_betaq_build<<<grid, QNT, sm, s>>>(L, QG, pref, c->delta, dtrig, dmb, (const int2*)dtask, (int)tasks.size(), dq);
  c->launches++;
  const cudaError_t e = cudaGetLastError();
  const cudaError_t e2 = cudaStreamSynchronize(s);
  cudaFree(dtask);
  SCV_CUDA(c, e);
  SCV_CUDA(c, e2);
  return SCV_OK;
}

// 1 (default): tensor-core GEMM build; 0: k_betaq_build (env SCV_BETAQ_BUILD, read once)
static int betaq_method() {
  static const char* e = getenv("SCV_BETAQ_BUILD");
  return (e && e[0] == '0') ? 0 : 1;
}

// Allocate and fill the table of band limit L (method: 1 GEMM, 0 direct).
static int betaq_build(scv_ctx* c, int L, int method, int qb0, int qnb, cudaStream_t s, double** qout,
                       long long** mbout, long long* nq) {
  SCV_TRY(scv_ensure_delta(c, L, s));
  const int K = 2 * L - 1;
  if (qb0 != 0 || qnb != L) method = 1;  // the direct build writes whole blocks only
  std::vector<long long> mb(2 * L - 1);
  long long acc = 0;
  for (int m = -(L - 1); m <= L - 1; ++m) {
    mb[m + L - 1] = acc;
    acc += (long long)qnb * (L - std::abs(m));
  }
  const ld pi = 3.141592653589793238462643383279502884L;
  std::vector<double> trig(4 * (size_t)K);
  for (int j = 0; j < 2 * K; ++j) {
    trig[2 * j] = (double)cosl(pi * (ld)j / (ld)K);
    trig[2 * j + 1] = (double)sinl(pi * (ld)j / (ld)K);
  }
  double* dq = nullptr;
  long long* dmb = nullptr;
  void* dtrig = nullptr;
  SCV_CUDA(c, cudaMalloc(&dq, (size_t)acc * sizeof(double)));
  SCV_CUDA(c, cudaMalloc(&dmb, mb.size() * sizeof(long long)));
  SCV_CUDA(c, cudaMalloc(&dtrig, trig.size() * sizeof(double)));
  SCV_CUDA(c, cudaMemcpyAsync(dmb, mb.data(), mb.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  SCV_CUDA(c, cudaMemcpyAsync(dtrig, trig.data(), trig.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  int rc;
  {
    SCV_PROF(c, s, "betaq_build");
    rc = method ? betaq_fill_gemm(c, L, qb0, qnb, s, dq, dmb, (const double*)dtrig)
                : betaq_fill_direct(c, L, s, dq, dmb, (const double*)dtrig);
  }
  cudaStreamSynchronize(s);
  cudaFree(dtrig);
  if (rc != SCV_OK) {
    cudaFree(dq);
    cudaFree(dmb);
    return rc;
  }
  *qout = dq;
  *mbout = dmb;
  *nq = acc;
  return SCV_OK;
}

// Debug: build the table with `method` (1 GEMM, 0 direct) and copy its first `n` doubles to the
// device buffer `out` (tools/betaq_check.py compares the two builds); nothing is cached.
extern "C" int scv_debug_betaq_build(scv_ctx* c, int L, int method, double* out, long long n, void* stream) {
  if (!c || L < 2 || !out) return SCV_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  double* dq = nullptr;
  long long* dmb = nullptr;
  long long nq = 0;
  SCV_TRY(betaq_build(c, L, method, 0, L, s, &dq, &dmb, &nq));
  const cudaError_t e = cudaMemcpyAsync(out, dq, (size_t)std::min(n, nq) * sizeof(double), cudaMemcpyDeviceToDevice, s);
  cudaStreamSynchronize(s);
  cudaFree(dq);
  cudaFree(dmb);
  SCV_CUDA(c, e);
  return SCV_OK;
}

// The table of band limit L, built once per context: all L beta rows, or the rows the context
// was restricted to (scv_betaq_restrict).
int scv_betaq_table(scv_ctx* c, int L, cudaStream_t s, const double** qtab, const long long** mbase, int* qb0,
                    int* qrows) {
  const std::string key = "betaq_" + std::to_string(L);
  const std::string kb = "betaqb_" + std::to_string(L);
  auto rg = c->betaq_rows.find(L);
  *qb0 = rg == c->betaq_rows.end() ? 0 : rg->second.first;
  *qrows = rg == c->betaq_rows.end() ? L : rg->second.second;
  auto it = c->aux.find(key);
  if (it != c->aux.end()) {
    *qtab = (const double*)it->second;
    *mbase = (const long long*)c->aux[kb];
    return SCV_OK;
  }
  double* dq = nullptr;
  long long* dmb = nullptr;
  long long acc = 0;
  SCV_TRY(betaq_build(c, L, betaq_method(), *qb0, *qrows, s, &dq, &dmb, &acc));
  c->aux[key] = dq;
  c->aux[kb] = dmb;
  c->table_bytes += (long long)acc * (long long)sizeof(double) + (long long)(2 * L - 1) * (long long)sizeof(long long);
  *qtab = dq;
  *mbase = dmb;
  return SCV_OK;
}

extern "C" int scv_betaq_restrict(scv_ctx* c, int L, int b0, int nb) {
  if (!c) return SCV_EINVAL;
  if (L < 2 || b0 < 0 || nb < 0 || b0 + nb > L)
    return scv_fail(c, SCV_EINVAL, "beta rows [" + std::to_string(b0) + ", " + std::to_string(b0 + nb) +
                                       ") outside [0, " + std::to_string(L) + ")");
  auto rg = c->betaq_rows.find(L);
  const int ob0 = rg == c->betaq_rows.end() ? 0 : rg->second.first;
  const int onb = rg == c->betaq_rows.end() ? L : rg->second.second;
  const int nb0 = nb == 0 ? 0 : b0, nnb = nb == 0 ? L : nb;
  if (nb0 == ob0 && nnb == onb) return SCV_OK;
  // a table built for the old range is dropped (rebuilt on next use)
  const std::string key = "betaq_" + std::to_string(L), kb = "betaqb_" + std::to_string(L);
  auto it = c->aux.find(key);
  if (it != c->aux.end()) {
    SCV_TRY(scv_check_unpinned(c, "dropping a beta-quadrature table"));
    SCV_CUDA(c, cudaSetDevice(c->device));
    SCV_CUDA(c, cudaDeviceSynchronize());
    long long cols = 0;
    for (int m = -(L - 1); m <= L - 1; ++m) cols += L - std::abs(m);
    c->table_bytes -= cols * onb * (long long)sizeof(double) + (long long)(2 * L - 1) * (long long)sizeof(long long);
    cudaFree(it->second);
    c->aux.erase(it);
    auto ib = c->aux.find(kb);
    if (ib != c->aux.end()) {
      cudaFree(ib->second);
      c->aux.erase(ib);
    }
  }
  if (nb == 0) c->betaq_rows.erase(L);
  else c->betaq_rows[L] = std::make_pair(b0, nb);
  return SCV_OK;
}
