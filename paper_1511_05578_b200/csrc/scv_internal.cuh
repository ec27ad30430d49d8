// Internal declarations shared by the scurve_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/scurve_b200.h"

#ifndef SCV_PI
#define SCV_PI 3.14159265358979323846
#endif

// ---------------------------------------------------------------------------
// complex128 helpers
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) {
  return make_double2(a.x * s, a.y * s);
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// a * i^k  (exact: swaps and sign flips only)
__host__ __device__ __forceinline__ double2 cipow(double2 a, int k) {
  switch (((k % 4) + 4) % 4) {
    case 0: return a;
    case 1: return make_double2(-a.y, a.x);
    case 2: return make_double2(-a.x, -a.y);
    default: return make_double2(a.y, -a.x);
  }
}

// ---------------------------------------------------------------------------
// Delta(pi/2) wedge indexing: element (l, a, b), 0 <= b <= a <= l
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ long long wedge_plane_base(int l) {
  return (long long)l * (l + 1) * (l + 2) / 6;
}
__host__ __device__ __forceinline__ long long wedge_size(int L) { return wedge_plane_base(L); }

// Delta^l_{mp,m} from the wedge using the three symmetries
//   D_{-m',m} = (-1)^{l+m} D_{m'm},  D_{m',-m} = (-1)^{l+m'} D_{m'm},
//   D_{m'm}  = (-1)^{m'-m} D_{mm'}.
__device__ __forceinline__ double wedge_get(const double* __restrict__ W, int l, int mp, int m) {
  int neg = 0;
  if (mp < 0) { mp = -mp; neg ^= (l + m) & 1; }
  if (m < 0) { m = -m; neg ^= (l + mp) & 1; }
  if (mp < m) { int t = mp; mp = m; m = t; neg ^= (mp - m) & 1; }
  double v = __ldg(W + wedge_plane_base(l) + (long long)mp * (mp + 1) / 2 + m);
  return neg ? -v : v;
}

// ---------------------------------------------------------------------------
// Per-band-limit constant tables (built once per L, cached in the context)
// ---------------------------------------------------------------------------
struct BetaTables {
  int L = 0, K = 0, P = 0, logP = 0;
  double2* tw = nullptr;     // P   : exp(-2 pi i k / P)
  double2* chirpA = nullptr; // K   : exp(-i pi b^2 / K)                 (Bluestein pre-chirp)
  double2* Hf = nullptr;     // P   : FFT_P(h)/P, h[j] = exp(+i pi j^2/K)  (Bluestein filter)
  double2* chirpC = nullptr; // K   : (1/K) exp(-i pi (m''^2 + m'')/K)      (post-chirp * offset phase)
  double2* Vf = nullptr;     // P   : FFT_P(v)/P, v[q] = w_even(2(L-1) - q)
  double* Aalt = nullptr;    // K   : sum_{m''} w_even(m''-m') (-1)^{m''}
  double* sinh = nullptr;    // L   : log sin(beta_b / 2)
  double* cosh = nullptr;    // L   : log cos(beta_b / 2)
  // prime-factor beta stage (K and K2 = 4L-1 both prime-factor lengths)
  // centred Bluestein (register-FFT beta stage, beta2.cu)
  double2* a2 = nullptr;     // L     : exp(-i pi b'^2/K), b' = 0..L-1 (even in b')
  double2* hf2 = nullptr;    // P/2+1 : FFT_P(h')/P, h'[j] = exp(+i pi j^2/K), |j| <= 2L-2 (even)
  double* vf2 = nullptr;     // P/2+1 : FFT_P(w_even wrapped)/P (real, even)
};

struct FftPlan {
  cufftHandle h = 0;
  size_t work = 0;
};

struct scv_ctx {
  int device = 0;
  std::string err;
  // Delta(pi/2) wedge (grow-only, like halfpi_table, wigner.py:226-240)
  int delta_L = 0;
  double* delta = nullptr;
  // half log binomials: hlb[l(l+1)/2 + k] = 0.5*ln C(2l, l+k), k = 0..l
  int hlb_L = 0;
  double* hlb = nullptr;
  std::map<int, BetaTables> beta;   // by band limit
  std::map<std::string, FftPlan> plans;
  // cuFFT work area shared by all plans (grow-only)
  void* fft_work = nullptr;
  size_t fft_work_bytes = 0;
  // general scratch (grow-only), two independent slots
  void* scratch[3] = {nullptr, nullptr, nullptr};
  size_t scratch_bytes[3] = {0, 0, 0};
  // small int tables by key
  std::map<std::string, void*> aux;
  // beta rows [first, first + second) the quadrature table of band limit L covers
  // (scv_betaq_restrict; absent = all L rows)
  std::map<int, std::pair<int, int>> betaq_rows;
  long long table_bytes = 0;  // persistent per-L tables in `aux` (quadrature, prime-factor, tasks)
  long long small_table_bytes = 0;  // the part of table_bytes that scv_trim keeps (prime-factor, task tables)
  // stage profiler (scv_profile): event pairs around every launch group
  bool prof = false;
  long long launches = 0;  // kernels of this library launched (scv_launch_count)
  struct Rec { std::string name; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  // options (scv_set_option): -1 = library default
  int opt_chunkt = 0;  // synthesis chunk layout: 1 = [b][m][g] (strided alpha writes), 0 = [b][g][m]
  int opt_colgen = 1;  // analysis order: 1 = gamma-first column generation + in-place alpha rows, 0 = alpha-first
  int opt_betaq = -1;  // synthesis beta stage: 1 = quadrature table, 0 = per-column FFTs
  // > 0 while CUDA graphs captured on this context are alive (scv_set_option
  // "pin"): the graphs hold raw pointers into the workspace, so every path
  // that would free or move a workspace buffer fails instead
  int pinned = 0;
};

// SCV_EINVAL if the context is pinned (a live graph references its buffers)
int scv_check_unpinned(scv_ctx* c, const char* what);

// RAII stage timer: records a start/stop event pair on `s` when profiling is on
struct ProfScope {
  scv_ctx* c;
  cudaStream_t s;
  int idx = -1;
  ProfScope(scv_ctx* c_, cudaStream_t s_, const char* name);
  ~ProfScope();
};
#define SCV_PROF_CAT2(a, b) a##b
#define SCV_PROF_CAT(a, b) SCV_PROF_CAT2(a, b)
#define SCV_PROF(c, s, name) ProfScope SCV_PROF_CAT(prof_scope_, __LINE__)(c, s, name)

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
int scv_fail(scv_ctx* c, int code, const std::string& msg);

#define SCV_CUDA(ctx, expr)                                                              \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return scv_fail(ctx, SCV_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define SCV_CUFFT(ctx, expr)                                                             \
  do {                                                                                   \
    cufftResult r_ = (expr);                                                             \
    if (r_ != CUFFT_SUCCESS)                                                             \
      return scv_fail(ctx, SCV_ECUFFT, std::string(#expr) + ": cufft error " + std::to_string((int)r_)); \
  } while (0)

#define SCV_TRY(expr)           \
  do {                          \
    int rc_ = (expr);           \
    if (rc_ != SCV_OK) return rc_; \
  } while (0)

// context services (ctx.cu)
int scv_ensure_delta(scv_ctx* c, int L, cudaStream_t s);
int scv_ensure_hlb(scv_ctx* c, int L, cudaStream_t s);
int scv_get_beta_tables(scv_ctx* c, int L, cudaStream_t s, const BetaTables** out);
int scv_scratch(scv_ctx* c, int slot, size_t bytes, void** out);
// many-dimensional cuFFT plan with advanced layout; cached by a string key
int scv_plan(scv_ctx* c, const std::string& key, int rank, int* n, int* inembed, int istride,
             int idist, int* onembed, int ostride, int odist, cufftType type, int batch,
             cufftHandle* out);
int scv_plan_exec_setup(scv_ctx* c, cufftHandle h, cudaStream_t s);

// kernels launched from other units
int scv_launch_delta_wedge(scv_ctx* c, int L, const double* edge, const int* edge_e, double* out, cudaStream_t s);
int scv_beta_sht(scv_ctx* c, int L, int spin, int real, const double2* G, double2* Gw, double pref,
                 cudaStream_t s);
int scv_beta_so3(scv_ctx* c, int L, int real, const double2* W1p, double2* w, double pref,
                 cudaStream_t s);
bool scv_beta2_supported(int L);
int scv_beta2_so3(scv_ctx* c, int L, int real, const double2* W1p, double2* w, double pref,
                  const BetaTables* t, const int2* tasks, int ntasks, cudaStream_t s);

// prime-factor alpha/gamma kernels (pfa.cu), K = 2^k - 1
bool scv_pfa_supported(int K);
int scv_pfa_ana_alpha(scv_ctx* c, int K, int real, const double2* w, const double* hlb, const double* ls,
                      const double* lc, double2* out, cudaStream_t s);
int scv_pfa_ana_colgen(scv_ctx* c, int K, const double2* w, const double* hlb, const double* ls, const double* lc,
                       int b0, int nb, double2* out, cudaStream_t s);
int scv_pfa_ana_real_gf(scv_ctx* c, int K, const double2* w, const double* hlb, const double* ls, const double* lc,
                        int b0, int nb, double2* T, double* out, cudaStream_t s);
int scv_pfa_rows_inplace(scv_ctx* c, int K, int dir, long long nrows, double2* x, cudaStream_t s);
int scv_pfa_ana_blocked(scv_ctx* c, int K, const double2* w, const double* hlb, const double* ls, const double* lc,
                        int b0, int nb, double2* sig, cudaStream_t s);
int scv_pfa_ana_gamma(scv_ctx* c, int K, int real, double2* src, double* dst, cudaStream_t s);
int scv_pfa_syn_alpha(scv_ctx* c, int K, int real, int tr, const void* in, int lsig, int b0, int nbb, double2* chunk,
                      cudaStream_t s);
int scv_pfa_syn_gamma(scv_ctx* c, int K, int real, const double2* chunk, int b0, int nbb, double2* W1p,
                      cudaStream_t s);
int scv_pfa_pos_host(int K, int k);  // CRT output position of frequency k
// fused gamma pass + beta quadrature (synthesis), betaq.cu tables
int scv_pfa_syn_gamma_q(scv_ctx* c, int K, int real, int tr, const double2* chunk, int b0, int nbb, const double* qtab,
                        const long long* mbase, int qrows, double2* wout, cudaStream_t s);
int scv_wout_mirror(scv_ctx* c, int L, double2* wout, cudaStream_t s);
bool scv_betaq_enabled(int L);
// table of band limit L: rows [*qb0, *qb0 + *qrows) of every (m, l) block (all L rows unless restricted)
int scv_betaq_table(scv_ctx* c, int L, cudaStream_t s, const double** qtab, const long long** mbase, int* qb0,
                    int* qrows);

inline int next_pow2_log(int x) {
  int lg = 0;
  while ((1 << lg) < x) ++lg;
  return lg;
}
