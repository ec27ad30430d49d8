// Curvelet-sparse Wigner transforms on SO(3) (so3.py:185-285, 349-417).
//
// Inverse (analysis direction).  The reference builds, per gamma frequency
// n, the (2l+1)^2 bin plane fac D_{m'm} D_{m'n} i^{n-m} W_{mn} e^{im'pi/K}
// and runs a 2-D IFFT over (beta-ext, alpha), keeping rows b<L
// (so3.py:247-285).  Summed over m' that beta transform is exactly
// i^{m-n} d^l_{mn}(beta_b) (the Fourier expansion the reference itself uses
// in wigner_d_matrix, wigner.py:287-301), and for the sparse columns
// n=+-l d^l_{mn} has the closed form of wigner_d_edge_columns
// (wigner.py:304-322):
//     d^l_{m,+l}(b) = sqrt(C(2l,l+m)) sin(b/2)^{l-m} cos(b/2)^{l+m}
//     d^l_{m,-l}(b) = (-1)^{l-m} sqrt(C(2l,l+m)) sin(b/2)^{l+m} cos(b/2)^{l-m}
// so the signal is generated directly as fac W_{mn} d^l_{mn}(beta_b) in
// (n, b, alpha-bin) order (k_so3inv_gen: one coalesced pass over the output
// volume, O(L^3) work, no beta FFT), followed by the alpha and gamma
// inverse FFTs in place (cuFFT, the stages the north star allows it for).
//
// Forward (synthesis direction).  Per beta-slab chunk: 2-D forward FFT over
// (gamma, alpha) (cuFFT) into a chunk buffer, then k_so3_extract keeps only
// the |m| <= |n| entries the beta stage consumes (so3.py:240) and transposes
// them to beta-contiguous columns W1p[(n,m)][b].  The beta stage and Delta
// contraction are the hand-written k_beta_so3 (beta.cu).

#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "scv_internal.cuh"

__global__ void __launch_bounds__(128) k_so3inv_gen(int L, int real, const double2* __restrict__ w,
                                                    const double* __restrict__ hlb,
                                                    const double* __restrict__ lsin,
                                                    const double* __restrict__ lcos,
                                                    double2* __restrict__ out) {
  const int K = 2 * L - 1;
  const int gi = blockIdx.x / L;  // gamma-frequency slot
  const int b = blockIdx.x - gi * L;
  const int n = real ? gi : (gi <= L - 1 ? gi : gi - K);
  const int l = n < 0 ? -n : n;
  const double2* wrow = w + ((long long)(n >= 0 ? 0 : 1) * L + l) * K + (L - 1);
  const double fac = (double)(2 * l + 1) / (8.0 * SCV_PI * SCV_PI);
  const double ls = lsin[b], lc = lcos[b];
  const double* hrow = hlb + (long long)l * (l + 1) / 2;
  double2* orow = out + ((long long)gi * L + b) * K;
  for (int idx = threadIdx.x; idx < K; idx += blockDim.x) {
    const int m = idx <= L - 1 ? idx : idx - K;
    double2 v = make_double2(0.0, 0.0);
    if (m >= -l && m <= l) {
      const int am = m < 0 ? -m : m;
      const int es = n >= 0 ? l - m : l + m;  // power of sin(b/2)
      const int ec = n >= 0 ? l + m : l - m;  // power of cos(b/2)
      double lg = hrow[am];
      if (es) lg += (double)es * ls;
      if (ec) lg += (double)ec * lc;
      double d = exp(lg);
      if (n < 0 && ((l - m) & 1)) d = -d;
      const double2 c = wrow[m];
      const double f = fac * d;
      v = make_double2(f * c.x, f * c.y);
    }
    orow[idx] = v;
  }
}

// chunk (complex): [bb][gi][ai] K x K per beta;  (real): [bb][gi][ai'] K x L
__global__ void k_so3_extract(int L, int real, int b0, int nbb, const double2* __restrict__ chunk,
                              double2* __restrict__ W1p) {
  const int K = 2 * L - 1;
  const int bb = threadIdx.x;
  const int n = real ? (int)blockIdx.y : (int)blockIdx.y - (L - 1);
  const int l = n < 0 ? -n : n;
  const int m = -l + (int)(blockIdx.x * blockDim.y + threadIdx.y);
  if (bb >= nbb || m > l) return;
  long long cb;
  if (real) cb = (long long)l * l;
  else if (l == 0) cb = 0;
  else cb = n > 0 ? 2LL * l * l - 1 : 2LL * l * l + 2 * l;
  double2 v;
  if (!real) {
    const int gi = ((n % K) + K) % K, ai = ((m % K) + K) % K;
    v = chunk[((long long)bb * K + gi) * K + ai];
  } else if (m >= 0) {
    v = chunk[((long long)bb * K + n) * L + m];
  } else {
    const int gi = (K - n) % K;
    double2 t = chunk[((long long)bb * K + gi) * L + (-m)];
    v = make_double2(t.x, -t.y);
  }
  W1p[(cb + m + l) * (long long)L + b0 + bb] = v;
}

__global__ void k_zero_imag(double2* x, long long count) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) x[t].y = 0.0;
}

// Run a batched 1-D transform over `total` batches in bounded chunks.
// Batch q of a chunk starting at q0 reads in + (q0+q)*idist and writes out + (q0+q)*odist.
static int fft1d_chunked(scv_ctx* c, const std::string& tag, int len, int inembed, int istride,
                         int idist, int onembed, int ostride, int odist, cufftType type,
                         long long total, void* in, void* out, int dir, cudaStream_t s,
                         size_t in_elem, size_t out_elem) {
  int n[1] = {len}, ie[1] = {inembed}, oe[1] = {onembed};
  auto key_of = [&](long long nb) {
    return tag + "_" + std::to_string(len) + "_" + std::to_string(istride) + "_" + std::to_string(idist) +
           "_" + std::to_string(ostride) + "_" + std::to_string(odist) + "_" + std::to_string(nb);
  };
  // create every plan first (shrinking the chunk if a plan or its work area
  // does not fit), then execute: a failure never leaves a half-transformed buffer
  long long B = std::min<long long>(total, 1LL << 16);
  cufftHandle hB = 0, hR = 0;
  for (;;) {
    int rc = scv_plan(c, key_of(B), 1, n, ie, istride, idist, oe, ostride, odist, type, (int)B, &hB);
    const long long rem = total % B;
    if (rc == SCV_OK && rem)
      rc = scv_plan(c, key_of(rem), 1, n, ie, istride, idist, oe, ostride, odist, type, (int)rem, &hR);
    if (rc == SCV_OK) break;
    if (B <= 256) return rc;
    B /= 4;
  }
  for (long long q0 = 0; q0 < total; q0 += B) {
    const long long nb = std::min(B, total - q0);
    cufftHandle h = (nb == B) ? hB : hR;
    SCV_TRY(scv_plan_exec_setup(c, h, s));
    char* ip = (char*)in + (size_t)q0 * idist * in_elem;
    char* op = (char*)out + (size_t)q0 * odist * out_elem;
    if (type == CUFFT_Z2Z)
      SCV_CUFFT(c, cufftExecZ2Z(h, (cufftDoubleComplex*)ip, (cufftDoubleComplex*)op, dir));
    else if (type == CUFFT_Z2D)
      SCV_CUFFT(c, cufftExecZ2D(h, (cufftDoubleComplex*)ip, (double*)op));
    else
      SCV_CUFFT(c, cufftExecD2Z(h, (double*)ip, (cufftDoubleComplex*)op));
  }
  return SCV_OK;
}

static int check_so3(scv_ctx* c, int L) {
  if (L < 1) return scv_fail(c, SCV_EINVAL, "band limit must be positive, got " + std::to_string(L));
  if (L > 2048) return scv_fail(c, SCV_EINVAL, "band limit above 2048 not supported");
  return SCV_OK;
}


// Synthesis over the beta rows [sb0, sb0 + snb) of the scale signal, held as
// a (K, snb, K) beta slab at `sig` (the full signal is the slab (0, L)):
// alpha DFT rows -> beta chunk; gamma DFT fused with the beta quadrature,
// accumulated into w (the partial sum over this slab's beta rows).
static bool use_betaq(scv_ctx* c, int L) {
  return scv_pfa_supported(2 * L - 1) && L >= 128 && L <= 2048 && c->opt_betaq != 0 &&
         (c->opt_betaq == 1 || scv_betaq_enabled(L));
}

// bytes of one beta row of the chunk between the alpha and gamma passes; covers the transposed
// layout K x (nbb K rounded up to even) too (pfa.cu, SCV_SYN_PAIR)
static size_t syn_chunk_row_bytes(int L) {
  const size_t K = 2 * (size_t)L - 1;
  return (K + 1) * K * 16;
}
// Beta rows per launch pair of the synthesis.  4.3 GB: 64 rows at L_j = 1024, the size of the
// blocked analysis' scratch in the same slot (launches of 16 rows measured 6 ms/map slower:
// ring fill/drain per launch).  The quadrature sum over a slab is formed chunk by chunk, so
// callers that want the whole-scale summation order cut their slabs at multiples of this.
extern "C" int scv_syn_chunk_rows(int L) {
  if (L < 1) return 0;
  static const long long chunk_bytes = getenv("SCV_SYN_CHUNK") ? atoll(getenv("SCV_SYN_CHUNK")) : 4300000000LL;
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)L, (size_t)chunk_bytes / syn_chunk_row_bytes(L)));
}

static int forward_q_slab(scv_ctx* c, int L, int real, const void* sig, int sb0, int snb, double* w, cudaStream_t s) {
  const int K = 2 * L - 1;
  const double* qtab = nullptr;
  const long long* mbase = nullptr;
  int qb0 = 0, qrows = L;
  SCV_TRY(scv_betaq_table(c, L, s, &qtab, &mbase, &qb0, &qrows));
  if (sb0 < qb0 || sb0 + snb > qb0 + qrows)
    return scv_fail(c, SCV_EINVAL, "beta rows [" + std::to_string(sb0) + ", " + std::to_string(sb0 + snb) +
                                       ") are outside the rows [" + std::to_string(qb0) + ", " +
                                       std::to_string(qb0 + qrows) + ") this context's quadrature table of L=" +
                                       std::to_string(L) + " is restricted to (scv_betaq_restrict)");
  const size_t per_bc = syn_chunk_row_bytes(L);
  const int nbc = std::min(snb, scv_syn_chunk_rows(L));
  void* ch = nullptr;
  SCV_TRY(scv_scratch(c, 1, per_bc * nbc, &ch));
  for (int b0 = sb0; b0 < sb0 + snb; b0 += nbc) {
    const int nbb = std::min(nbc, sb0 + snb - b0);
    {
      SCV_PROF(c, s, "so3fwd_alpha");
      // real: the alpha pass keeps only the m >= 0 half (real = 2) the gamma+quadrature pass reads
      SCV_TRY(scv_pfa_syn_alpha(c, K, real ? 2 : 0, c->opt_chunkt | 4, sig, snb, b0 - sb0, nbb, (double2*)ch, s));
    }
    SCV_PROF(c, s, "so3fwd_gamma_q");
    SCV_TRY(scv_pfa_syn_gamma_q(c, K, real, c->opt_chunkt, (const double2*)ch, b0 - qb0, nbb, qtab, mbase, qrows, (double2*)w, s));
  }
  if (real) {
    SCV_PROF(c, s, "so3fwd_mirror");
    SCV_TRY(scv_wout_mirror(c, L, (double2*)w, s));
  }
  return SCV_OK;
}

static int check_slab(scv_ctx* c, int L, int b0, int nb) {
  if (b0 < 0 || nb < 1 || b0 + nb > L)
    return scv_fail(c, SCV_EINVAL, "beta slab [" + std::to_string(b0) + ", " + std::to_string(b0 + nb) +
                                       ") outside [0, " + std::to_string(L) + ")");
  return SCV_OK;
}

extern "C" int scv_so3_inverse_curvelet_slab(scv_ctx* c, int L, const double* w, int b0, int nb, void* sig,
                                             void* stream) {
  if (!c) return SCV_EINVAL;
  SCV_TRY(check_so3(c, L));
  SCV_TRY(check_slab(c, L, b0, nb));
  const int K = 2 * L - 1;
  if (!scv_pfa_supported(K))
    return scv_fail(c, SCV_EINVAL, "beta-slab analysis needs a prime-factor grid length, got K=" + std::to_string(K));
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_TRY(scv_ensure_hlb(c, L, s));
  const BetaTables* t = nullptr;
  SCV_TRY(scv_get_beta_tables(c, L, s, &t));
  {
    const int rc = scv_pfa_ana_blocked(c, K, (const double2*)w, c->hlb, t->sinh, t->cosh, b0, nb, (double2*)sig, s);
    if (rc <= 0) return rc;
  }
  {
    SCV_PROF(c, s, "so3inv_colgen");
    SCV_TRY(scv_pfa_ana_colgen(c, K, (const double2*)w, c->hlb, t->sinh, t->cosh, b0, nb, (double2*)sig, s));
  }
  SCV_PROF(c, s, "so3inv_rows");
  SCV_TRY(scv_pfa_rows_inplace(c, K, +1, (long long)K * nb, (double2*)sig, s));
  return SCV_OK;
}

extern "C" int scv_so3_forward_curvelet_slab(scv_ctx* c, int L, int real, const void* sig, int b0, int nb,
                                             double* w, int accumulate, void* stream) {
  if (!c) return SCV_EINVAL;
  SCV_TRY(check_so3(c, L));
  SCV_TRY(check_slab(c, L, b0, nb));
  if (!use_betaq(c, L))
    return scv_fail(c, SCV_EINVAL, "beta-slab synthesis needs the beta-quadrature path (prime-factor K, 128 <= L <= 2048)");
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_TRY(scv_ensure_delta(c, L, s));
  if (!accumulate) SCV_CUDA(c, cudaMemsetAsync(w, 0, (size_t)2 * L * (2 * L - 1) * 16, s));
  return forward_q_slab(c, L, real, sig, b0, nb, w, s);
}

extern "C" int scv_so3_inverse_curvelet(scv_ctx* c, int L, int real, const double* w, void* sig,
                                        void* stream) {
  if (!c) return SCV_EINVAL;
  SCV_TRY(check_so3(c, L));
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_TRY(scv_ensure_hlb(c, L, s));
  const BetaTables* t = nullptr;
  SCV_TRY(scv_get_beta_tables(c, L, s, &t));
  const int K = 2 * L - 1;
  const long long LK = (long long)L * K;
  if (scv_pfa_supported(K)) {
    // hand-written prime-factor path: fused generate + alpha IDFT, then gamma IDFT
    if (!real && c->opt_colgen) {
      {
        const int rc = scv_pfa_ana_blocked(c, K, (const double2*)w, c->hlb, t->sinh, t->cosh, 0, L, (double2*)sig, s);
        if (rc <= 0) return rc;
      }
      {
        SCV_PROF(c, s, "so3inv_colgen");
        SCV_TRY(scv_pfa_ana_colgen(c, K, (const double2*)w, c->hlb, t->sinh, t->cosh, 0, L, (double2*)sig, s));
      }
      SCV_PROF(c, s, "so3inv_rows");
      SCV_TRY(scv_pfa_rows_inplace(c, K, +1, (long long)K * L, (double2*)sig, s));
      return SCV_OK;
    }
    if (!real) {
      {
        SCV_PROF(c, s, "so3inv_alpha");
        SCV_TRY(scv_pfa_ana_alpha(c, K, 0, (const double2*)w, c->hlb, t->sinh, t->cosh, (double2*)sig, s));
      }
      SCV_PROF(c, s, "so3inv_gamma");
      SCV_TRY(scv_pfa_ana_gamma(c, K, 0, (double2*)sig, nullptr, s));
      return SCV_OK;
    }
    void* T = nullptr;
    SCV_TRY(scv_scratch(c, 0, (size_t)L * LK * 16, &T));
    if (c->opt_colgen) {  // gamma first: Hermitian-half columns, then two real rows per transform
      SCV_TRY(scv_pfa_ana_real_gf(c, K, (const double2*)w, c->hlb, t->sinh, t->cosh, 0, L, (double2*)T,
                                  (double*)sig, s));
      return SCV_OK;
    }
    {
      SCV_PROF(c, s, "so3inv_alpha");
      SCV_TRY(scv_pfa_ana_alpha(c, K, 1, (const double2*)w, c->hlb, t->sinh, t->cosh, (double2*)T, s));
    }
    SCV_PROF(c, s, "so3inv_gamma");
    SCV_TRY(scv_pfa_ana_gamma(c, K, 1, (double2*)T, (double*)sig, s));
    return SCV_OK;
  }
  if (!real) {
    {
    SCV_PROF(c, s, "so3inv_gen");
    k_so3inv_gen<<<K * L, 128, 0, s>>>(L, 0, (const double2*)w, c->hlb, t->sinh, t->cosh, (double2*)sig);
    c->launches++;
    SCV_CUDA(c, cudaGetLastError());
    }
    // alpha: contiguous rows, in place
    {
    SCV_PROF(c, s, "so3inv_alpha_fft");
    SCV_TRY(fft1d_chunked(c, "a_inv", K, K, 1, K, K, 1, K, CUFFT_Z2Z, (long long)K * L, sig, sig,
                          CUFFT_INVERSE, s, 16, 16));
    }
    // gamma: stride L*K, batches are the (b, a) pairs
    SCV_PROF(c, s, "so3inv_gamma_fft");
    SCV_TRY(fft1d_chunked(c, "g_inv", K, K, (int)LK, 1, K, (int)LK, 1, CUFFT_Z2Z, LK, sig, sig,
                          CUFFT_INVERSE, s, 16, 16));
    return SCV_OK;
  }
  void* T = nullptr;
  SCV_TRY(scv_scratch(c, 0, (size_t)L * LK * 16, &T));
  SCV_PROF(c, s, "so3inv_real");
  k_so3inv_gen<<<L * L, 128, 0, s>>>(L, 1, (const double2*)w, c->hlb, t->sinh, t->cosh, (double2*)T);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  SCV_TRY(fft1d_chunked(c, "a_inv", K, K, 1, K, K, 1, K, CUFFT_Z2Z, (long long)L * L, T, T,
                        CUFFT_INVERSE, s, 16, 16));
  // irfft along gamma ignores Im of the n=0 bin (scipy semantics, so3.py:416)
  k_zero_imag<<<(int)((LK + 255) / 256), 256, 0, s>>>((double2*)T, LK);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  SCV_TRY(fft1d_chunked(c, "g_c2r", K, L, (int)LK, 1, K, (int)LK, 1, CUFFT_Z2D, LK, T, sig, 0, s, 16, 8));
  return SCV_OK;
}

extern "C" int scv_so3_forward_curvelet(scv_ctx* c, int L, int real, const void* sig, double* w,
                                        void* stream) {
  if (!c) return SCV_EINVAL;
  SCV_TRY(check_so3(c, L));
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_TRY(scv_ensure_delta(c, L, s));
  const int K = 2 * L - 1;
  SCV_CUDA(c, cudaMemsetAsync(w, 0, (size_t)2 * L * K * 16, s));
  const bool use_q = use_betaq(c, L);
  if (use_q) return forward_q_slab(c, L, real, sig, 0, L, w, s);
  const long long cols = real ? (long long)L * L : 2LL * L * L - 1;
  void* W1p = nullptr;
  SCV_TRY(scv_scratch(c, 0, (size_t)(cols * L) * 16, &W1p));
  const size_t per_b = (size_t)K * (real ? L : K) * 16;
  int nb = (int)std::max<size_t>(1, std::min<size_t>((size_t)L, (size_t)(1u << 30) / per_b));
  void* chunk = nullptr;
  SCV_TRY(scv_scratch(c, 1, per_b * nb, &chunk));
  if (scv_pfa_supported(K)) {
    // hand-written prime-factor path: alpha DFT rows -> chunk, gamma DFT + pruning -> W1p
    const size_t per_bc = (size_t)K * K * 16;
    // chunk of beta slabs between the alpha and gamma passes (1 GB; an
    // L2-resident single-slab chunk measured slower: launch + tail overheads)
    static const long long chunk_bytes = getenv("SCV_SYN_CHUNK") ? atoll(getenv("SCV_SYN_CHUNK")) : (1LL << 30);
    int nbc = (int)std::max<size_t>(1, std::min<size_t>((size_t)L, (size_t)chunk_bytes / per_bc));
    void* ch = nullptr;
    SCV_TRY(scv_scratch(c, 1, per_bc * nbc, &ch));
    for (int b0 = 0; b0 < L; b0 += nbc) {
      const int nbb = std::min(nbc, L - b0);
      {
        SCV_PROF(c, s, "so3fwd_alpha");
        SCV_TRY(scv_pfa_syn_alpha(c, K, real, 0, sig, L, b0, nbb, (double2*)ch, s));
      }
      SCV_PROF(c, s, "so3fwd_gamma");
      SCV_TRY(scv_pfa_syn_gamma(c, K, real, (const double2*)ch, b0, nbb, (double2*)W1p, s));
    }
  } else
  for (int b0 = 0; b0 < L; b0 += nb) {
    const int nbb = std::min(nb, L - b0);
    int n2[2] = {K, K};
    int ie[2] = {K, L * K};
    cufftHandle h;
    {
    SCV_PROF(c, s, "so3fwd_fft2d");
    if (!real) {
      int oe[2] = {K, K};
      SCV_TRY(scv_plan(c, "fwd2d_z2z_" + std::to_string(L) + "_" + std::to_string(nbb), 2, n2, ie, 1, K,
                       oe, 1, K * K, CUFFT_Z2Z, nbb, &h));
      SCV_TRY(scv_plan_exec_setup(c, h, s));
      SCV_CUFFT(c, cufftExecZ2Z(h, (cufftDoubleComplex*)((const double2*)sig + (size_t)b0 * K),
                                (cufftDoubleComplex*)chunk, CUFFT_FORWARD));
    } else {
      int oe[2] = {K, L};
      SCV_TRY(scv_plan(c, "fwd2d_d2z_" + std::to_string(L) + "_" + std::to_string(nbb), 2, n2, ie, 1, K,
                       oe, 1, K * L, CUFFT_D2Z, nbb, &h));
      SCV_TRY(scv_plan_exec_setup(c, h, s));
      SCV_CUFFT(c, cufftExecD2Z(h, (double*)((const double*)sig + (size_t)b0 * K), (cufftDoubleComplex*)chunk));
    }
    }
    SCV_PROF(c, s, "so3fwd_extract");
    dim3 blk(32, 8);
    for (int bs = 0; bs < nbb; bs += 32) {
      const int nsub = std::min(32, nbb - bs);
      const double2* csub = (const double2*)chunk + (size_t)bs * (per_b / 16);
      dim3 grd((K + 7) / 8, real ? L : K);
      k_so3_extract<<<grd, blk, 0, s>>>(L, real, b0 + bs, nsub, csub, (double2*)W1p);
      c->launches++;
      SCV_CUDA(c, cudaGetLastError());
    }
  }
  const double pref = 4.0 * SCV_PI * SCV_PI / ((double)K * (double)K);
  SCV_PROF(c, s, "beta_so3");
  SCV_TRY(scv_beta_so3(c, L, real, (const double2*)W1p, (double2*)w, pref, s));
  return SCV_OK;
}
