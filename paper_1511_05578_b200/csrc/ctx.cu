// Context, constant tables, cuFFT plan cache and scratch management.
//
// The reference keeps three process-global caches: the Delta(pi/2) table
// (wigner.py:226-240), the weight-kernel FFT (fourier.py:68-81) and the
// tiling step table.  Here the device-side equivalents live in a per-device
// context: the Delta wedge (built on the GPU by the degree recursion), the
// Bluestein / weight-convolution spectra used by the beta stage, cuFFT plans
// for the alpha/gamma stages, and grow-only scratch.  Host-side constants
// are computed in long double so the device tables carry correctly rounded
// float64 values.

#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>

#include "scv_internal.cuh"

typedef long double ld;
typedef std::complex<ld> cld;

static const ld kPi = 3.141592653589793238462643383279502884L;

static cudaEvent_t pool_get(scv_ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

ProfScope::ProfScope(scv_ctx* c_, cudaStream_t s_, const char* name) : c(c_), s(s_) {
  if (!c->prof) return;
  scv_ctx::Rec r{name, pool_get(c), pool_get(c)};
  cudaEventRecord(r.a, s);
  c->recs.push_back(r);
  idx = (int)c->recs.size() - 1;
}

ProfScope::~ProfScope() {
  if (idx >= 0) cudaEventRecord(c->recs[idx].b, s);
}

int scv_fail(scv_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

// ---------------------------------------------------------------------------
// long-double host helpers
// ---------------------------------------------------------------------------
static std::vector<ld> log_factorials(int n) {
  std::vector<ld> lf(n + 1);
  lf[0] = 0.0L;
  for (int i = 1; i <= n; ++i) lf[i] = lf[i - 1] + logl((ld)i);
  return lf;
}

// exp(i*pi*num/den) with num reduced exactly mod 2*den
static cld expipi(long long num, long long den) {
  long long r = num % (2 * den);
  if (r < 0) r += 2 * den;
  ld a = kPi * (ld)r / (ld)den;
  return cld(cosl(a), sinl(a));
}

static void fft_ld(std::vector<cld>& a) {  // forward, in place, radix-2
  size_t n = a.size();
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    for (size_t i = 0; i < n; i += len)
      for (size_t k = 0; k < len / 2; ++k) {
        cld w = expipi(-2LL * (long long)k, (long long)len);
        cld u = a[i + k], v = a[i + k + len / 2] * w;
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
  }
}

static inline ld w_even(long long k) {  // even part of w(k)=int_0^pi sin e^{ik}
  if (k & 1) return 0.0L;
  return 2.0L / (1.0L - (ld)k * (ld)k);
}

template <typename T>
static int upload(scv_ctx* c, T** dst, const std::vector<T>& src, cudaStream_t s) {
  SCV_CUDA(c, cudaMalloc((void**)dst, src.size() * sizeof(T)));
  SCV_CUDA(c, cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  SCV_CUDA(c, cudaStreamSynchronize(s));
  return SCV_OK;
}

static std::vector<double2> to_d2(const std::vector<cld>& v) {
  std::vector<double2> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = make_double2((double)v[i].real(), (double)v[i].imag());
  return o;
}

// ---------------------------------------------------------------------------
// tables
// ---------------------------------------------------------------------------
int scv_check_unpinned(scv_ctx* c, const char* what) {
  if (c->pinned > 0)
    return scv_fail(c, SCV_EINVAL, std::string("context is pinned by a captured CUDA graph; refusing to ") + what +
                                       " (use a private context for graphs, or release the graph first)");
  return SCV_OK;
}

int scv_ensure_hlb(scv_ctx* c, int L, cudaStream_t s) {
  if (c->hlb && c->hlb_L >= L) return SCV_OK;
  if (c->hlb) SCV_TRY(scv_check_unpinned(c, "grow the log-binomial table"));
  int Lb = L;
  std::vector<ld> lf = log_factorials(2 * Lb + 2);
  std::vector<double> h((size_t)Lb * (Lb + 1) / 2);
  for (int l = 0; l < Lb; ++l)
    for (int k = 0; k <= l; ++k)
      h[(size_t)l * (l + 1) / 2 + k] = (double)(0.5L * (lf[2 * l] - lf[l + k] - lf[l - k]));
  if (c->hlb) cudaFree(c->hlb);
  c->hlb = nullptr;
  SCV_TRY(upload(c, &c->hlb, h, s));
  c->hlb_L = Lb;
  return SCV_OK;
}

int scv_ensure_delta(scv_ctx* c, int L, cudaStream_t s) {
  if (c->delta && c->delta_L >= L) return SCV_OK;
  if (c->delta) SCV_TRY(scv_check_unpinned(c, "grow the Delta table"));
  // edge rows Delta^l_{l,m} = (-1)^{l-m} sqrt(C(2l,l+m)) / 2^l  (wigner.py:153-161),
  // as a double mantissa in [0.5, 1) and a power-of-two exponent: above
  // l ~ 1022 the edge values near |m| = l fall below the double range (2^-l),
  // while the interior entries the recursion grows from them do not, so the
  // kernel carries an exponent shift until the values are representable.
  // Seeds inside the double range reproduce (double)v exactly.
  std::vector<ld> lf = log_factorials(2 * L + 2);
  std::vector<double> edge((size_t)L * (L + 1) / 2);
  std::vector<int> edge_e((size_t)L * (L + 1) / 2);
  for (int l = 0; l < L; ++l)
    for (int m = 0; m <= l; ++m) {
      const ld lg2 = (0.5L * (lf[2 * l] - lf[l + m] - lf[l - m])) / logl(2.0L) - (ld)l;  // log2 |v|
      int e = (int)floorl(lg2) + 1;
      ld mant = exp2l(lg2 - (ld)e);  // in [0.5, 1)
      if (mant >= 1.0L) { mant *= 0.5L; ++e; }
      if (mant < 0.5L) { mant *= 2.0L; --e; }
      if ((l - m) & 1) mant = -mant;
      edge[(size_t)l * (l + 1) / 2 + m] = (double)mant;
      edge_e[(size_t)l * (l + 1) / 2 + m] = e;
    }
  if (L > 1) {  // seed plane of build_halfpi_table (wigner.py:214-218) uses 1/sqrt(2.0)
    int e;
    edge[1] = std::frexp(-1.0 / std::sqrt(2.0), &e);
    edge_e[1] = e;
    edge[2] = std::frexp(0.5, &e);
    edge_e[2] = e;
  }
  double* d_edge = nullptr;
  SCV_TRY(upload(c, &d_edge, edge, s));
  int* d_edge_e = nullptr;
  {
    cudaError_t ee = cudaMalloc((void**)&d_edge_e, edge_e.size() * sizeof(int));
    if (ee != cudaSuccess) return scv_fail(c, SCV_ENOMEM, "cudaMalloc(delta edge)");
    SCV_CUDA(c, cudaMemcpyAsync(d_edge_e, edge_e.data(), edge_e.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  }
  double* tab = nullptr;
  cudaError_t e = cudaMalloc((void**)&tab, (size_t)wedge_size(L) * sizeof(double));
  if (e != cudaSuccess) {
    cudaFree(d_edge);
    cudaFree(d_edge_e);
    return scv_fail(c, SCV_ENOMEM, "cudaMalloc(delta wedge): " + std::string(cudaGetErrorString(e)));
  }
  int rc = scv_launch_delta_wedge(c, L, d_edge, d_edge_e, tab, s);
  cudaStreamSynchronize(s);
  cudaFree(d_edge);
  cudaFree(d_edge_e);
  if (rc != SCV_OK) {
    cudaFree(tab);
    return rc;
  }
  if (c->delta) cudaFree(c->delta);
  c->delta = tab;
  c->delta_L = L;
  return SCV_OK;
}

int scv_get_beta_tables(scv_ctx* c, int L, cudaStream_t s, const BetaTables** out) {
  auto it = c->beta.find(L);
  if (it != c->beta.end()) {
    *out = &it->second;
    return SCV_OK;
  }
  BetaTables t;
  t.L = L;
  t.K = 2 * L - 1;
  t.logP = next_pow2_log(4 * L - 3);
  if (t.logP < 4) t.logP = 4;
  t.P = 1 << t.logP;
  const int K = t.K, P = t.P;
  std::vector<cld> tw(P), A(K), h(P, cld(0, 0)), C(K), v(P, cld(0, 0));
  for (int k = 0; k < P; ++k) tw[k] = expipi(-2LL * k, P);
  for (int b = 0; b < K; ++b) A[b] = expipi(-(long long)b * b, K);
  // h[j] = exp(+i pi j^2 / K) for j in [-(3L-3), L-1], stored at j mod P
  for (int j = -(3 * L - 3); j <= L - 1; ++j) h[((j % P) + P) % P] = expipi((long long)j * j, K);
  for (int q = 0; q < K; ++q) {
    long long mpp = q - (L - 1);
    C[q] = expipi(-(mpp * mpp + mpp), K) / (ld)K;
  }
  for (int q = 0; q <= 4 * L - 4; ++q) v[q] = cld(w_even(2LL * (L - 1) - q), 0);
  fft_ld(h);
  fft_ld(v);
  for (int k = 0; k < P; ++k) {
    h[k] /= (ld)P;
    v[k] /= (ld)P;
  }
  std::vector<double> Aalt(K), lsin(L), lcos(L);
  for (int q = 0; q < K; ++q) {
    long long mp = q - (L - 1);
    ld acc = 0;
    for (long long mpp = -(L - 1); mpp <= L - 1; ++mpp) acc += w_even(mpp - mp) * ((mpp & 1) ? -1.0L : 1.0L);
    Aalt[q] = (double)acc;
  }
  for (int b = 0; b < L; ++b) {
    // beta_b/2 = pi(2b+1)/(2K); cos(beta_b/2) = sin(pi(K-2b-1)/(2K)) keeps the
    // beta=pi node (b=L-1) exactly at cos=0 -> log = -inf (d vanishes there)
    lsin[b] = (double)logl(sinl(kPi * (ld)(2 * b + 1) / (ld)(2 * K)));
    const int r = K - 2 * b - 1;
    lcos[b] = r == 0 ? -HUGE_VAL : (double)logl(sinl(kPi * (ld)r / (ld)(2 * K)));
  }
  {  // centred Bluestein tables (beta2.cu)
    std::vector<cld> a2(L), h2(P, cld(0, 0)), v2(P, cld(0, 0));
    for (int i = 0; i < L; ++i) a2[i] = expipi(-(long long)i * i, K);
    for (int j = -(2 * L - 2); j <= 2 * L - 2; ++j) {
      h2[((j % P) + P) % P] = expipi((long long)j * j, K);
      v2[((j % P) + P) % P] = cld(w_even(j), 0);
    }
    fft_ld(h2);
    fft_ld(v2);
    std::vector<cld> hh(P / 2 + 1);
    std::vector<double> vv(P / 2 + 1);
    for (int k = 0; k <= P / 2; ++k) {
      hh[k] = h2[k] / (ld)P;
      vv[k] = (double)(v2[k].real() / (ld)P);
    }
    SCV_TRY(upload(c, &t.a2, to_d2(a2), s));
    SCV_TRY(upload(c, &t.hf2, to_d2(hh), s));
    SCV_TRY(upload(c, &t.vf2, vv, s));
  }
  SCV_TRY(upload(c, &t.tw, to_d2(tw), s));
  SCV_TRY(upload(c, &t.chirpA, to_d2(A), s));
  SCV_TRY(upload(c, &t.Hf, to_d2(h), s));
  SCV_TRY(upload(c, &t.chirpC, to_d2(C), s));
  SCV_TRY(upload(c, &t.Vf, to_d2(v), s));
  SCV_TRY(upload(c, &t.Aalt, Aalt, s));
  SCV_TRY(upload(c, &t.sinh, lsin, s));
  SCV_TRY(upload(c, &t.cosh, lcos, s));
  auto res = c->beta.emplace(L, t);
  *out = &res.first->second;
  return SCV_OK;
}

int scv_scratch(scv_ctx* c, int slot, size_t bytes, void** out) {
  if (bytes == 0) bytes = 16;
  if (c->scratch_bytes[slot] < bytes) {
    if (c->scratch[slot]) SCV_TRY(scv_check_unpinned(c, "grow a scratch buffer"));
    if (c->scratch[slot]) {
      cudaDeviceSynchronize();
      cudaFree(c->scratch[slot]);
      c->scratch[slot] = nullptr;
      c->scratch_bytes[slot] = 0;
    }
    cudaError_t e = cudaMalloc(&c->scratch[slot], bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      char buf[128];
      snprintf(buf, sizeof buf, "cudaMalloc(scratch %d, %.3f GB): ", slot, bytes / 1e9);
      return scv_fail(c, SCV_ENOMEM, std::string(buf) + cudaGetErrorString(e));
    }
    c->scratch_bytes[slot] = bytes;
  }
  *out = c->scratch[slot];
  return SCV_OK;
}

// ---------------------------------------------------------------------------
// cuFFT plans (alpha / gamma / phi stages only; the beta stage is hand-written)
// ---------------------------------------------------------------------------
int scv_plan(scv_ctx* c, const std::string& key, int rank, int* n, int* inembed, int istride,
             int idist, int* onembed, int ostride, int odist, cufftType type, int batch,
             cufftHandle* out) {
  auto it = c->plans.find(key);
  if (it != c->plans.end()) {
    *out = it->second.h;
    return SCV_OK;
  }
  FftPlan p;
  SCV_CUFFT(c, cufftCreate(&p.h));
  SCV_CUFFT(c, cufftSetAutoAllocation(p.h, 0));
  size_t work = 0;
  cufftResult r = cufftMakePlanMany(p.h, rank, n, inembed, istride, idist, onembed, ostride, odist,
                                    type, batch, &work);
  if (r != CUFFT_SUCCESS) {
    cufftDestroy(p.h);
    return scv_fail(c, SCV_ECUFFT, "cufftMakePlanMany(" + key + ") failed: " + std::to_string((int)r));
  }
  p.work = work;
  if (work > c->fft_work_bytes && c->fft_work) {
    const int rc = scv_check_unpinned(c, "grow the cuFFT work area");
    if (rc != SCV_OK) {
      cufftDestroy(p.h);
      return rc;
    }
  }
  if (work > c->fft_work_bytes) {
    if (c->fft_work) {
      cudaDeviceSynchronize();
      cudaFree(c->fft_work);
    }
    c->fft_work = nullptr;
    c->fft_work_bytes = 0;
    cudaError_t e = cudaMalloc(&c->fft_work, work);
    if (e != cudaSuccess) {
      cufftDestroy(p.h);
      cudaGetLastError();
      return scv_fail(c, SCV_ENOMEM, "cudaMalloc(cufft work " + std::to_string(work) + ")");
    }
    c->fft_work_bytes = work;
  }
  c->plans[key] = p;
  *out = p.h;
  return SCV_OK;
}

int scv_plan_exec_setup(scv_ctx* c, cufftHandle h, cudaStream_t s) {
  SCV_CUFFT(c, cufftSetStream(h, s));
  SCV_CUFFT(c, cufftSetWorkArea(h, c->fft_work));
  return SCV_OK;
}

// ---------------------------------------------------------------------------
// C ABI: lifecycle
// ---------------------------------------------------------------------------
extern "C" {

int scv_version(void) { return 102; }

int scv_create(int device, scv_ctx** out) {
  if (!out) return SCV_EINVAL;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return SCV_ECUDA;
  }
  if (device < 0 || device >= n) return SCV_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return SCV_ECUDA;
  scv_ctx* c = new scv_ctx();
  c->device = device;
  *out = c;
  return SCV_OK;
}

int scv_destroy(scv_ctx* c) {
  if (!c) return SCV_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto& kv : c->plans) cufftDestroy(kv.second.h);
  for (auto& kv : c->beta) {
    BetaTables& t = kv.second;
    cudaFree(t.tw); cudaFree(t.chirpA); cudaFree(t.Hf); cudaFree(t.chirpC);
    cudaFree(t.Vf); cudaFree(t.Aalt); cudaFree(t.sinh); cudaFree(t.cosh);
    cudaFree(t.a2); cudaFree(t.hf2); cudaFree(t.vf2);
  }
  for (auto& kv : c->aux) cudaFree(kv.second);
  for (auto& r : c->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : c->pool) cudaEventDestroy(e);
  if (c->fft_work) cudaFree(c->fft_work);
  for (int i = 0; i < 3; ++i)
    if (c->scratch[i]) cudaFree(c->scratch[i]);
  if (c->delta) cudaFree(c->delta);
  if (c->hlb) cudaFree(c->hlb);
  delete c;
  return SCV_OK;
}

const char* scv_last_error(const scv_ctx* c) { return c ? c->err.c_str() : "null context"; }

long long scv_launch_count(const scv_ctx* c) { return c ? c->launches : 0; }

int scv_profile(scv_ctx* c, int enable) {
  if (!c) return SCV_EINVAL;
  c->prof = enable != 0;
  return SCV_OK;
}

int scv_profile_report(scv_ctx* c, char* buf, int len) {
  if (!c || !buf || len <= 0) return SCV_EINVAL;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_CUDA(c, cudaDeviceSynchronize());
  std::map<std::string, std::pair<int, double>> agg;
  for (auto& r : c->recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& e = agg[r.name];
    e.first += 1;
    e.second += ms;
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->recs.clear();
  std::string out;
  char line[256];
  for (auto& kv : agg) {
    snprintf(line, sizeof line, "%s %d %.6f\n", kv.first.c_str(), kv.second.first, kv.second.second);
    out += line;
  }
  if ((int)out.size() + 1 > len) return scv_fail(c, SCV_EINVAL, "profile report buffer too small");
  memcpy(buf, out.c_str(), out.size() + 1);
  return SCV_OK;
}

long long scv_workspace_bytes(const scv_ctx* c) {
  if (!c) return 0;
  long long b = (long long)c->fft_work_bytes;
  for (int i = 0; i < 3; ++i) b += (long long)c->scratch_bytes[i];
  if (c->delta) b += wedge_size(c->delta_L) * 8;
  b += c->table_bytes;
  return b;
}

int scv_set_option(scv_ctx* c, const char* name, int value) {
  if (!c || !name) return SCV_EINVAL;
  const std::string n(name);
  if (n == "betaq") {
    if (value < -1 || value > 1) return scv_fail(c, SCV_EINVAL, "betaq option must be -1, 0 or 1");
    c->opt_betaq = value;
    return SCV_OK;
  }
  if (n == "chunkt") {
    if (value < -1 || value > 1) return scv_fail(c, SCV_EINVAL, "chunkt option must be -1, 0 or 1");
    c->opt_chunkt = value < 0 ? 0 : value;
    return SCV_OK;
  }
  if (n == "pin") {  // 1: a graph captured on this context is alive; 0: it was released
    if (value != 0 && value != 1) return scv_fail(c, SCV_EINVAL, "pin option must be 0 or 1");
    c->pinned = value ? c->pinned + 1 : (c->pinned > 0 ? c->pinned - 1 : 0);
    return SCV_OK;
  }
  if (n == "colgen") {
    if (value < -1 || value > 1) return scv_fail(c, SCV_EINVAL, "colgen option must be -1, 0 or 1");
    c->opt_colgen = value < 0 ? 1 : value;
    return SCV_OK;
  }
  return scv_fail(c, SCV_EINVAL, "unknown option " + n);
}

int scv_trim(scv_ctx* c) {
  if (!c) return SCV_EINVAL;
  SCV_TRY(scv_check_unpinned(c, "trim the workspace"));
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int i = 0; i < 3; ++i) {
    if (c->scratch[i]) cudaFree(c->scratch[i]);
    c->scratch[i] = nullptr;
    c->scratch_bytes[i] = 0;
  }
  for (auto& kv : c->plans) cufftDestroy(kv.second.h);
  c->plans.clear();
  if (c->fft_work) cudaFree(c->fft_work);
  c->fft_work = nullptr;
  c->fft_work_bytes = 0;
  // the large per-L tables are rebuilt on next use: the beta-quadrature tables
  // (8 L^3 bytes each; the small prime-factor / task tables stay) and the
  // Delta wedge
  for (auto it = c->aux.begin(); it != c->aux.end();) {
    if (it->first.rfind("betaq", 0) == 0) {
      cudaFree(it->second);
      it = c->aux.erase(it);
    } else {
      ++it;
    }
  }
  c->table_bytes = c->small_table_bytes;
  if (c->delta) cudaFree(c->delta);
  c->delta = nullptr;
  c->delta_L = 0;
  return SCV_OK;
}

int scv_halfpi_wedge(scv_ctx* c, int L, double* out, void* stream) {
  if (!c) return SCV_EINVAL;
  if (L < 1) return scv_fail(c, SCV_EINVAL, "band limit must be positive, got " + std::to_string(L));
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_TRY(scv_ensure_delta(c, L, s));
  SCV_CUDA(c, cudaMemcpyAsync(out, c->delta, (size_t)wedge_size(L) * 8, cudaMemcpyDeviceToDevice, s));
  return SCV_OK;
}

}  // extern "C"
