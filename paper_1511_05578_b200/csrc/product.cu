// Per-scale harmonic products and the synthesis accumulation
// (transform.py:104-115, 128-136, 170-186, 246-252).  O(L^2) elementwise
// kernels; one thread per output coefficient.

#include "scv_internal.cuh"

// w[sheet, l, c+m] for the (2, Lj, Kj) layout; zero outside 1<=l<Lj, |m|<=l
__global__ void k_scale_product(int Lj, const double2* __restrict__ flm, const double* __restrict__ pos,
                                const double* __restrict__ neg, double2* __restrict__ w) {
  const int K = 2 * Lj - 1;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2LL * Lj * K) return;
  const int sheet = (int)(t / ((long long)Lj * K));
  const int rem = (int)(t - (long long)sheet * Lj * K);
  const int l = rem / K;
  const int m = rem - l * K - (Lj - 1);
  double2 v = make_double2(0.0, 0.0);
  if (l >= 1 && m >= -l && m <= l) {
    const double p = pos[l], q = neg[l];
    if (!(p == 0.0 && q == 0.0)) {
      const double fac = 8.0 * SCV_PI * SCV_PI / (double)(2 * l + 1);
      const double2 f = flm[(long long)l * l + l + m];
      const double2 row = make_double2(fac * f.x, fac * f.y);
      const double s = sheet == 0 ? p : q;
      v = make_double2(row.x * s, row.y * s);
    }
  }
  w[t] = v;
}

__global__ void k_scaling_product(int Ls, const double2* __restrict__ flm, const double* __restrict__ scaling,
                                  double2* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Ls * Ls) return;
  int l = (int)sqrt((double)t);
  while (l * l > t) --l;
  while ((l + 1) * (l + 1) <= t) ++l;
  double2 v = make_double2(0.0, 0.0);
  double a = scaling[l];
  if (a != 0.0) {
    a *= sqrt(4.0 * SCV_PI / (double)(2 * l + 1));
    const double2 f = flm[t];
    v = make_double2(a * f.x, a * f.y);
  }
  out[t] = v;
}

__global__ void k_accumulate(int Lj, const double2* __restrict__ w, const double* __restrict__ pos,
                             const double* __restrict__ neg, double2* __restrict__ acc) {
  const int K = 2 * Lj - 1;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Lj * Lj) return;
  int l = (int)sqrt((double)t);
  while (l * l > t) --l;
  while ((l + 1) * (l + 1) <= t) ++l;
  if (l < 1) return;
  const double p = pos[l], q = neg[l];
  if (p == 0.0 && q == 0.0) return;
  const int m = t - l * l - l;
  const double2 a = w[(long long)l * K + (Lj - 1) + m];
  const double2 b = w[((long long)Lj + l) * K + (Lj - 1) + m];
  const double2 add = make_double2(a.x * p + b.x * q, a.y * p + b.y * q);
  double2 r = acc[t];
  acc[t] = make_double2(r.x + add.x, r.y + add.y);
}

__global__ void k_accumulate_scaling(int Ls, const double2* __restrict__ slm, const double* __restrict__ scaling,
                                     double2* __restrict__ acc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Ls * Ls) return;
  int l = (int)sqrt((double)t);
  while (l * l > t) --l;
  while ((l + 1) * (l + 1) <= t) ++l;
  double a = scaling[l];
  if (a == 0.0) return;
  a *= sqrt(4.0 * SCV_PI / (double)(2 * l + 1));
  const double2 s = slm[t];
  double2 r = acc[t];
  acc[t] = make_double2(r.x + a * s.x, r.y + a * s.y);
}

__global__ void k_finish_acc(int L, int spin, int real, double2* __restrict__ acc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L * L) return;
  if (t < spin * spin) {
    acc[t] = make_double2(0.0, 0.0);
    return;
  }
  if (!real) return;
  int l = (int)sqrt((double)t);
  while (l * l > t) --l;
  while ((l + 1) * (l + 1) <= t) ++l;
  const int m = t - l * l - l;
  if (m == 0) {
    acc[t].y = 0.0;
  } else if (m < 0) {
    const double2 v = acc[l * l + l - m];
    acc[t] = ((-m) & 1) ? make_double2(-v.x, v.y) : make_double2(v.x, -v.y);
  }
}

extern "C" {

int scv_scale_product(scv_ctx* c, int L, int Lj, const double* flm, const double* pos, const double* neg,
                      double* w, void* stream) {
  if (!c) return SCV_EINVAL;
  if (Lj < 1 || Lj > L) return scv_fail(c, SCV_EINVAL, "scale band limit must lie in [1, L]");
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "product");
  const long long tot = 2LL * Lj * (2 * Lj - 1);
  k_scale_product<<<(int)((tot + 255) / 256), 256, 0, s>>>(Lj, (const double2*)flm, pos, neg, (double2*)w);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

int scv_scaling_product(scv_ctx* c, int L, int Ls, const double* flm, const double* scaling, double* out,
                        void* stream) {
  if (!c) return SCV_EINVAL;
  if (Ls < 1 || Ls > L) return scv_fail(c, SCV_EINVAL, "scaling band limit must lie in [1, L]");
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "product");
  k_scaling_product<<<(Ls * Ls + 255) / 256, 256, 0, s>>>(Ls, (const double2*)flm, scaling, (double2*)out);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

int scv_accumulate(scv_ctx* c, int L, int Lj, const double* w, const double* pos, const double* neg, double* acc,
                   void* stream) {
  if (!c) return SCV_EINVAL;
  if (Lj < 1 || Lj > L) return scv_fail(c, SCV_EINVAL, "scale band limit must lie in [1, L]");
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "product");
  k_accumulate<<<(Lj * Lj + 255) / 256, 256, 0, s>>>(Lj, (const double2*)w, pos, neg, (double2*)acc);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

int scv_accumulate_scaling(scv_ctx* c, int L, int Ls, const double* slm, const double* scaling, double* acc,
                           void* stream) {
  if (!c) return SCV_EINVAL;
  if (Ls < 1 || Ls > L) return scv_fail(c, SCV_EINVAL, "scaling band limit must lie in [1, L]");
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "product");
  k_accumulate_scaling<<<(Ls * Ls + 255) / 256, 256, 0, s>>>(Ls, (const double2*)slm, scaling, (double2*)acc);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

int scv_finish_acc(scv_ctx* c, int L, int spin, int real, double* acc, void* stream) {
  if (!c) return SCV_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  const int as = spin < 0 ? -spin : spin;
  k_finish_acc<<<(L * L + 255) / 256, 256, 0, s>>>(L, as, real, (double2*)acc);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

}  // extern "C"
