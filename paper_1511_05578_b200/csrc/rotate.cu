// Frame rotation of one scale's Wigner coefficients to / from the frame of
// the pole-centred curvelet:
//   rotate_to_north   transform.py:256-277
//   rotate_from_north transform.py:280-297
//   wigner_d_edge_columns wigner.py:304-322
//
// Dense Wigner coefficients are stored as the reference's list of planes,
// packed back to back: plane l (rows m + l, columns k + l, (2l+1)^2 complex128)
// starts at l(4l^2 - 1)/3.  Row m of plane l is then the contiguous run of
// 2l+1 entries at plane_off(l) + (m + l)(2l + 1), and the flat row index
// l^2 + l + m is the harmonic index, so one warp owns one row.
//
// Both directions are HBM-bound streams over the dense volume (16 bytes per
// entry, L(4L^2-1)/3 entries: 22.9 GB at L=1024); the edge columns
// d^l_{k,+-l}(theta) are an O(L^2) table (33 MB at L=1024) that stays in L2.
#include "scv_internal.cuh"

namespace {

__device__ __forceinline__ long long plane_off(int l) { return (long long)l * (4LL * l * l - 1) / 3; }

__device__ __forceinline__ int isqrt_row(int r) {
  int l = (int)sqrt((double)r);
  while (l * l > r) --l;
  while ((l + 1) * (l + 1) <= r) ++l;
  return l;
}

// xlogy(n, e^lg): 0 when n == 0 (also for lg = -inf), else n * lg
__device__ __forceinline__ double xlogy_n(int n, double lg) { return n == 0 ? 0.0 : __dmul_rn((double)n, lg); }

// E[l * K + k + L - 1] = (d^l_{k,+l}(theta), d^l_{k,-l}(theta)) for |k| <= l, 0 elsewhere:
//   pos = exp(hlb + (l-k) ln sin(theta/2) + (l+k) ln cos(theta/2))
//   neg = (-1)^(l-k) exp(hlb + (l+k) ln sin(theta/2) + (l-k) ln cos(theta/2))
// with hlb = 0.5 ln C(2l, l+k) (wigner.py:304-322).
__global__ void k_edge_cols(int L, const double* __restrict__ hlb, double ls, double lc, double2* __restrict__ E) {
  const int K = 2 * L - 1;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)L * K) return;
  const int l = (int)(t / K);
  const int k = (int)(t - (long long)l * K) - (L - 1);
  double2 v = make_double2(0.0, 0.0);
  if (k >= -l && k <= l) {
    const double h = hlb[(long long)l * (l + 1) / 2 + (k < 0 ? -k : k)];
    const double ap = __dadd_rn(xlogy_n(l - k, ls), xlogy_n(l + k, lc));
    const double an = __dadd_rn(xlogy_n(l + k, ls), xlogy_n(l - k, lc));
    v.x = exp(__dadd_rn(h, ap));
    v.y = exp(__dadd_rn(h, an));
    if ((l - k) & 1) v.y = -v.y;
  }
  E[t] = v;
}

__device__ __forceinline__ double2 rot_entry(int l, double2 a, double2 b, double2 d) {
  double2 v;
  if (l > 0) {
    v.x = __dadd_rn(__dmul_rn(a.x, d.x), __dmul_rn(b.x, d.y));
    v.y = __dadd_rn(__dmul_rn(a.y, d.x), __dmul_rn(b.y, d.y));
  } else {
    v.x = __dmul_rn(a.x, d.x);
    v.y = __dmul_rn(a.y, d.x);
  }
  return v;
}

// plane_l[m][k] = w0[l][m] pos_l[k] + w1[l][m] neg_l[k]  (w1 term for l >= 1),
// products and sum rounded separately (no FMA), as numpy's outer products.
__global__ void __launch_bounds__(256) k_rot_to_north(int L, const double2* __restrict__ w,
                                                      const double2* __restrict__ E, double2* __restrict__ out) {
  const int K = 2 * L - 1;
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < L * L; r += nw) {
    const int l = isqrt_row(r);
    const int m = r - l * l - l;
    const int n = 2 * l + 1;
    const double2 a = w[(long long)l * K + (L - 1) + m];
    const double2 b = l > 0 ? w[((long long)L + l) * K + (L - 1) + m] : make_double2(0.0, 0.0);
    const double2* e = E + (long long)l * K + (L - 1) - l;
    double2* o = out + plane_off(l) + (long long)(m + l) * n;
    // (a four-deep batch of edge-table loads before the stores measured 2% slower:
    // 4.37 vs 4.28 ms at L=1024)
    for (int k = lane; k < n; k += 32) __stcs(o + k, rot_entry(l, a, b, __ldg(e + k)));
  }
}

// w[0][l][m] = sum_k plane_l[m][k] pos_l[k], w[1][l][m] = sum_k plane_l[m][k] neg_l[k]
// (l >= 1); a warp streams one row with four 16-byte loads in flight per lane
// and reduces by shuffles.  w must be zero outside |m| <= l (memset by the caller).
__global__ void __launch_bounds__(256) k_rot_from_north(int L, const double2* __restrict__ dense,
                                                        const double2* __restrict__ E, double2* __restrict__ w) {
  const int K = 2 * L - 1;
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < L * L; r += nw) {
    const int l = isqrt_row(r);
    const int m = r - l * l - l;
    const int n = 2 * l + 1;
    const double2* e = E + (long long)l * K + (L - 1) - l;
    const double2* x = dense + plane_off(l) + (long long)(m + l) * n;
    double pr = 0.0, pi = 0.0, nr = 0.0, ni = 0.0;
    int k = lane;
    for (; k + 96 < n; k += 128) {
      double2 v[4], d[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(x + k + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) d[u] = __ldg(e + k + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        pr = fma(v[u].x, d[u].x, pr);
        pi = fma(v[u].y, d[u].x, pi);
        nr = fma(v[u].x, d[u].y, nr);
        ni = fma(v[u].y, d[u].y, ni);
      }
    }
    for (; k < n; k += 32) {
      const double2 v = __ldcs(x + k), d = __ldg(e + k);
      pr = fma(v.x, d.x, pr);
      pi = fma(v.y, d.x, pi);
      nr = fma(v.x, d.y, nr);
      ni = fma(v.y, d.y, ni);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      pr += __shfl_xor_sync(0xffffffffu, pr, o);
      pi += __shfl_xor_sync(0xffffffffu, pi, o);
      nr += __shfl_xor_sync(0xffffffffu, nr, o);
      ni += __shfl_xor_sync(0xffffffffu, ni, o);
    }
    if (lane == 0) {
      w[(long long)l * K + (L - 1) + m] = make_double2(pr, pi);
      if (l > 0) w[((long long)L + l) * K + (L - 1) + m] = make_double2(nr, ni);
    }
  }
}

int rot_grid() {
  static int g = 0;
  if (!g) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g = sms * 8;  // 8 CTAs x 8 warps per SM
  }
  return g;
}

int edge_table(scv_ctx* c, int L, double theta, cudaStream_t s, double2** E) {
  if (L < 1) return scv_fail(c, SCV_EINVAL, "band limit must be positive");
  if (!(theta >= 0.0 && theta <= SCV_PI + 1e-12)) return scv_fail(c, SCV_EINVAL, "rotation angle must lie in [0, pi]");
  SCV_TRY(scv_ensure_hlb(c, L, s));
  const int K = 2 * L - 1;
  void* p = nullptr;
  SCV_TRY(scv_scratch(c, 2, (size_t)L * K * 16, &p));
  const double sh = std::sin(0.5 * theta), ch = std::cos(0.5 * theta);
  const double ls = sh > 0.0 ? std::log(sh) : -INFINITY;
  const double lc = ch > 0.0 ? std::log(ch) : -INFINITY;
  const long long tot = (long long)L * K;
  k_edge_cols<<<(int)((tot + 255) / 256), 256, 0, s>>>(L, c->hlb, ls, lc, (double2*)p);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  *E = (double2*)p;
  return SCV_OK;
}

}  // namespace

extern "C" {

int scv_edge_columns(scv_ctx* c, int L, double theta, double* out, void* stream) {
  if (!c) return SCV_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "rotate");
  double2* E = nullptr;
  SCV_TRY(edge_table(c, L, theta, s, &E));
  SCV_CUDA(c, cudaMemcpyAsync(out, E, (size_t)L * (2 * L - 1) * 16, cudaMemcpyDeviceToDevice, s));
  return SCV_OK;
}

int scv_rotate_to_north(scv_ctx* c, int L, double theta, const double* w, double* dense, void* stream) {
  if (!c) return SCV_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "rotate");
  double2* E = nullptr;
  SCV_TRY(edge_table(c, L, theta, s, &E));
  k_rot_to_north<<<rot_grid(), 256, 0, s>>>(L, (const double2*)w, E, (double2*)dense);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

int scv_rotate_from_north(scv_ctx* c, int L, double theta, const double* dense, double* w, void* stream) {
  if (!c) return SCV_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "rotate");
  double2* E = nullptr;
  SCV_TRY(edge_table(c, L, theta, s, &E));
  SCV_CUDA(c, cudaMemsetAsync(w, 0, (size_t)2 * L * (2 * L - 1) * 16, s));
  k_rot_from_north<<<rot_grid(), 256, 0, s>>>(L, (const double2*)dense, E, (double2*)w);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

}  // extern "C"
