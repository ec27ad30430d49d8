// Sparsity statistics of curvelet coefficients on the device (SURVEY 8(f)
// row 4): the reference's `scurve sparsity` command (cli.py:268-320) and
// `gini_coefficient` (cli.py:59-70), per scale:
//   mags = |c| over the scale volume; top = max mags;
//   counts = np.histogram(mags / top, bins, range=(0, 1))  (numpy's uniform-bin rule, exact);
//   gini = sum_i (2 i - n - 1) x_(i) / (n sum_i x_i), x sorted ascending, i = 1..n.
// Magnitudes are one HBM stream; the Gini needs the sorted sample (a device
// radix sort of float64 keys, CUB), then one deterministic reduction.
#include <cub/device/device_radix_sort.cuh>

#include "scv_internal.cuh"

namespace {

// |c| (complex: hypot, as numpy's abs) into mags; running max into *top via
// the order of non-negative doubles as unsigned integers
__global__ void k_abs_max(long long n, int is_complex, const void* __restrict__ v, double* __restrict__ mags,
                          unsigned long long* __restrict__ top) {
  double m = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double a;
    if (is_complex) {
      const double2 c = __ldcs((const double2*)v + i);
      a = hypot(c.x, c.y);
    } else {
      a = fabs(__ldcs((const double*)v + i));
    }
    if (mags) mags[i] = a;
    m = fmax(m, a);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(top, (unsigned long long)__double_as_longlong(m));
}

// np.histogram(x / top, bins, range=(0, 1)) with numpy's index rule for
// uniform bins (lib/_histograms_impl.py): i = floor(x * bins), clipped to
// bins-1 at x == 1, then moved down if x < edge[i] and up if x >= edge[i+1]
// (except in the last bin).  Edges are numpy's linspace(0, 1, bins+1).
__global__ void k_hist(long long n, const double* __restrict__ mags, const unsigned long long* __restrict__ top,
                       int bins, const double* __restrict__ edges, unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned long long sh[];
  for (int b = threadIdx.x; b < bins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const double t = __longlong_as_double((long long)*top);
  const double norm = (double)bins / (edges[bins] - edges[0]);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double x = mags[i] / t;
    if (!(x >= edges[0] && x <= edges[bins])) continue;
    long long k = (long long)((x - edges[0]) * norm);
    if (k == bins) k -= 1;
    if (x < edges[k]) k -= 1;
    else if (k != bins - 1 && x >= edges[k + 1]) k += 1;
    atomicAdd(&sh[k], 1ULL);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < bins; b += blockDim.x)
    if (sh[b]) atomicAdd(&counts[b], sh[b]);
}

// per-block partial sums of (2 i - n - 1) x_i (i = 1-based rank) and x_i over
// a fixed grid-stride partition; summed in block order by k_gini_final
constexpr int GINI_BLOCKS = 1184, GINI_NT = 256;
__global__ void __launch_bounds__(GINI_NT) k_gini_part(long long n, const double* __restrict__ x, double2* __restrict__ part) {
  __shared__ double sa[GINI_NT], sb[GINI_NT];
  double a = 0.0, b = 0.0;
  const double nn = (double)n;
  for (long long i = (long long)blockIdx.x * GINI_NT + threadIdx.x; i < n; i += (long long)gridDim.x * GINI_NT) {
    const double v = __ldcs(x + i);
    a = fma(2.0 * (double)(i + 1) - nn - 1.0, v, a);
    b += v;
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int s = GINI_NT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sa[threadIdx.x] += sa[threadIdx.x + s];
      sb[threadIdx.x] += sb[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = make_double2(sa[0], sb[0]);
}

__global__ void k_gini_final(int nparts, const double2* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int i = 0; i < nparts; ++i) {
    a += part[i].x;
    b += part[i].y;
  }
  out[0] = a;
  out[1] = b;
}

int grid_for(long long n, int nt) {
  long long g = (n + nt - 1) / nt;
  return (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

}  // namespace

extern "C" {

int scv_abs_max(scv_ctx* c, long long n, int is_complex, const void* v, double* mags, double* top, void* stream) {
  if (!c) return SCV_EINVAL;
  if (n < 0) return scv_fail(c, SCV_EINVAL, "negative element count");
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "sparsity");
  if (n == 0) return SCV_OK;
  k_abs_max<<<grid_for(n, 256), 256, 0, s>>>(n, is_complex, v, mags, (unsigned long long*)top);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

int scv_histogram(scv_ctx* c, long long n, const double* mags, const double* top, int bins, const double* edges,
                  unsigned long long* counts, void* stream) {
  if (!c) return SCV_EINVAL;
  if (bins < 1) return scv_fail(c, SCV_EINVAL, "--bins must be at least 1");
  if (bins > 4096) return scv_fail(c, SCV_EINVAL, "at most 4096 bins");
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "sparsity");
  if (n == 0) return SCV_OK;
  k_hist<<<grid_for(n, 256), 256, (size_t)bins * 8, s>>>(n, mags, (const unsigned long long*)top, bins, edges, counts);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

int scv_sort_f64(scv_ctx* c, long long n, double* keys, double* alt, int* in_alt, void* stream) {
  if (!c) return SCV_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "sparsity");
  *in_alt = 0;
  if (n <= 1) return SCV_OK;
  cub::DoubleBuffer<double> db(keys, alt);
  size_t tmp = 0;
  SCV_CUDA(c, cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, n, 0, 64, s));
  void* t = nullptr;
  SCV_TRY(scv_scratch(c, 0, tmp, &t));
  SCV_CUDA(c, cub::DeviceRadixSort::SortKeys(t, tmp, db, n, 0, 64, s));
  c->launches++;
  *in_alt = db.Current() == alt ? 1 : 0;
  return SCV_OK;
}

int scv_gini_sums(scv_ctx* c, long long n, const double* sorted, double* out, void* stream) {
  if (!c) return SCV_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_PROF(c, s, "sparsity");
  void* part = nullptr;
  SCV_TRY(scv_scratch(c, 2, (size_t)GINI_BLOCKS * 16, &part));
  k_gini_part<<<GINI_BLOCKS, GINI_NT, 0, s>>>(n, sorted, (double2*)part);
  k_gini_final<<<1, 32, 0, s>>>(GINI_BLOCKS, (const double2*)part, out);
  c->launches += 2;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}

}  // extern "C"
