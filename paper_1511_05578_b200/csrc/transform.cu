// Whole-map entry points: the scale loop of the reference's analyze / synthesize
// (transform.py:139-187, real variants :190-253) as ONE C call each, so a binding
// crosses the FFI twice per round trip instead of ~4 times per scale.  They only
// sequence the per-stage entry points of this library on the caller's stream: same
// kernels, same order, bit-identical to calling the stages one by one
// (tests/test_whole_map_abi.py).
#include "scv_internal.cuh"

namespace {
// carve a 256-byte aligned piece out of the caller's work buffer
struct Carver {
  char* p;
  long long left;
  void* take(long long bytes) {
    const long long b = (bytes + 255) & ~255LL;
    if (b > left) return nullptr;
    void* r = p;
    p += b;
    left -= b;
    return r;
  }
};
long long aligned(long long bytes) { return (bytes + 255) & ~255LL; }
int check_scales(scv_ctx* c, int L, int spin, int real, int nscales, const int* Lj, int Ls) {
  if (L < 1) return scv_fail(c, SCV_EINVAL, "band limit must be positive");
  if (real && spin != 0) return scv_fail(c, SCV_EINVAL, "real maps must have spin 0");
  if ((spin < 0 ? -spin : spin) >= L) return scv_fail(c, SCV_EINVAL, "spin out of range for the band limit");
  if (nscales < 0 || (nscales > 0 && !Lj)) return scv_fail(c, SCV_EINVAL, "scale band limits missing");
  for (int j = 0; j < nscales; ++j)
    if (Lj[j] < 1 || Lj[j] > L) return scv_fail(c, SCV_EINVAL, "scale band limit must lie in [1, L]");
  if (Ls < 1 || Ls > L) return scv_fail(c, SCV_EINVAL, "scaling band limit must lie in [1, L]");
  return SCV_OK;
}
}  // namespace

extern "C" {

long long scv_map_work_bytes(int L, int Lmax, int Ls) {
  if (L < 1 || Lmax < 1 || Ls < 1) return 0;
  return aligned(16LL * L * L) + aligned(16LL * 2 * Lmax * (2LL * Lmax - 1)) + aligned(16LL * Ls * Ls);
}

int scv_analyze(scv_ctx* c, int L, int spin, int real, int nscales, const int* Lj, const double* const* psi_pos,
                const double* const* psi_neg, const double* scaling, int Ls, const void* f, void* const* sig,
                void* scaling_map, void* work, long long work_bytes, void* stream) {
  if (!c) return SCV_EINVAL;
  SCV_TRY(check_scales(c, L, spin, real, nscales, Lj, Ls));
  if (!f || !scaling || !scaling_map || !work || (nscales > 0 && (!psi_pos || !psi_neg || !sig)))
    return scv_fail(c, SCV_EINVAL, "scv_analyze: null buffer");
  int Lmax = 1;
  for (int j = 0; j < nscales; ++j) Lmax = Lj[j] > Lmax ? Lj[j] : Lmax;
  Carver cv{(char*)work, work_bytes};
  double* flm = (double*)cv.take(16LL * L * L);
  double* w = (double*)cv.take(16LL * 2 * Lmax * (2LL * Lmax - 1));
  double* s = (double*)cv.take(16LL * Ls * Ls);
  if (!flm || !w || !s) return scv_fail(c, SCV_EINVAL, "scv_analyze: work buffer smaller than scv_map_work_bytes");
  SCV_TRY(scv_sht_forward(c, L, spin, real, f, flm, stream));
  for (int j = 0; j < nscales; ++j) {  // transform.py:146-149
    SCV_TRY(scv_scale_product(c, L, Lj[j], flm, psi_pos[j], psi_neg[j], w, stream));
    SCV_TRY(scv_so3_inverse_curvelet(c, Lj[j], real, w, sig[j], stream));
  }
  SCV_TRY(scv_scaling_product(c, L, Ls, flm, scaling, s, stream));  // transform.py:150-151
  return scv_sht_inverse(c, Ls, 0, real, s, scaling_map, stream);
}

int scv_synthesize(scv_ctx* c, int L, int spin, int real, int nscales, const int* Lj, const double* const* psi_pos,
                   const double* const* psi_neg, const double* scaling, int Ls, const void* const* sig,
                   const void* scaling_map, void* f, void* work, long long work_bytes, void* stream) {
  if (!c) return SCV_EINVAL;
  SCV_TRY(check_scales(c, L, spin, real, nscales, Lj, Ls));
  if (!f || !scaling || !scaling_map || !work || (nscales > 0 && (!psi_pos || !psi_neg || !sig)))
    return scv_fail(c, SCV_EINVAL, "scv_synthesize: null buffer");
  int Lmax = 1;
  for (int j = 0; j < nscales; ++j) Lmax = Lj[j] > Lmax ? Lj[j] : Lmax;
  Carver cv{(char*)work, work_bytes};
  double* acc = (double*)cv.take(16LL * L * L);
  double* w = (double*)cv.take(16LL * 2 * Lmax * (2LL * Lmax - 1));
  double* slm = (double*)cv.take(16LL * Ls * Ls);
  if (!acc || !w || !slm)
    return scv_fail(c, SCV_EINVAL, "scv_synthesize: work buffer smaller than scv_map_work_bytes");
  cudaStream_t st = (cudaStream_t)stream;
  SCV_CUDA(c, cudaSetDevice(c->device));
  SCV_CUDA(c, cudaMemsetAsync(acc, 0, 16LL * L * L, st));
  for (int j = 0; j < nscales; ++j) {  // coarse -> fine, transform.py:164-178
    SCV_TRY(scv_so3_forward_curvelet(c, Lj[j], real, sig[j], w, stream));
    SCV_TRY(scv_accumulate(c, L, Lj[j], w, psi_pos[j], psi_neg[j], acc, stream));
  }
  SCV_TRY(scv_sht_forward(c, Ls, 0, real, scaling_map, slm, stream));  // transform.py:179-185
  SCV_TRY(scv_accumulate_scaling(c, L, Ls, slm, scaling, acc, stream));
  SCV_TRY(scv_finish_acc(c, L, spin, real, acc, stream));
  return scv_sht_inverse(c, L, spin, real, acc, f, stream);
}

}  // extern "C"
