// Delta^l_{m'm} = d^l_{m'm}(pi/2) by the three-term degree recursion,
// restated from the reference's build_halfpi_table (wigner.py:164-223):
//
//   Delta^l = l / sqrt((l^2-m'^2)(l^2-m^2)) * (a Delta^{l-1} - b Delta^{l-2}),
//   a = -(2l-1) m' m / ((l-1) l),  b = sqrt(((l-1)^2-m'^2)((l-1)^2-m^2)) / (l-1),
//
// interior of every plane, with the border row m'=l from the closed form
// (wigner.py:153-161) and the rest of the plane from the symmetries.
//
// B200 design: the recursion is element-wise in (m', m) -- entry (m', m) of
// plane l needs only entry (m', m) of planes l-1 and l-2.  So one thread owns
// one wedge element (0 <= m <= m' < L), carries its two predecessors in
// registers and walks l upward, writing plane after plane.  No inter-thread
// communication, no reads after the edge row, and consecutive threads write
// consecutive addresses of every plane (coalesced).  The products are
// evaluated with explicit round-to-nearest intrinsics (no FMA contraction)
// in the reference's operation order, so planes match numpy's arithmetic.

#include "scv_internal.cuh"

__global__ void __launch_bounds__(256) k_delta_wedge(int L, const double* __restrict__ edge,
                                                     double* __restrict__ out) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long total = (long long)L * (L + 1) / 2;
  if (t >= total) return;
  int a = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((long long)(a + 1) * (a + 2) / 2 <= t) ++a;
  while ((long long)a * (a + 1) / 2 > t) --a;
  const int b = (int)(t - (long long)a * (a + 1) / 2);
  const double mp = (double)a, m = (double)b;
  const double mp2 = __dmul_rn(mp, mp), m2 = __dmul_rn(m, m);
  double p1 = 0.0, p2 = 0.0;
  for (int l = a; l < L; ++l) {
    double v;
    if (l == a) {
      v = edge[t];
    } else if (l == 1) {
      v = 0.0;  // Delta^1_{00} of the seed plane (wigner.py:214-218)
    } else {
      const double dl = (double)l, lm1 = dl - 1.0;
      // a = -(2l-1) * m' * m / ((l-1) * l)
      double ac = __ddiv_rn(__dmul_rn(__dmul_rn(-(__dsub_rn(__dmul_rn(2.0, dl), 1.0)), mp), m),
                            __dmul_rn(lm1, dl));
      double lm12 = __dmul_rn(lm1, lm1);
      double bc = __ddiv_rn(__dsqrt_rn(__dmul_rn(__dsub_rn(lm12, mp2), __dsub_rn(lm12, m2))), lm1);
      double l2 = __dmul_rn(dl, dl);
      double sc = __ddiv_rn(dl, __dsqrt_rn(__dmul_rn(__dsub_rn(l2, mp2), __dsub_rn(l2, m2))));
      double q2 = (a <= l - 2) ? p2 : 0.0;
      v = __dmul_rn(sc, __dsub_rn(__dmul_rn(ac, p1), __dmul_rn(bc, q2)));
    }
    out[wedge_plane_base(l) + t] = v;
    p2 = p1;
    p1 = v;
  }
}

int scv_launch_delta_wedge(scv_ctx* c, int L, const double* edge, double* out, cudaStream_t s) {
  long long total = (long long)L * (L + 1) / 2;
  int blocks = (int)((total + 255) / 256);
  k_delta_wedge<<<blocks, 256, 0, s>>>(L, edge, out);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}
