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
//
// Range: the border values 2^-l sqrt(C(2l, l+m)) leave the double range near
// |m| = l once l > ~1022, where the reference's float64 closed form
// underflows to 0 and the recursion then keeps the entries grown from it at 0
// (wrong for L > 1024: the SHT round trip fails near |m'|, |m| ~ 0.7 l).
// The seed arrives as mantissa + exponent; a seed below the normal range
// starts the recursion scaled by 2^e (exact: the recursion is linear and
// homogeneous), the shift is released as the values grow, and each plane
// entry is written as ldexp(v, -e) (rounding correctly to a subnormal / 0
// only where the true value is that small).  Seeds inside the normal range
// run unscaled, bit-identical to the plain recursion.

#include "scv_internal.cuh"

__global__ void __launch_bounds__(256) k_delta_wedge(int L, const double* __restrict__ edge,
                                                     const int* __restrict__ edge_e, double* __restrict__ out) {
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
  int sh = 0;  // values held scaled by 2^sh (sh > 0 only while below the normal range)
  for (int l = a; l < L; ++l) {
    double v;
    if (l == a) {
      const int ex = edge_e[t];
      if (ex >= -1021) {
        v = ldexp(edge[t], ex);  // normal: exactly the rounded double seed
      } else {
        v = edge[t];
        sh = -ex;
      }
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
    if (sh > 0 && v != 0.0) {
      // release the shift as the scaled value grows past 1 (both carried
      // predecessors move by the same power of two)
      const int k = min(ilogb(v), sh);
      if (k > 0) {
        v = ldexp(v, -k);
        p1 = ldexp(p1, -k);
        sh -= k;
      }
    }
    out[wedge_plane_base(l) + t] = sh > 0 ? ldexp(v, -sh) : v;
    p2 = p1;
    p1 = v;
  }
}

int scv_launch_delta_wedge(scv_ctx* c, int L, const double* edge, const int* edge_e, double* out, cudaStream_t s) {
  long long total = (long long)L * (L + 1) / 2;
  int blocks = (int)((total + 255) / 256);
  k_delta_wedge<<<blocks, 256, 0, s>>>(L, edge, edge_e, out);
  c->launches++;
  SCV_CUDA(c, cudaGetLastError());
  return SCV_OK;
}
