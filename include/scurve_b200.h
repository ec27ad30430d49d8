/*
 * scurve_b200 — C ABI of the B200-native curvelet hot path.
 *
 * One shared library (libscurve_b200.so, sm_100a) exports the entry points
 * below.  They replace, one for one, the Python functions of the reference
 * package `scurve` that make up the curvelet analysis/synthesis path (paths
 * relative to /root/reference/pkg/src/scurve/):
 *
 *   scv_sht_forward            <- sht_forward / sht_forward_real   sphere.py:155-182, 210-236
 *   scv_sht_inverse            <- sht_inverse / sht_inverse_real   sphere.py:185-207, 239-260
 *   scv_scale_product          <- transform._scale_wigner          transform.py:104-115
 *   scv_scaling_product        <- transform._scaling_coeffs        transform.py:128-136
 *   scv_so3_inverse_curvelet   <- so3_inverse_curvelet(_real)      so3.py:259-285, 386-417
 *   scv_so3_forward_curvelet   <- so3_forward_curvelet(_real)      so3.py:214-244, 349-383
 *   scv_accumulate             <- the acc += W psi loop of synthesize  transform.py:170-178
 *   scv_finish_acc             <- acc[:s^2]=0 (+ real symmetry)    transform.py:186, 246-252
 *   scv_analyze                <- analyze / analyze_real (whole map) transform.py:139-152, 190-210
 *   scv_synthesize             <- synthesize / synthesize_real       transform.py:155-187, 213-253
 *   scv_halfpi_wedge           <- build_halfpi_table / halfpi_table wigner.py:209-240
 *   scv_edge_columns           <- wigner_d_edge_columns            wigner.py:304-322
 *   scv_rotate_to_north        <- rotate_to_north                  transform.py:256-277
 *   scv_rotate_from_north      <- rotate_from_north                transform.py:280-297
 *   scv_so3_inverse_general    <- so3_inverse_general (dense O(L^4)) so3.py:317-346
 *   scv_so3_forward_general    <- so3_forward_general (dense O(L^4)) so3.py:288-314
 *   scv_abs_max, scv_histogram,
 *   scv_sort_f64, scv_gini_sums <- cmd_sparsity / gini_coefficient  cli.py:59-70, 268-320
 *   scv_so3_inverse_curvelet_slab  <- so3_inverse_curvelet restricted to beta rows [b0, b0+nb)
 *   scv_so3_forward_curvelet_slab  <- the beta sum of so3_forward_curvelet over beta rows [b0, b0+nb)
 *                                     (so3.py:203-243; the multi-GPU beta-slab shards)
 *
 * Conventions
 *   - All data pointers are DEVICE pointers owned by the caller.  Complex
 *     values are interleaved float64 pairs (re, im), i.e. complex128.
 *   - Layouts are the reference's, byte for byte:
 *       sphere map     (L, 2L-1)             theta-major (complex128, or float64 when real)
 *       harmonic f_lm  (L*L,)                index l*l + l + m
 *       Wigner coeffs  (2, L, 2L-1)          sheet 0: n=+l, sheet 1: n=-l, m at m+L-1
 *       SO(3) signal   (2L-1, L, 2L-1)       (gamma, beta, alpha); complex128, or float64 when real
 *   - `stream` is a cudaStream_t passed as void*; every call is ordered on it
 *     and returns without synchronising.  Inputs are never modified.
 *   - A context is bound to one device and is not thread-safe.  It owns only
 *     its workspace: Delta(pi/2) wedge table, Bluestein/weight tables, cuFFT
 *     plans and scratch.  Workspace grows lazily and is freed by scv_destroy.
 *   - Return 0 on success or a negative SCV_E* code; scv_last_error() gives
 *     the message.  SCV_EINVAL corresponds to the reference's ValueError,
 *     SCV_ETYPE to TypeError, the rest to RuntimeError.
 */
#ifndef SCURVE_B200_H
#define SCURVE_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define SCV_OK 0
#define SCV_EINVAL (-1)
#define SCV_ETYPE (-2)
#define SCV_ECUDA (-3)
#define SCV_ENOMEM (-4)
#define SCV_ECUFFT (-5)

typedef struct scv_ctx scv_ctx;

/* ABI version (major*100 + minor). */
int scv_version(void);

/* Create a context on CUDA device `device`. */
int scv_create(int device, scv_ctx** out);
int scv_destroy(scv_ctx* ctx);
const char* scv_last_error(const scv_ctx* ctx);

/* Bytes of device memory currently held by the context: scratch workspace,
 * the Delta wedge and the per-L tables (beta quadrature, prime-factor). */
long long scv_workspace_bytes(const scv_ctx* ctx);
/* Release every lazily grown scratch buffer, the beta-quadrature tables and
 * the Delta wedge (all rebuilt on next use; the small prime-factor tables
 * stay).  Fails with SCV_EINVAL while a captured graph pins the context. */
int scv_trim(scv_ctx* ctx);

/* Stage profiler: when enabled, every launch group is bracketed by CUDA
 * events on its stream.  scv_profile_report synchronises the device and
 * writes "stage count total_ms\n" lines (then clears the records). */
int scv_profile(scv_ctx* ctx, int enable);
int scv_profile_report(scv_ctx* ctx, char* buf, int len);
/* Set a context option; value -1 restores the library default.
 *   "betaq": synthesis beta stage. 1 = precomputed beta quadrature table fused
 *            into the gamma pass (default for 128 <= L <= 2048 on the
 *            prime-factor lengths), 0 = per-column Bluestein/convolution FFTs
 *            and Delta contraction.  Both compute so3.py:203-243.
 *   "colgen": analysis order. 1 = gamma-first (closed-form columns over n,
 *            gamma IDFT, then the alpha IDFT over contiguous rows in place;
 *            default), 0 = alpha rows first, then gamma columns in place.
 *   "chunkt": synthesis beta-chunk layout. 0 = [b][g][m] (default),
 *            1 = [b][m][g] (strided alpha writes, contiguous gamma reads).
 * Returns SCV_EINVAL for an unknown name. */
int scv_set_option(scv_ctx* ctx, const char* name, int value);
/* Number of this library's own kernels launched by the context so far. */
long long scv_launch_count(const scv_ctx* ctx);

/* Measured FP64 FMA throughput of this device (TFLOP/s, 2 flops per DFMA),
 * from a register-resident DFMA loop over every SM; used as the roofline
 * denominator for FP64-bound stages (MEASURED_PEAKS.json has no FP64 entry). */
int scv_fp64_peak(scv_ctx* ctx, double* tflops);
/* measured FP64 tensor-core (DMMA m8n8k4) peak of this device, TFLOP/s:
   the denominator of the executed-DMMA fraction (bench.py) */
int scv_dmma_peak(scv_ctx* ctx, double* tflops);

/* Batched K-point DFT of `nrows` contiguous complex128 rows with the
 * hand-written prime-factor engine (K = 2^k - 1 up to 4095):
 * out[r][k] = sum_n in[r][n] exp(dir * 2 pi i n k / K), dir = -1 or +1.
 * Exposed for testing and benchmarking the engine in isolation. */
int scv_debug_dft(scv_ctx* ctx, int K, int dir, int nrows, const double* in, double* out,
                  void* stream);
/* Host-only views of the engine's shared-memory position maps (no device
 * needed): out_pos[k] = position of output frequency k, in_pos[n] = position
 * of input sample n (K ints each); and the storage order of a radix-89
 * butterfly's elements, sigma_in[j] / sigma_out[k] (89 ints each).  Tests
 * emulate the stages on these maps against numpy.fft (tests/test_pfa_maps.py). */
int scv_debug_pfa_maps(int K, int* out_pos, int* in_pos);
int scv_debug_r89_sigma(int* sigma_in, int* sigma_out);
/* Lane schedule of the ring kernels' slot copies (host arithmetic only): for each group of 32
 * consecutive output frequencies / input samples, entry [32 j + lane] = position | (e << 11)
 * says that the lane moves element 32 j + e.  K = 1023 or 2047 (positions fit 11 bits). */
int scv_debug_pfa_sched(int K, int* out_sched, int* in_sched);
/* Pipeline timing counters of the ring kernels (only counted in builds with
 * -DSCV_PIPE_STATS=1, zeros otherwise): 36 clock-cycle sums (kinds 3 and 4 are
 * sub-phases of the generator / quadrature teams), kernel kind
 * (rows, column generation, gamma+quadrature) * 6 + {transform groups waiting
 * for a full slot, transforming; load/store warps waiting for a transform,
 * draining, filling; unused}.  reset != 0 clears them. */
int scv_debug_pipe_stats(unsigned long long* out36, int reset);
/* Beta rows per alpha/gamma launch pair of the quadrature synthesis at band limit L.  The sum over
 * beta (so3.py:226-243 via the table) is formed chunk by chunk, so a caller that cuts a scale into
 * slabs at multiples of this gets the whole-scale summation order (roundtrip_streamed relies on it). */
int scv_syn_chunk_rows(int L);
/* Build the beta-quadrature table of band limit L (csrc/betaq.cu; the weights that
 * replace the reference's beta FFT + quadrature convolution + Delta contraction,
 * so3.py:203-243) with method 1 (two tensor-core GEMMs, the default) or 0 (direct
 * sums) and copy its first n doubles to the device buffer out.  Nothing is cached;
 * used to compare the two builds and to time them. */
int scv_debug_betaq_build(scv_ctx* ctx, int L, int method, double* out, long long n, void* stream);
/* Restrict this context's beta-quadrature table of band limit L to the beta rows [b0, b0 + nb):
 * the table a rank of the beta-slab decomposition needs (8 L^2 nb bytes instead of 8 L^3, and
 * 1/world of the second build GEMM).  Call before the first synthesis at L, or any time: a table
 * already built for another range is dropped and rebuilt on next use.  nb = 0 lifts the
 * restriction.  scv_so3_forward_curvelet(_slab) on rows outside the range then fails with
 * SCV_EINVAL.  The reference has no counterpart (its Delta cache, wigner.py:226-240, is global). */
int scv_betaq_restrict(scv_ctx* ctx, int L, int b0, int nb);

/* Delta^l_{m'm}(pi/2) for l < L in the 1/8 symmetry wedge 0 <= m <= m' <= l:
 * element (l, m', m) at l(l+1)(l+2)/6 + m'(m'+1)/2 + m.  Copies the context's
 * table (built on the device by the degree recursion) into `out`
 * (L(L+1)(L+2)/6 doubles).  wigner.py:153-240. */
int scv_halfpi_wedge(scv_ctx* ctx, int L, double* out, void* stream);

/* Forward spin SHT.  f: (L, 2L-1) complex128, or float64 if real (spin 0).
 * flm: (L*L) complex128. */
int scv_sht_forward(scv_ctx* ctx, int L, int spin, int real, const void* f, double* flm,
                    void* stream);

/* Inverse spin SHT.  flm (L*L) complex128 -> f (L, 2L-1) complex128, or
 * float64 if real (flm must then carry the real-signal symmetry). */
int scv_sht_inverse(scv_ctx* ctx, int L, int spin, int real, const double* flm, void* f,
                    void* stream);

/* Per-scale harmonic product: w (2, Lj, 2Lj-1) with
 * w[0,l,m] = 8pi^2/(2l+1) f_lm psi_pos[l], w[1,l,m] = ... psi_neg[l], 1<=l<Lj.
 * flm has band limit L >= Lj; psi_* are device arrays of length >= Lj. */
int scv_scale_product(scv_ctx* ctx, int L, int Lj, const double* flm, const double* psi_pos,
                      const double* psi_neg, double* w, void* stream);

/* Scaling coefficients: out (Ls*Ls) = sqrt(4pi/(2l+1)) scaling[l] f_lm, l<Ls. */
int scv_scaling_product(scv_ctx* ctx, int L, int Ls, const double* flm, const double* scaling,
                        double* out, void* stream);

/* Sparse inverse Wigner transform (analysis direction): w (2, Lj, 2Lj-1)
 * complex128 -> sig (2Lj-1, Lj, 2Lj-1), complex128 or float64 if real. */
int scv_so3_inverse_curvelet(scv_ctx* ctx, int Lj, int real, const double* w, void* sig,
                             void* stream);

/* Beta-slab variants (complex path; K = 2Lj-1 must be a prime-factor length).
 * A slab holds the beta rows [b0, b0+nb) of the scale signal as a
 * (2Lj-1, nb, 2Lj-1) array (gamma, beta-in-slab, alpha): slabs of one scale
 * on different GPUs hold disjoint rows of the same SO(3) signal.
 * inverse: w (2, Lj, 2Lj-1) -> the slab (rows b0.. of the full transform).
 * forward: the beta quadrature summed over the slab's rows only, written into
 * w (accumulate = 0) or added to it (accumulate = 1); the sum of the partials
 * of all slabs is scv_so3_forward_curvelet of the full signal.  Needs the
 * beta-quadrature path (128 <= Lj <= 2048); real = 1 reads a float64 slab. */
int scv_so3_inverse_curvelet_slab(scv_ctx* ctx, int Lj, const double* w, int b0, int nb, void* sig,
                                  void* stream);
int scv_so3_forward_curvelet_slab(scv_ctx* ctx, int Lj, int real, const void* sig, int b0, int nb,
                                  double* w, int accumulate, void* stream);

/* Sparse forward Wigner transform (synthesis direction): sig -> w. */
int scv_so3_forward_curvelet(scv_ctx* ctx, int Lj, int real, const void* sig, double* w,
                             void* stream);

/* acc (L*L) += w[0,l,m] psi_pos[l] + w[1,l,m] psi_neg[l] for 1 <= l < Lj. */
int scv_accumulate(scv_ctx* ctx, int L, int Lj, const double* w, const double* psi_pos,
                   const double* psi_neg, double* acc, void* stream);

/* acc += sqrt(4pi/(2l+1)) scaling[l] slm for l < Ls (slm has band limit Ls). */
int scv_accumulate_scaling(scv_ctx* ctx, int L, int Ls, const double* slm,
                           const double* scaling, double* acc, void* stream);

/* acc[: spin^2] = 0; if real, re-impose f_{l,-m} = (-1)^m conj f_{lm}, f_l0 real. */
int scv_finish_acc(scv_ctx* ctx, int L, int spin, int real, double* acc, void* stream);

/* Whole-map entry points: the reference's analyze / synthesize (transform.py:139-187; real = 1:
 * analyze_real / synthesize_real, :190-253) as one call each.  They sequence the per-stage entry
 * points above on `stream` (same kernels and order: bit-identical to calling the stages one by one).
 *   nscales, Lj[j]       scales coarse -> fine and the band limit each scale signal is stored at
 *                        (host array; min(ceil(lambda^(j+1)), L) in multiresolution mode, else L)
 *   psi_pos[j], psi_neg[j]  host arrays of DEVICE pointers: the curvelet kernel's n = +l / n = -l
 *                        harmonic columns of scale j (float64, length >= Lj[j])
 *   scaling, Ls          device array (float64, length >= Ls) and band limit of the scaling part
 *   f                    (L, 2L-1) complex128 map, float64 if real
 *   sig[j]               host array of DEVICE pointers: (2Lj-1, Lj, 2Lj-1) complex128 (float64 if
 *                        real) scale signals; written by scv_analyze, read by scv_synthesize
 *   scaling_map          (Ls, 2Ls-1) spin-0 scaling signal, complex128 (float64 if real)
 *   work                 device scratch of at least scv_map_work_bytes(L, max_j Lj[j], Ls) bytes
 * All device buffers are only touched by work enqueued on `stream`. */
long long scv_map_work_bytes(int L, int Lmax, int Ls);
int scv_analyze(scv_ctx* ctx, int L, int spin, int real, int nscales, const int* Lj,
                const double* const* psi_pos, const double* const* psi_neg, const double* scaling, int Ls,
                const void* f, void* const* sig, void* scaling_map, void* work, long long work_bytes,
                void* stream);
int scv_synthesize(scv_ctx* ctx, int L, int spin, int real, int nscales, const int* Lj,
                   const double* const* psi_pos, const double* const* psi_neg, const double* scaling, int Ls,
                   const void* const* sig, const void* scaling_map, void* f, void* work, long long work_bytes,
                   void* stream);

/* Frame rotation of one scale.  Dense Wigner coefficients
 * (the reference's WignerCoeffs.planes) are packed plane after plane: plane l,
 * (2l+1) x (2l+1) complex128 with rows m+l and columns k+l, starts at entry
 * l(4l^2-1)/3; L(4L^2-1)/3 entries in total.  theta is the scale's tiling
 * angle (Tiling.angles, in [pi/2, pi]).
 *
 * edge_columns: out (L, 2L-1, 2) float64, out[l][k+L-1] = (d^l_{k,+l}(theta),
 * d^l_{k,-l}(theta)) for |k| <= l, zero elsewhere.
 * rotate_to_north: w (2, L, 2L-1) -> dense planes,
 *   plane_l = outer(w[0,l], d_{.,+l}) + outer(w[1,l], d_{.,-l}) (l >= 1).
 * rotate_from_north: dense planes -> w (2, L, 2L-1), w[0,l] = plane_l d_{.,+l},
 *   w[1,l] = plane_l d_{.,-l} (l >= 1), zero outside |m| <= l and at w[1,0]. */
int scv_edge_columns(scv_ctx* ctx, int L, double theta, double* out, void* stream);
int scv_rotate_to_north(scv_ctx* ctx, int L, double theta, const double* w, double* dense,
                        void* stream);
int scv_rotate_from_north(scv_ctx* ctx, int L, double theta, const double* dense, double* w,
                          void* stream);

/* Dense inverse Wigner transform, O(L^4) (the reference's cross-check path):
 * planes = packed dense WignerCoeffs of band limit L (as for the rotation),
 * out (2gN-1, gL, 2gM-1) complex128 on the SO3Grid(gL, gM, gN); L <= gL, gM, gN. */
int scv_so3_inverse_general(scv_ctx* ctx, int L, int gL, int gM, int gN, const double* planes, double* out,
                            void* stream);
/* Dense forward Wigner transform, O(L^4): sig (2gN-1, gL, 2gM-1) complex128 ->
 * packed dense planes of band limit L <= gL, gM, gN. */
int scv_so3_forward_general(scv_ctx* ctx, int L, int gL, int gM, int gN, const double* sig, double* planes,
                            void* stream);

/* Sparsity statistics (cli.py:59-70, 268-320).
 * abs_max: mags[i] = |v[i]| (complex128 if is_complex, else float64; mags may
 *   be NULL), and *top = max(*top, max_i |v[i]|) on the device (*top >= 0).
 * histogram: counts[k] += #{i : x_i = mags[i] / *top falls in bin k} with
 *   numpy's uniform-bin rule over edges (bins+1 doubles, linspace(0, 1));
 *   counts are uint64.
 * sort_f64: ascending radix sort of n doubles; the result is in `keys`
 *   (*in_alt = 0) or `alt` (*in_alt = 1); both buffers are overwritten.
 * gini_sums: out[0] = sum_i (2(i+1) - n - 1) x_i, out[1] = sum_i x_i over the
 *   sorted x (deterministic reduction order). */
int scv_abs_max(scv_ctx* ctx, long long n, int is_complex, const void* v, double* mags, double* top,
                void* stream);
int scv_histogram(scv_ctx* ctx, long long n, const double* mags, const double* top, int bins,
                  const double* edges, unsigned long long* counts, void* stream);
int scv_sort_f64(scv_ctx* ctx, long long n, double* keys, double* alt, int* in_alt, void* stream);
int scv_gini_sums(scv_ctx* ctx, long long n, const double* sorted, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SCURVE_B200_H */
