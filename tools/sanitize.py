"""Small analysis + synthesis round trips for compute-sanitizer (memcheck / racecheck):
complex spin 2 and real paths, slabs and the streamed round trip, on the prime-factor
lengths (L = 64, 128: K = 127 cuFFT fallback, 255 engine)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1511_05578_b200 as sc
from bench import gaussian_flm
torch.cuda.set_device(0)
for L, s, J0 in [(64, 2, 2), (128, 0, 2), (256, 0, 6)]:
    t = sc.build_tiling(sc.TilingParams(L, s, 2.0, J0))
    f = sc.sht_inverse(sc.HarmonicCoeffs(L, s, gaussian_flm(L, s, 0, s == 0)))
    g = sc.synthesize(sc.analyze(f, t), t)
    e = float((g.values - f.values).abs().max() / f.values.abs().max())
    g2 = sc.roundtrip_streamed(f, t, slab_bytes=1 << 20)
    e2 = float((g2.values - f.values).abs().max() / f.values.abs().max())
    msg = f"L={L} s={s}: round trip {e:.2e}, streamed {e2:.2e}"
    if s == 0:
        fr = sc.SphereSignal(f.grid, 0, f.values.real.contiguous(), real=True)
        gr = sc.synthesize_real(sc.analyze_real(fr, t), t)
        msg += f", real {float((gr.values - fr.values).abs().max() / fr.values.abs().max()):.2e}"
    print(msg, flush=True)
# the K = 2047 kernels (blocked column generation, grouped row kernels, gamma +
# quadrature) on a 2-row beta slab of an L_j = 1024 scale
L = 1024
rng = np.random.default_rng(1)
w = np.zeros((2, L, 2 * L - 1), complex)
for l in range(L):
    w[:, l, L - 1 - l:L + l] = rng.standard_normal((2, 2 * l + 1)) + 1j * rng.standard_normal((2, 2 * l + 1))
cw = sc.CurveletWignerCoeffs(L, torch.as_tensor(w, device="cuda"))
slab = sc.so3_inverse_curvelet_slab(cw, sc.SO3Grid(L, L, L), 500, 2)
part = sc.so3_forward_curvelet_slab(slab)
torch.cuda.synchronize()
print("L=1024 slab ok", float(part.values.abs().max()))
print("sanitize workload done")
