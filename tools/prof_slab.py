"""Full-size (L=1024) kernels on a beta slab, for ncu: one slab analysis
(k_ana_colgen + k_pfa_rows) and one slab synthesis (k_syn_alpha +
k_syn_gamma_q) over `nb` beta rows.  usage: prof_slab.py [L] [nb]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1511_05578_b200 as sc

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 16
rng = np.random.default_rng(0)
w = (rng.standard_normal((2, L, 2 * L - 1)) + 1j * rng.standard_normal((2, L, 2 * L - 1)))
cw = sc.CurveletWignerCoeffs(L, w)
grid = sc.SO3Grid(L, L, L)
b0 = L // 2 - nb // 2
for _ in range(2):
    slab = sc.so3_inverse_curvelet_slab(cw, grid, b0, nb)
    part = sc.so3_forward_curvelet_slab(slab)
torch.cuda.synchronize()
print("ok", float(part.values.abs().max()))
