import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_05578_b200 import _cabi
ctx = _cabi.context(0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 2047
n = (1 << 27) // (K * 16)
x = torch.randn(n, K, dtype=torch.complex128, device="cuda"); y = torch.empty_like(x)
for _ in range(3):
    ctx.call("debug_dft", K, -1, n, _cabi.ptr(x), _cabi.ptr(y))
torch.cuda.synchronize()
print("ok")
