"""One dense pixel convolution of a 1024^3 volume (for ncu): warm-up, then one pass."""
import sys
import torch
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import _lib as L  # noqa: E402
acc = L.ACCUM_EXACT if (sys.argv[1] if len(sys.argv) > 1 else "exact") == "exact" else L.ACCUM_FAST
ctx = P.default_context()
x = torch.rand(1024 ** 3, device="cuda")
y = torch.empty_like(x)
w = P.gaussian_stencil(1.0, 3)
for _ in range(2):
    P.convolve_pixels_ptr(ctx, x.data_ptr(), (1024, 1024, 1024), w, 1, acc, y.data_ptr(), 0)
torch.cuda.synchronize()
