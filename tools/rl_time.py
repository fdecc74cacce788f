"""rl_apr on C3 (3^3 PSF, FAST): wall time of iterations = 1, 2, 10, 20 (device
pointers, warm) -> setup vs per-iteration cost."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import synth  # noqa: E402

apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
dev = apr.device()
v = torch.from_numpy(values).cuda()
out = torch.empty_like(v)
s = torch.cuda.Stream()
w = P.gaussian_stencil(1.0, 3)
for it in (1, 1, 2, 2, 10, 10, 20, 20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.rl_ptr(v.data_ptr(), w, it, 0.0, 1, out.data_ptr(), s.cuda_stream)
    s.synchronize()
    print(it, round((time.perf_counter() - t0) * 1e3, 3), "ms")
