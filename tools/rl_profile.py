"""Two rl_apr calls of one iteration on C3 (for ncu: the second call's two
convolutions -- ratio epilogue, then multiply epilogue)."""
import os
import sys

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
for _ in range(2):
    dev.rl_ptr(v.data_ptr(), w, 1, 0.0, 1, out.data_ptr(), s.cuda_stream)
    s.synchronize()
print("ok")
