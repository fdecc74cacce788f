"""One warm C3 convolution pass for ncu captures: builds C3 on the device,
fills the tree, runs two warm-up passes (gather maps built), flushes L2, then
one pass.  Launches of k_conv_map per pass: 1 for a 3^3 pyramid, 2 for 5^3
(the restricted 3^3 levels + the 5^3 finest level) -- so capture with
  ncu -k regex:k_conv_map -s <2*per_pass> -c <per_pass> ... python tools/one_pass.py <k> <exact|fast>"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import _lib as L  # noqa: E402
from paper_2112_03592_b200 import synth  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
acc = L.ACCUM_EXACT if (sys.argv[2] if len(sys.argv) > 2 else "exact") == "exact" else L.ACCUM_FAST
apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
s = stream.cuda_stream
dapr = apr.device()
a = apr.access
pyr = P.make_pyramid(P.gaussian_stencil(1.0, k), a.l_min, a.l_max, P.PyramidMode.Restricted).device()
v = torch.from_numpy(np.ascontiguousarray(values, np.float32)).cuda()
tv = torch.empty(max(dapr.n_tree, 1), dtype=torch.float32, device="cuda")
out = torch.empty_like(v)
dapr.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for i in range(3):
    flush.zero_()
    dapr.convolve_ptr(v.data_ptr(), tv.data_ptr(), pyr, 1, acc, out.data_ptr(), s)
torch.cuda.synchronize()
print("one_pass done")
