"""Host-side cost of one convolve call (device pointers, no sync) on C3, and the
pipelined host-pointer call's wall time for several chunk counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import _lib as L  # noqa: E402
from paper_2112_03592_b200 import synth  # noqa: E402

apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
dev = apr.device()
tree = P.fill_tree(apr, values)
pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), apr.access.l_min, apr.access.l_max, P.PyramidMode.Restricted)
dpyr = pyr.device(dev.ctx)
v = torch.from_numpy(values).cuda()
t = torch.from_numpy(tree).cuda()
o = torch.empty_like(v)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    dev.convolve_ptr(v.data_ptr(), t.data_ptr(), dpyr, 1, L.ACCUM_FAST, o.data_ptr(), s)
torch.cuda.synchronize()
a = time.perf_counter()
for _ in range(50):
    dev.convolve_ptr(v.data_ptr(), t.data_ptr(), dpyr, 1, L.ACCUM_FAST, o.data_ptr(), s)
b = time.perf_counter()
torch.cuda.synchronize()
c = time.perf_counter()
print("host us per device call", round((b - a) / 50 * 1e6, 1), " gpu+host us per call", round((c - a) / 50 * 1e6, 1))
hv = torch.from_numpy(values).pin_memory()
ht = torch.from_numpy(tree).pin_memory()
ho = torch.empty_like(hv).pin_memory()
for ch in ("1", "2", "4", "8", "16"):
    os.environ["APRGPU_HOST_CHUNKS"] = ch
    ts = []
    for i in range(8):
        a = time.perf_counter()
        L.check(L.lib().aprgpu_convolve(dev.handle, hv.data_ptr(), ht.data_ptr(), dpyr.handle, 1, L.ACCUM_FAST,
                                        ho.data_ptr(), L.HOST, None))
        ts.append(time.perf_counter() - a)
    print("chunks", ch, "ms", round(1e3 * float(np.median(ts[2:])), 3))
