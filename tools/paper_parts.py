"""Times the parts of the paper protocol step on C3, each with
L2 flushed before it: the index rebuild, fill_tree, the conv pass."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import _lib as L  # noqa: E402
from paper_2112_03592_b200 import synth  # noqa: E402

apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
s = stream.cuda_stream
d = apr.device()
a = apr.access
pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted).device()
v = torch.from_numpy(np.ascontiguousarray(values, np.float32)).cuda()
tv = torch.empty(max(d.n_tree, 1), dtype=torch.float32, device="cuda")
out = torch.empty_like(v)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
parts = {"rebuild_index": lambda: d.rebuild_index_ptr(s),
         "fill_tree": lambda: d.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s),
         "conv": lambda: d.convolve_ptr(v.data_ptr(), tv.data_ptr(), pyr, 1, L.ACCUM_EXACT, out.data_ptr(), s)}
for f in parts.values():
    f()
for name, f in parts.items():
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name:14s} {np.median(ts) * 1e3:8.1f} us (median of 20, L2 flushed)")
