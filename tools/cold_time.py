"""Cold first-call timing (fresh handles): upload, first fill_tree, first
convolve_apr (tree links, tile probe/runs, gather maps + placement).  Needs a GPU:
python tools/cold_time.py [c1|c3] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if cfg == "c1":
    import goldens as G
    d = G.load("c1_256")
    apr, values = G.product_apr(d), d["values"]
else:
    from paper_2112_03592_b200 import synth
    apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
ctx = P.default_context(0)
a = apr.access
dpyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted).device(ctx)
st = torch.cuda.Stream()
s = st.cuda_stream
v = torch.from_numpy(np.ascontiguousarray(values, np.float32)).cuda()
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fresh = P.aprkit.DeviceApr.upload(ctx, P.APR(apr.access, apr.tree_access, apr.source_dims))
    t1 = time.perf_counter()
    tv = torch.empty(max(fresh.n_tree, 1), dtype=torch.float32, device="cuda")
    out = torch.empty(fresh.n_particles, dtype=torch.float32, device="cuda")
    fresh.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
    st.synchronize()
    t2 = time.perf_counter()
    fresh.convolve_ptr(v.data_ptr(), tv.data_ptr(), dpyr, 1, L.ACCUM_EXACT, out.data_ptr(), s)
    st.synchronize()
    t3 = time.perf_counter()
    fresh.convolve_ptr(v.data_ptr(), tv.data_ptr(), dpyr, 1, L.ACCUM_EXACT, out.data_ptr(), s)
    st.synchronize()
    t4 = time.perf_counter()
    print(cfg, "upload %.1f fill %.1f first_conv %.1f second_conv %.2f ms" % (
        (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3), flush=True)
    del fresh, tv, out
