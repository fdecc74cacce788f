"""rl_apr on C4 (the C3 APR tiled 4x4x2 on the device): wall time of
iterations = 1, 2, 10 (device pointers, warm) next to one fill_tree and one
convolve_apr -> where an RL iteration's time goes.  Needs a GPU."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import _lib as L  # noqa: E402
from paper_2112_03592_b200 import synth  # noqa: E402

apr3, values3 = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
d3 = apr3.device()
dapr = synth.tile_apr(d3, 4, 4, 2)
v3 = torch.from_numpy(np.ascontiguousarray(values3, np.float32)).cuda()
v = torch.empty(dapr.n_particles, dtype=torch.float32, device="cuda")
synth.tile_values(d3, dapr, 4, 4, 2, v3.data_ptr(), v.data_ptr())
li = dapr.info(L.LEAF)
out = torch.empty_like(v)
tv = torch.empty(max(dapr.n_tree, 1), dtype=torch.float32, device="cuda")
st = torch.cuda.Stream()
s = st.cuda_stream
w = P.gaussian_stencil(1.0, 3)


def timed(f, n=3):
    r = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        st.synchronize()
        r.append((time.perf_counter() - t0) * 1e3)
    return [round(x, 2) for x in r]


t0 = time.perf_counter()
pyr = P.make_pyramid(w, int(li.l_min), int(li.l_max), P.PyramidMode.Restricted)
print("levels", li.l_min, li.l_max, "make_pyramid ms", round((time.perf_counter() - t0) * 1e3, 1), flush=True)
dp = pyr.device()
print("fill_tree ms", timed(lambda: dapr.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)), flush=True)
print("convolve ms", timed(lambda: dapr.convolve_ptr(v.data_ptr(), tv.data_ptr(), dp, 1, L.ACCUM_EXACT,
                                                     out.data_ptr(), s)), flush=True)
for it in (1, 2, 10):
    print("rl", it, "ms", timed(lambda: dapr.rl_ptr(v.data_ptr(), w, it, 0.0, L.ACCUM_EXACT, out.data_ptr(), s), 2),
          flush=True)
os.environ["APRGPU_RL_GRAPH"] = "0"
print("rl 10 eager ms", timed(lambda: dapr.rl_ptr(v.data_ptr(), w, 10, 0.0, L.ACCUM_EXACT, out.data_ptr(), s), 2),
      flush=True)
