"""Per-rank setup with and without aprgpu_apr_restrict on C3: one z-slab of N
(as slab.py would give rank 0), the first convolution's wall time (tile
probe, source runs, staged lists, gather maps, then the pass) and the map
records held."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import _lib as L  # noqa: E402
from paper_2112_03592_b200 import synth  # noqa: E402
from paper_2112_03592_b200.slab import SlabPlan  # noqa: E402

apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
a = apr.access
ctx = P.default_context()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
s = stream.cuda_stream
pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted).device(ctx)
v = torch.from_numpy(np.ascontiguousarray(values, np.float32)).cuda()
for world in (1, 2, 4, 8):
    plan = SlabPlan.make(a, apr.tree_access, apr.source_dims, world, 0, halo=2)
    z_lo, z_hi = plan.bounds[0]
    dev = P.DeviceApr.upload(ctx, apr)
    if world > 1:
        dev.restrict(plan.lc, z_lo, z_hi)
    tv = torch.empty(max(dev.n_tree, 1), dtype=torch.float32, device="cuda")
    out = torch.empty(dev.n_particles, dtype=torch.float32, device="cuda")
    dev.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.check(L.lib().aprgpu_convolve_slab_band(dev.handle, v.data_ptr(), tv.data_ptr(), pyr.handle, 1, L.ACCUM_EXACT,
                                              plan.lc if world > 1 else 1 << 20, z_lo, z_hi, 1, out.data_ptr(), s))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    built, n_tiles = dev.map_tiles()
    print(f"world {world}: rank-0 slab planes [{z_lo}, {z_hi}), first slab convolution {1e3 * (t1 - t0):.1f} ms, "
          f"map records {built} of {n_tiles} tiles", flush=True)
    del dev
