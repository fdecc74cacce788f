"""Workload for compute-sanitizer (tests/test_sanitizer_gpu.py): the C1
fixture through every hot-path kernel -- upload (tree build, row/tile lists),
fill_tree, convolve_apr 3^3 and 5^3 in both accumulation modes (gather-map
build + map kernel, and the reconstruction kernel), the generic-extent kernel,
rl_apr, the pipelined host call -- small enough for racecheck."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import goldens as G  # noqa: E402
import paper_2112_03592_b200 as P  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
d = G.load("c1_256" if which != "small" else "spheres64")
apr = G.product_apr(d)
v = np.asarray(d["values"], np.float32)
tv = P.fill_tree(apr, v)
a = apr.access
for k in (3, 5):
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, k), a.l_min, a.l_max, P.PyramidMode.Restricted)
    for acc in ("exact", "fast"):
        P.convolve_apr(apr, v, tv, pyr, P.PadMode.Reflect, P.ConvolveOptions(accum=acc))
        P.convolve_apr(apr, v, tv, pyr, P.PadMode.Zero, P.ConvolveOptions(accum=acc))
os.environ["APRGPU_TILE_MAP"] = "0"  # the reconstruction kernel
pyr3 = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted)
P.convolve_apr(apr, v, tv, pyr3)
os.environ.pop("APRGPU_TILE_MAP")
w7 = P.gaussian_stencil(1.0, 7)  # generic-extent kernel
P.convolve_apr(apr, v, tv, P.make_pyramid(w7, a.l_min, a.l_max, P.PyramidMode.Rescaled))
P.rl_apr(apr, v, P.RLConfig(iterations=2, psf=P.gaussian_stencil(1.0, 3)))
print("sanitize workload done")
