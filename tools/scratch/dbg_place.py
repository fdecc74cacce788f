import os, sys
sys.path[:0] = ["/root/repo", "/root/repo/tests", "/root/repo/oracle"]
import numpy as np
import goldens as G
import paper_2112_03592_b200 as P
from test_parity_gpu import golden_pyramid
name = sys.argv[1] if len(sys.argv) > 1 else "random_apr_01"
d = G.load(name)
apr = G.product_apr(d)
print("dims", apr.access.l_min, apr.access.l_max, [int(x) for x in apr.access.y_dim])
for c in G.conv_names(d):
    pyr = golden_pyramid(d, c)
    pad = P.PadMode(int(d[f"conv_{c}_pad"][0]))
    out = P.convolve_apr(apr, d["values"], d["tree_values"], pyr, pad)
    ref = d[f"conv_{c}_out"]
    bad = np.nonzero(G.bits(out) != G.bits(ref))[0]
    print(c, pad, [ (s.kz, s.kx, s.ky) for s in pyr.stencils][:3], "mismatch", len(bad), bad[:10])
