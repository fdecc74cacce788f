"""The gather maps' bank-aware placement pass (k_map_place, conv_tile.cu) only
moves staged values within shared memory and drops chunks no active block
reads: results must equal the unplaced maps' bit for bit.  The switches are
read once per process (APRGPU_MAP_PLACE, APRGPU_MAP_DROP), so each setting
runs in its own subprocess on the same inputs (3^3 and 5^3, both modes, both
pads, C1 and a random APR)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [{root!r}, {tests!r}, {oracle!r}]
import goldens as G
import paper_2112_03592_b200 as P
outs = []
for name in ("c1_256", "random_apr_02"):
    d = G.load(name)
    apr = G.product_apr(d)
    a = apr.access
    tv = P.fill_tree(apr, d["values"])
    for k in (3, 5):
        pyr = P.make_pyramid(P.gaussian_stencil(1.0, k), a.l_min, a.l_max, P.PyramidMode.Restricted)
        for pad in (P.PadMode.Reflect, P.PadMode.Zero):
            for acc in ("exact", "fast"):
                outs.append(P.convolve_apr(apr, d["values"], tv, pyr, pad, P.ConvolveOptions(accum=acc)))
np.save(sys.argv[1], np.concatenate(outs).view(np.uint32))
"""


def _run(tmp_path, tag, env):
    path = str(tmp_path / f"{tag}.npy")
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), oracle=os.path.join(ROOT, "oracle"))
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", code, path], env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(path)


def test_placement_and_drops_change_nothing(tmp_path):
    base = _run(tmp_path, "off", {"APRGPU_MAP_PLACE": "0"})
    placed = _run(tmp_path, "placed", {"APRGPU_MAP_PLACE": "1", "APRGPU_MAP_DROP": "0"})
    dropped = _run(tmp_path, "dropped", {"APRGPU_MAP_PLACE": "1", "APRGPU_MAP_DROP": "1"})
    assert np.array_equal(base, placed)
    assert np.array_equal(base, dropped)
