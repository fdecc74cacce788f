"""NVTX ranges: every compute entry point of the C-ABI opens a range named
after it (internal.cuh NvtxRange / guard(name, ...)), so a profiler can scope
to one.  ncu --nvtx-include "aprgpu_convolve/" on a small convolution must
profile the tile kernel and nothing from fill_tree, which runs outside it."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys; sys.path[:0] = [sys.argv[1], sys.argv[1] + '/tests']
import goldens as G, paper_2112_03592_b200 as P
d = G.load('spheres64'); apr = G.product_apr(d); a = apr.access
tv = P.fill_tree(apr, d['values'])
pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted)
P.convolve_apr(apr, d['values'], tv, pyr)
print('done')
"""


@pytest.mark.skipif(shutil.which("ncu") is None, reason="ncu not on PATH")
def test_nvtx_range_scopes_the_convolution(tmp_path):
    log = tmp_path / "k.csv"
    r = subprocess.run(["ncu", "--nvtx", "--nvtx-include", "aprgpu_convolve/", "--metrics", "gpu__time_duration.sum",
                        "--csv", "--log-file", str(log), sys.executable, "-c", SCRIPT, ROOT],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "done" in r.stdout, r.stderr[-2000:]
    text = log.read_text()
    assert "k_conv" in text, text[-2000:]
    assert "k_fill_tree" not in text
