"""The C-ABI multi-GPU z-slab path (aprgpu_multi_*, csrc/multi.cu): the
volume cut into N slabs driven from ONE process with peer-to-peer halos and
interior/boundary overlap.  On one B200 the slabs are virtual (all on device
0; the halo copies are device copies), which exercises the plan, the halo
ranges, the band split and the output assembly exactly as N GPUs would.
Every output must be bit-identical to the single-domain convolve_apr (EXACT)."""
import numpy as np
import pytest

import goldens as G
import paper_2112_03592_b200 as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["spheres64", "c1_256", "random_apr_03", "blobs32_1"])
@pytest.mark.parametrize("n_slabs", [1, 2, 3, 4])
def test_multi_slabs_bit_identical(name, n_slabs):
    d = G.load(name)
    apr = G.product_apr(d)
    a = apr.access
    rng = np.random.default_rng(n_slabs)
    v = rng.uniform(0, 100, a.particle_count()).astype(np.float32)
    tv = P.fill_tree(apr, v)
    try:
        m = P.MultiApr(apr, [0] * n_slabs, halo=2)
    except P.RangeError:
        pytest.skip(f"{name}: too thin for {n_slabs} slabs")
    for k in (3, 5):
        pyr = P.make_pyramid(P.gaussian_stencil(1.0, k), a.l_min, a.l_max, P.PyramidMode.Restricted)
        for pad in (P.PadMode.Reflect, P.PadMode.Zero):
            exp = P.convolve_apr(apr, v, tv, pyr, pad)
            got = m.convolve(v, tv, pyr, pad, "exact")
            assert np.array_equal(G.bits(got), G.bits(exp)), (k, pad, m.bounds)
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted)
    fast = m.convolve(v, tv, pyr, P.PadMode.Reflect, "fast")
    exp = P.convolve_apr(apr, v, tv, pyr, P.PadMode.Reflect, P.ConvolveOptions(accum="fast"))
    assert np.array_equal(G.bits(fast), G.bits(exp))


def test_multi_c3_eight_slabs():
    """C3 cut into 8 slabs (the 8-GPU layout), all on one device."""
    from paper_2112_03592_b200 import synth
    apr, v = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
    tv = P.fill_tree(apr, v)
    a = apr.access
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted)
    exp = P.convolve_apr(apr, v, tv, pyr)
    m = P.MultiApr(apr, [0] * 8, halo=2)
    assert len(m.bounds) == 8 and m.bounds[-1][1] == 1024
    got = m.convolve(v, tv, pyr)
    assert np.array_equal(G.bits(got), G.bits(exp))


def test_multi_rejects_halo_below_half_width():
    d = G.load("spheres64")
    apr = G.product_apr(d)
    a = apr.access
    m = P.MultiApr(apr, [0, 0], halo=1)
    v = np.ones(a.particle_count(), np.float32)
    tv = P.fill_tree(apr, v)
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 5), a.l_min, a.l_max, P.PyramidMode.Rescaled)
    with pytest.raises(P.RangeError):
        m.convolve(v, tv, pyr)
