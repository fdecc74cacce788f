"""GPU tests of the device APR builder (input side of the hot path) against the
reference: generate_spheres volume, build_apr structure and sampled values."""
import numpy as np
import pytest

import goldens as G
import paper_2112_03592_b200 as P
from paper_2112_03592_b200 import synth
from pyoracle import Oracle, Ref, ref_available

pytestmark = pytest.mark.gpu


def test_build_c1_matches_reference_golden():
    # BASELINE.md C1 built on the device == the reference build committed in c1_256.npz
    d = G.load("c1_256")
    apr, vals = synth.build_spheres_apr(256, count=12, rmin=6.0, rmax=20.0, blur=2.0, seed=42, rel_error=0.1)
    ref = G.product_apr(d)
    assert apr.access.equals(ref.access)
    assert apr.tree_access.equals(ref.tree_access)
    assert np.array_equal(G.bits(vals), G.bits(d["values"]))


def test_build_spheres64_matches_reference_golden():
    d = G.load("spheres64")
    apr, vals = synth.build_spheres_apr(64, count=10, rmin=3.0, rmax=10.0, blur=1.5, seed=5500, rel_error=0.1)
    ref = G.product_apr(d)
    assert apr.access.equals(ref.access)
    assert apr.tree_access.equals(ref.tree_access)
    assert np.array_equal(G.bits(vals), G.bits(d["values"]))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not shipped")
def test_generate_and_build_vs_live_reference():
    R = Ref()
    for dims, count, blur, seed in (((40, 33, 57), 6, 1.0, 7), ((64, 64, 64), 9, 2.0, 11), ((17, 80, 23), 4, 0.0, 3)):
        v_ref = R.generate_spheres(dims, count, 3.0, 10.0, blur, 0.0, seed)
        v = synth.generate_spheres(*dims, count=count, min_radius=3.0, max_radius=10.0, blur_sigma=blur, seed=seed)
        assert np.array_equal(G.bits(v), G.bits(v_ref))
        ra = R.build_apr(v_ref, 0.1)
        apr, vals = synth.build_apr(v, 0.1)
        assert apr.access.equals(P.LinearAccess(**vars(ra.leaf)))
        assert apr.tree_access.equals(P.LinearAccess(**vars(ra.tree)))
        assert np.array_equal(G.bits(vals), G.bits(ra.values()))


def test_built_apr_convolves_like_oracle():
    apr, vals = synth.build_spheres_apr(96, count=7, rmin=4.0, rmax=14.0, blur=2.0, seed=99, rel_error=0.1)
    tv = P.fill_tree(apr, vals)
    O = Oracle()
    assert np.array_equal(G.bits(tv), G.bits(O.fill_tree(apr.access, apr.tree_access, apr.source_dims, vals)))
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 5), apr.access.l_min, apr.access.l_max, P.PyramidMode.Restricted)
    out = P.convolve_apr(apr, vals, tv, pyr)
    levels = [((s.kz, s.kx, s.ky), s.weights) for s in pyr.stencils]
    exp = O.convolve(apr.access, apr.tree_access, vals, tv, levels, apr.access.l_min, 1)
    assert np.array_equal(G.bits(out), G.bits(exp))
