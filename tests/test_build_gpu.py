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


PARAMS = [  # (sigma_mode, sigma_value, sigma_window, sigma_floor, gradient_mode, smoothing_passes)
    (0, 250.0, 2, 0.0, 1, 0),    # Sobel
    (0, 250.0, 2, 0.0, 0, 2),    # two box passes on the gradient
    (1, 1.0, 2, 0.0, 0, 0),      # local range sigma, default floor
    (1, 1.0, 1, 5.0, 1, 1),      # local range r=1, explicit floor, Sobel, one pass
    (0, 1e-9, 2, 40.0, 0, 0),    # constant below the floor
]


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("params", PARAMS)
@pytest.mark.parametrize("dims,seed", [((40, 33, 57), 3), ((64, 64, 64), 11), ((9, 17, 6), 5)])
def test_build_apr_params_vs_live_reference(params, dims, seed):
    """build_apr with every BuildParams option (build.hpp:290-312): Sobel,
    smoothing passes, local-range sigma with its box pass and floor -- structure
    and sampled values bit-identical to the unmodified reference."""
    sm, sv, sw, sf, gm, sp = params
    R = Ref()
    vol = R.generate_spheres(dims, 5, 2.0, 8.0, 1.5, 20.0, seed)  # with noise: gradients everywhere
    r = R.build_apr_params(vol, 0.1, sm, sv, sw, sf, gm, sp)
    apr, vals = synth.build_apr_params(vol, P.aprkit.BuildParams(0.1, sm, sv, sw, sf, gm, sp))
    ra = r.leaf
    for f in ("y_idx", "xz_end"):
        assert np.array_equal(getattr(apr.access, f), getattr(ra, f)), f
    assert np.array_equal(apr.access.level_offset[ra.l_min:], ra.level_offset[ra.l_min:])
    assert np.array_equal(apr.tree_access.y_idx, r.tree.y_idx)
    assert np.array_equal(G.bits(vals), G.bits(r.values()))
