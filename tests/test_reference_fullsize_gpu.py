"""Parity at BASELINE's large configurations against the reference itself.

The unmodified reference (oracle/_ref/libaprref.so, compiled from
/root/reference's own headers; it travels to the GPU box) is run on the SAME
APR as the CUDA path, and the outputs are compared the way the reference's
acceptance criterion 3 does (proj/tests/acceptance.cpp:246-295):

  * C3 (1024^3 spheres, 17.1 M particles): the interior structure and
    fill_tree bit-identical; convolve_apr 3^3 and 5^3 EXACT bit-identical,
    FAST within max_rel_diff <= 1e-5 (scale max(|e|, |g|, 1)).  The 3^3
    pyramid is the reference's own make_pyramid; for 5^3 the repo's restricted
    levels are first checked against the reference's restrict_stencil wherever
    its O(8^delta k^3) loop is affordable, then handed to the reference as an
    explicit pyramid.
  * C5 (rl_apr x 10 on C3, Gaussian 3^3 PSF): bit-identical to the reference's
    rl_apr (which builds both pyramids itself).
  * C4 (the C3 APR tiled 4 x 4 x 2, 548 M particles): the device-tiled
    interior structure equals the reference's init_tree_structure, fill_tree
    and the whole 3^3 EXACT output bit-identical.
"""
import numpy as np
import pytest

import paper_2112_03592_b200 as P
from paper_2112_03592_b200 import _lib as L
from pyoracle import Ref, as_access, ref_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0))) if a.size else 0.0


def same_access(a, b):
    a, b = as_access(a), as_access(b)
    assert (a.l_min, a.l_max) == (b.l_min, b.l_max)
    assert np.array_equal(a.y_idx, b.y_idx)
    assert np.array_equal(a.xz_end, b.xz_end)
    assert np.array_equal(a.level_offset[a.l_min:], b.level_offset[b.l_min:])
    for f in ("z_dim", "x_dim", "y_dim"):
        assert np.array_equal(getattr(a, f)[a.l_min:], getattr(b, f)[b.l_min:]), f


@pytest.fixture(scope="module")
def c3():
    from paper_2112_03592_b200 import synth
    apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
    R = Ref()
    rapr = R.apr_from_arrays(apr.access, apr.source_dims)  # the reference's init_tree_structure
    tv = P.fill_tree(apr, values)
    tvr = R.fill_tree(rapr, values)
    return apr, values, tv, R, rapr, tvr


def test_c3_interior_structure_and_fill_tree(c3):
    apr, values, tv, R, rapr, tvr = c3
    assert apr.access.particle_count() == 17111578
    same_access(apr.tree_access, rapr.tree)  # device-built tree == init_tree_structure
    assert np.array_equal(bits(tv), bits(tvr))
    # nonempty_row_index (convolve.hpp:32-44), every level
    d = apr.device()
    for lv in range(apr.access.l_min, apr.access.l_max + 1):
        exp = R.nonempty_rows(rapr, lv)
        got = d.row_index(lv)
        for e, g in zip(exp, got):
            assert np.array_equal(np.asarray(e).astype(np.int64), np.asarray(g).astype(np.int64)), lv


def test_c3_k3_vs_reference(c3):
    apr, values, tv, R, rapr, tvr = c3
    a = apr.access
    k3, w = R.gaussian_stencil(1.0, 3)
    rpyr = R.make_pyramid(w, k3, a.l_min, a.l_max, 0)  # the reference's own restriction
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted)
    for s, (rk, rw) in zip(pyr.stencils, rpyr.levels()):
        assert (s.kz, s.kx, s.ky) == tuple(rk)
        assert np.array_equal(bits(s.weights), bits(rw))
    ref = R.convolve(rapr, values, tvr, rpyr, 1)
    got = P.convolve_apr(apr, values, tv, pyr)
    assert np.array_equal(bits(got), bits(ref))
    fast = P.convolve_apr(apr, values, tv, pyr, P.PadMode.Reflect, P.ConvolveOptions(accum="fast"))
    assert rel(fast, ref) <= 1e-5


def _checked_levels(R, w, k, l_min, l_max):
    """The repo's restricted pyramid, each level checked against the reference's
    restrict_stencil where its loop is affordable (8^delta k^3 <= ~4e9)."""
    pyr = P.make_pyramid(P.Stencil(k, k, k, weights=w), l_min, l_max, P.PyramidMode.Restricted)
    checked = 0
    for l, s in zip(range(l_min, l_max + 1), pyr.stencils):
        delta = l_max - l
        if (8 ** delta) * k ** 3 > 4e9:
            continue
        rk, rw = R.restrict_stencil(w, (k, k, k), delta)
        assert (s.kz, s.kx, s.ky) == tuple(rk), delta
        assert np.array_equal(bits(s.weights), bits(rw)), delta
        checked += 1
    # delta <= 9 at 3^3 and <= 8 at 5^3: every level of C3; at C4 (l_max 12) the
    # two coarsest levels (delta 10, 11) rely on the closed form alone (pinned
    # against the reference loop up to delta 6 for k <= 13, tests/test_library.py)
    assert checked >= min(l_max - l_min + 1, 9)
    return pyr


def test_c3_k5_vs_reference(c3):
    apr, values, tv, R, rapr, tvr = c3
    a = apr.access
    k5, w = R.gaussian_stencil(1.0, 5)
    pyr = _checked_levels(R, w, 5, a.l_min, a.l_max)
    rpyr = R.explicit_pyramid([((s.kz, s.kx, s.ky), s.weights) for s in pyr.stencils], a.l_min)
    ref = R.convolve(rapr, values, tvr, rpyr, 1)
    got = P.convolve_apr(apr, values, tv, pyr)
    assert np.array_equal(bits(got), bits(ref))
    fast = P.convolve_apr(apr, values, tv, pyr, P.PadMode.Reflect, P.ConvolveOptions(accum="fast"))
    assert rel(fast, ref) <= 1e-5


def test_c5_rl_apr_vs_reference(c3):
    apr, values, tv, R, rapr, tvr = c3
    k3, w = R.gaussian_stencil(1.0, 3)
    ref = R.rl_apr(rapr, values, w, k3, 10)
    got = P.rl_apr(apr, values, P.RLConfig(iterations=10, psf=P.Stencil(3, 3, 3, weights=w)))
    assert np.array_equal(bits(got), bits(ref))


def test_c4_vs_reference(c3):
    """The whole C4 EXACT output (548 M particles) against the reference."""
    import torch
    from paper_2112_03592_b200 import synth
    apr, values, tv, R, rapr, tvr = c3
    d3 = apr.device()
    big = synth.tile_apr(d3, 4, 4, 2)
    v3 = torch.from_numpy(np.ascontiguousarray(values, np.float32)).cuda()
    bv = torch.empty(big.n_particles, dtype=torch.float32, device="cuda")
    synth.tile_values(d3, big, 4, 4, 2, v3.data_ptr(), bv.data_ptr())
    torch.cuda.synchronize()
    del v3
    leaf = big.download(L.LEAF)
    assert leaf.particle_count() == 547570496
    big_values = bv.cpu().numpy()
    rbig = R.apr_from_arrays(leaf, tuple(big.dims))  # the reference's init_tree_structure (C4: ~20 s)
    same_access(big.download(L.TREE), rbig.tree)
    btv = torch.empty(big.n_tree, dtype=torch.float32, device="cuda")
    big.fill_tree_ptr(bv.data_ptr(), btv.data_ptr(), 0)
    torch.cuda.synchronize()
    rtv = R.fill_tree(rbig, big_values)
    assert np.array_equal(bits(btv.cpu().numpy()), bits(rtv))
    # explicit pyramid of the repo's restricted levels (the reference's own
    # make_pyramid at l_max = 12 would take ~30 min; levels checked as above)
    k3, w = R.gaussian_stencil(1.0, 3)
    pyr = _checked_levels(R, w, 3, leaf.l_min, leaf.l_max)
    rpyr = R.explicit_pyramid([((s.kz, s.kx, s.ky), s.weights) for s in pyr.stencils], leaf.l_min)
    ref = R.convolve(rbig, big_values, rtv, rpyr, 1)
    del rbig
    out = torch.empty_like(bv)
    big.convolve_ptr(bv.data_ptr(), btv.data_ptr(), pyr.device(big.ctx), 1, L.ACCUM_EXACT, out.data_ptr(), 0)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.array_equal(bits(got), bits(ref))
