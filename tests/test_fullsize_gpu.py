"""Parity at BASELINE.json's full sizes (C3: 1024^3 spheres -> 17.1 M particles,
built on the device; C4: C3 tiled 4 x 4 x 2): the whole C3 output against the
C oracle bit for bit,
and size-independent properties -- the device validator on the built
structure, constant fields through fill_tree and convolve_apr, linearity, and
the two independent tile paths (resident gather maps vs per-call
reconstruction) agreeing bit for bit.
"""
import numpy as np
import pytest

import goldens as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    from paper_2112_03592_b200 import synth
    apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
    return apr, values


def test_c3_structure_is_a_valid_apr(c3):
    import paper_2112_03592_b200 as P
    apr, values = c3
    assert apr.access.particle_count() == values.size > 17_000_000
    assert P.validate(apr).ok  # O(particles) partition proof of the whole C3 structure


def test_c3_constant_fields(c3):
    import paper_2112_03592_b200 as P
    apr, _ = c3
    one = np.full(apr.access.particle_count(), 1.5, np.float32)
    tv = P.fill_tree(apr, one)
    assert np.all(tv == np.float32(1.5))  # footprint-weighted mean of a constant, exactly
    w = P.box_stencil(3)
    pyr = P.make_pyramid(w, apr.access.l_min, apr.access.l_max, P.PyramidMode.Restricted)
    out = P.convolve_apr(apr, one, tv, pyr, P.PadMode.Reflect)  # EXACT
    # every output of level l is 1.5 x sum of level l's weights, in the reference's fp64 order
    a = apr.access
    ends = np.asarray(a.xz_end, np.int64)
    for i, l in enumerate(range(a.l_min, a.l_max + 1)):
        r0 = int(a.level_offset[l])
        n_rows = int(a.z_dim[l]) * int(a.x_dim[l])
        b = int(ends[r0 - 1]) if r0 else 0
        e = int(ends[r0 + n_rows - 1]) if n_rows else b
        if e == b:
            continue
        s = 0.0
        for wv in pyr.at(l).weights.astype(np.float32):
            s += float(wv) * 1.5
        assert np.all(out[b:e] == np.float32(s)), l


def test_c3_linearity_and_paths_agree(c3, monkeypatch):
    import paper_2112_03592_b200 as P
    apr, values = c3
    tv = P.fill_tree(apr, values)
    tv2 = P.fill_tree(apr, 2 * values)
    assert np.array_equal(tv2, 2 * tv)
    for k in (3, 5):
        pyr = P.make_pyramid(P.gaussian_stencil(1.0, k), apr.access.l_min, apr.access.l_max,
                             P.PyramidMode.Restricted)
        for accum in ("exact", "fast"):
            opt = P.ConvolveOptions(accum=accum)
            out = P.convolve_apr(apr, values, tv, pyr, P.PadMode.Reflect, opt)
            assert np.array_equal(P.convolve_apr(apr, 2 * values, tv2, pyr, P.PadMode.Reflect, opt), 2 * out)
            monkeypatch.setenv("APRGPU_TILE_MAP", "0")
            rec = P.convolve_apr(apr, values, tv, pyr, P.PadMode.Reflect, opt)
            monkeypatch.delenv("APRGPU_TILE_MAP")
            assert np.array_equal(G.bits(out), G.bits(rec)), (k, accum)


def test_c3_exact_convolution_equals_the_oracle(c3):
    import paper_2112_03592_b200 as P
    from pyoracle import Oracle
    apr, values = c3
    tv = P.fill_tree(apr, values)
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), apr.access.l_min, apr.access.l_max, P.PyramidMode.Restricted)
    out = P.convolve_apr(apr, values, tv, pyr, P.PadMode.Reflect)
    levels = [((s.kz, s.kx, s.ky), s.weights) for s in pyr.stencils]
    orc = Oracle()
    leaf, tree = G.as_oracle(apr.access), G.as_oracle(apr.tree_access)
    assert np.array_equal(G.bits(tv), G.bits(orc.fill_tree(leaf, tree, tuple(apr.source_dims), values)))
    exp = orc.convolve(leaf, tree, values, tv, levels, apr.access.l_min, 1)
    assert np.array_equal(G.bits(out), G.bits(exp))


def test_c4_paths_agree(c3, monkeypatch):
    """C4 (the C3 APR tiled 4 x 4 x 2 on the device, 548 M particles): the
    map and reconstruction paths agree bit for bit over the whole output."""
    import torch
    import paper_2112_03592_b200 as P
    from paper_2112_03592_b200 import _lib as L
    from paper_2112_03592_b200 import synth
    apr, values = c3
    ctx = P.default_context()
    d3 = apr.device(ctx)
    big = synth.tile_apr(d3, 4, 4, 2)
    assert big.n_particles == 32 * values.size
    v3 = torch.from_numpy(values).cuda()
    v = torch.empty(big.n_particles, dtype=torch.float32, device="cuda")
    synth.tile_values(d3, big, 4, 4, 2, v3.data_ptr(), v.data_ptr())
    tv = torch.empty(max(big.n_tree, 1), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    big.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
    li = big.info(L.LEAF)
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), int(li.l_min), int(li.l_max), P.PyramidMode.Restricted)
    dpyr = pyr.device(ctx)
    outs = []
    for path in ("1", "0"):
        monkeypatch.setenv("APRGPU_TILE_MAP", path)
        o = torch.empty_like(v)
        big.convolve_ptr(v.data_ptr(), tv.data_ptr(), dpyr, 1, L.ACCUM_FAST, o.data_ptr(), s)
        torch.cuda.synchronize()
        outs.append(o)
    assert torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32))
