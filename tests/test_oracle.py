"""CPU tests pinning the C oracle (oracle/aprk_oracle.c) to the reference.

(a) against the committed golden vectors produced by the real reference, and
(b) live against oracle/_ref/libaprref.so (the unmodified reference compiled
    where it lies) when that library is present.
All comparisons are bit-exact (the reference's own determinism tests demand it,
test_convolve.cpp:102-123, test_tree.cpp:87-96).
"""
import numpy as np
import pytest

import goldens as G
from pyoracle import Oracle, Ref, ref_available

ORC = Oracle()


@pytest.mark.parametrize("name", G.names("random_apr_*") + G.names("blobs32_*") + ["spheres64", "dense16"])
def test_oracle_tree_structure_matches_golden(name):
    d = G.load(name)
    t = ORC.init_tree_structure(G.oracle_access(d, "leaf_"), tuple(d["dims"]))
    g = G.oracle_access(d, "tree_")
    assert (t.l_min, t.l_max) == (g.l_min, g.l_max)
    assert np.array_equal(t.y_idx, g.y_idx)
    assert np.array_equal(t.xz_end, g.xz_end)
    assert np.array_equal(t.level_offset[t.l_min:], g.level_offset[g.l_min:])


@pytest.mark.parametrize("name", G.names("random_apr_*") + G.names("blobs32_*") + ["spheres64", "dense16"])
def test_oracle_fill_tree_matches_golden(name):
    d = G.load(name)
    tv = ORC.fill_tree(G.oracle_access(d, "leaf_"), G.oracle_access(d, "tree_"), tuple(d["dims"]), d["values"])
    assert np.array_equal(G.bits(tv), G.bits(d["tree_values"]))


@pytest.mark.parametrize("name", G.names("random_apr_*") + ["spheres64"])
def test_oracle_row_index_matches_golden(name):
    d = G.load(name)
    leaf = G.oracle_access(d, "leaf_")
    off = 0
    for i, l in enumerate(range(leaf.l_min, leaf.l_max + 1)):
        z, x, y0, y1 = ORC.nonempty_rows(leaf, l)
        n = int(d["rows_count"][i])
        assert z.size == n
        assert np.array_equal(z, d["rows_z"][off:off + n])
        assert np.array_equal(x, d["rows_x"][off:off + n])
        assert np.array_equal(y0, d["rows_ymin"][off:off + n])
        assert np.array_equal(y1, d["rows_ymax"][off:off + n])
        off += n


@pytest.mark.parametrize("name", G.names("random_apr_*") + G.names("blobs32_*") + ["spheres64", "dense16"])
def test_oracle_convolve_matches_golden(name):
    d = G.load(name)
    leaf, tree = G.oracle_access(d, "leaf_"), G.oracle_access(d, "tree_")
    for c in G.conv_names(d):
        levels = G.pyramid_levels(d, c)
        out = ORC.convolve(leaf, tree, d["values"], d["tree_values"], levels, leaf.l_min, int(d[f"conv_{c}_pad"][0]))
        assert np.array_equal(G.bits(out), G.bits(d[f"conv_{c}_out"])), c


def test_oracle_restrict_matches_golden():
    d = G.load("restrict")
    for i in range(int(d["n_cases"][0])):
        meta = d[f"c{i}_meta"]
        k3, delta, ok = tuple(meta[:3]), int(meta[3]), tuple(meta[4:7])
        got_k, got = ORC.restrict_stencil(d[f"c{i}_in"], k3, delta)
        assert got_k == ok
        assert np.array_equal(G.bits(got), G.bits(d[f"c{i}_out"])), (k3, delta)


def test_oracle_rl_matches_golden():
    d = G.load("rl_spheres64")
    leaf, tree = G.oracle_access(d, "leaf_"), G.oracle_access(d, "tree_")
    for k in (3, 5):
        out = ORC.rl_apr(leaf, tree, tuple(d["dims"]), d["values"], d[f"rl_g{k}_psf"], (k, k, k), 10)
        assert np.array_equal(G.bits(out), G.bits(d[f"rl_g{k}_out"])), k


def test_reflect_index_kats():
    # test_reconstruct.cpp:8-17
    for i, n, e in [(0, 5, 0), (4, 5, 4), (-1, 5, 0), (-2, 5, 1), (5, 5, 4), (6, 5, 3), (-7, 3, 0), (9, 3, 2)]:
        assert ORC.reflect_index(i, n) == e


def test_c1_golden_shape():
    # 278,769 particles, 39,824 interior nodes, CR 60.18
    d = G.load("c1_256")
    assert d["leaf_y_idx"].size == 278769
    assert d["tree_y_idx"].size == 39824
    assert abs(256 ** 3 / d["leaf_y_idx"].size - 60.18) < 0.01


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_vs_live_reference_random():
    R = Ref()
    rng = R.rng(4242)
    for trial in range(6):
        apr = R.random_apr(rng, 4, 36)
        leaf, tree, dims = apr.leaf, apr.tree, apr.dims
        v = R.random_values(rng, leaf.y_idx.size, -100, 100)
        tv = R.fill_tree(apr, v)
        assert np.array_equal(G.bits(tv), G.bits(ORC.fill_tree(leaf, tree, dims, v)))
        t2 = ORC.init_tree_structure(leaf, dims)
        assert np.array_equal(t2.y_idx, tree.y_idx) and np.array_equal(t2.xz_end, tree.xz_end)
        for k3 in ((3, 3, 3), (5, 5, 5), (3, 1, 5)):
            w = R.random_stencil(rng, *k3)
            pyr = R.make_pyramid(w, k3, leaf.l_min, leaf.l_max, 0)
            lv = pyr.levels()
            for pad in (0, 1):
                a = R.convolve(apr, v, tv, pyr, pad, threads=2)
                b = ORC.convolve(leaf, tree, v, tv, lv, leaf.l_min, pad)
                assert np.array_equal(G.bits(a), G.bits(b))


def test_oracle_builder_matches_c1_golden():
    """The multi-threaded C builder (oracle/build_oracle.c) reproduces the
    reference-built C1 fixture (256^3 spheres, BASELINE config 1) bit for bit:
    structure and sampled values."""
    d = G.load("c1_256")
    acc, vals = ORC.build_spheres(256, 12, 6.0, 20.0, blur=2.0, seed=42, rel_error=0.1)
    g = G.oracle_access(d, "leaf_")
    assert (acc.l_min, acc.l_max) == (g.l_min, g.l_max)
    assert np.array_equal(acc.y_idx, g.y_idx)
    assert np.array_equal(acc.xz_end, g.xz_end)
    assert np.array_equal(acc.level_offset[acc.l_min:], g.level_offset[g.l_min:])
    assert np.array_equal(G.bits(vals), G.bits(d["values"]))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("dims,count,rmin,rmax,seed", [((64, 64, 64), 6, 3.0, 10.0, 7), ((40, 33, 57), 5, 2.0, 8.0, 3),
                                                       ((7, 9, 5), 2, 1.0, 3.0, 1), ((48, 40, 56), 7, 2.5, 9.0, 42)])
def test_oracle_builder_matches_live_reference(dims, count, rmin, rmax, seed):
    """generate_spheres + build_apr of the C builder vs the unmodified reference
    (oracle/_ref), non-power-of-two and anisotropic dims included."""
    R = Ref()
    vol = ORC.generate_spheres(dims, count, rmin, rmax, 2.0, seed, threads=4)
    rvol = R.generate_spheres(dims, count, rmin, rmax, 2.0, 0.0, seed)
    assert np.array_equal(G.bits(vol), G.bits(rvol))
    acc, vals = ORC.build_apr(vol, 0.1, threads=4)
    r = R.build_apr(rvol, 0.1)
    ra = r.leaf
    for f in ("y_idx", "xz_end", "level_offset", "z_dim", "x_dim", "y_dim"):
        assert np.array_equal(getattr(acc, f), getattr(ra, f)), f
    assert np.array_equal(G.bits(vals), G.bits(r.values()))
