"""Dense reconstruction (reconstruct.hpp:73-129).

CPU: the C oracle's reconstruct_level / reconstruct_patch against golden vectors
made by the real reference (tests/golden/make_recon_golden.py) -- pins the
oracle.  GPU: the device path (aprgpu_reconstruct_level / _patch through the
C-ABI) against the same golden vectors and, on fresh random values, against
the oracle; all bit-for-bit (reconstruction copies values, no arithmetic).
"""
import numpy as np
import pytest

import goldens as G
from pyoracle import Oracle

ORC = Oracle()
RECON = G.load("recon")
CASES = sorted({k.split("__")[0] for k in RECON})


def _patch_keys(name):
    return sorted(k[: -len("_spec")] for k in RECON if k.startswith(name + "__patch") and k.endswith("_spec"))


@pytest.mark.parametrize("name", CASES)
def test_oracle_reconstruction_matches_reference(name):
    d = G.load(name)
    leaf, tree = G.oracle_access(d, "leaf_"), G.oracle_access(d, "tree_")
    v, tv = d["values"], d["tree_values"]
    assert np.array_equal(ORC.reconstruct_level(leaf, tree, v, None, leaf.l_max), RECON[f"{name}__full"])
    for l in range(leaf.l_min, leaf.l_max + 1):
        assert np.array_equal(ORC.reconstruct_level(leaf, tree, v, tv, l), RECON[f"{name}__level{l}"]), l
    for k in _patch_keys(name):
        got = ORC.reconstruct_patch(leaf, tree, v, tv, tuple(RECON[k + "_spec"]))
        assert np.array_equal(got, RECON[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_reconstruction_bit_identical(name):
    import paper_2112_03592_b200 as P
    d = G.load(name)
    apr = G.product_apr(d)
    v, tv = d["values"], d["tree_values"]
    assert np.array_equal(G.bits(P.reconstruct_full(apr, v)), G.bits(RECON[f"{name}__full"]))
    for l in range(apr.access.l_min, apr.access.l_max + 1):
        got = P.reconstruct_level(apr, v, tv, l)
        assert np.array_equal(G.bits(got), G.bits(RECON[f"{name}__level{l}"])), l
    for k in _patch_keys(name):
        s = [int(x) for x in RECON[k + "_spec"]]
        spec = P.PatchSpec(s[0], s[1], s[2], s[3], s[4], s[5], P.PadMode(s[6]))
        got = P.reconstruct_patch(apr, v, tv, spec)
        assert np.array_equal(G.bits(got), G.bits(RECON[k])), k


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2])
def test_device_reconstruction_random_values_vs_oracle(seed):
    import paper_2112_03592_b200 as P
    rng = np.random.default_rng(seed)
    for name in G.names("random_apr_*")[seed::2] + ["c1_256"]:
        d = G.load(name)
        apr = G.product_apr(d)
        leaf, tree = G.oracle_access(d, "leaf_"), G.oracle_access(d, "tree_")
        v = rng.uniform(-1e3, 1e3, leaf.y_idx.size).astype(np.float32)
        tv = rng.uniform(-1e3, 1e3, tree.y_idx.size).astype(np.float32)
        for l in (leaf.l_min, leaf.l_max):
            exp = ORC.reconstruct_level(leaf, tree, v, tv, l)
            assert np.array_equal(G.bits(P.reconstruct_level(apr, v, tv, l)), G.bits(exp)), (name, l)
        l = leaf.l_max
        zd, xd = int(leaf.z_dim[l]), int(leaf.x_dim[l])
        for pad_mode in (P.PadMode.Zero, P.PadMode.Reflect):
            spec = P.PatchSpec(l, zd // 3, zd, 0, max(1, xd // 2), 2, pad_mode)
            exp = ORC.reconstruct_patch(leaf, tree, v, tv, (l, zd // 3, zd, 0, max(1, xd // 2), 2, int(pad_mode)))
            assert np.array_equal(G.bits(P.reconstruct_patch(apr, v, tv, spec)), G.bits(exp)), (name, pad_mode)


@pytest.mark.gpu
def test_reconstruction_errors_are_range_errors():
    import paper_2112_03592_b200 as P
    d = G.load("spheres64")
    apr = G.product_apr(d)
    with pytest.raises(P.RangeError):
        P.reconstruct_level(apr, d["values"], d["tree_values"], apr.access.l_max + 1)
    with pytest.raises(P.RangeError):
        l = apr.access.l_max
        P.reconstruct_patch(apr, d["values"], d["tree_values"], P.PatchSpec(l, 0, 10 ** 6, 0, 1, 0))
    with pytest.raises(P.RangeError):
        P.reconstruct_patch(apr, d["values"], d["tree_values"], P.PatchSpec(apr.access.l_max, 0, 1, 0, 1, -1))
