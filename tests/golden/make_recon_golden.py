"""Golden vectors for the dense reconstruction (reconstruct.hpp:73-129), from
the REAL reference (oracle/_ref/libaprref.so, built from /root/reference --
so this only runs in the container that has it).  Structures and values are
those of the committed fixtures; the outputs go to tests/golden/recon.npz,
which travels to the GPU box for tests/test_reconstruct.py.

    python tests/golden/make_recon_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, ".."))
import goldens as G  # noqa: E402
from pyoracle import Ref  # noqa: E402

R = Ref()
CASES = ["spheres64", "dense16", "blobs32_0", "random_apr_00", "random_apr_03", "random_apr_07"]


def patches(leaf):
    """(level, z_begin, z_end, x_begin, x_end, pad, pad_mode) windows: interior,
    corner and whole-grid, both pad modes, pads past one cell and past the grid."""
    out = []
    for l in sorted({leaf.l_max, max(leaf.l_min, leaf.l_max - 1)}):
        zd, xd = int(leaf.z_dim[l]), int(leaf.x_dim[l])
        out.append((l, zd // 4, max(zd // 4 + 1, 3 * zd // 4), xd // 3, max(xd // 3 + 1, 2 * xd // 3), 2, 1))
        out.append((l, 0, min(zd, 3), 0, min(xd, 4), 3, 0))
        out.append((l, 0, zd, 0, xd, 1, 1))
        out.append((l, zd - 1, zd, 0, xd, min(zd, 5) + 2, 1))  # pad wider than the grid: multi-fold reflection
    return out


def main():
    res = {}
    for name in CASES:
        d = G.load(name)
        leaf = G.oracle_access(d, "leaf_")
        dims = tuple(int(v) for v in d["dims"])
        apr = R.apr_from_arrays(leaf, dims)
        v, tv = d["values"], d["tree_values"]
        res[f"{name}__full"] = R.reconstruct_full(apr, v)
        for l in range(leaf.l_min, leaf.l_max + 1):
            res[f"{name}__level{l}"] = R.reconstruct_level(apr, v, tv, l)
        for k, sp in enumerate(patches(leaf)):
            res[f"{name}__patch{k}_spec"] = np.array(sp, np.int32)
            res[f"{name}__patch{k}"] = R.reconstruct_patch(apr, v, tv, sp)
    np.savez_compressed(os.path.join(HERE, "recon.npz"), **res)
    print("recon.npz:", len(res), "arrays,", sum(a.nbytes for a in res.values()) // 1024, "KiB raw")


if __name__ == "__main__":
    main()
