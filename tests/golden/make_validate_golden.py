"""Golden verdicts of validate (apr.hpp:61-134) on valid and deliberately broken
leaf structures, from the REAL reference (oracle/_ref/libaprref.so; runs only
in the container that has /root/reference).  Each case stores the (mutated)
leaf arrays, the image dims and the reference's (ok, message); the device
validator (aprgpu_validate_access) must reproduce both.

    python tests/golden/make_validate_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, ".."))
import goldens as G  # noqa: E402
from pyoracle import Access, Ref  # noqa: E402

R = Ref()
BASES = ["dense16", "blobs32_0", "random_apr_00", "random_apr_02", "random_apr_05", "spheres64"]


def arrays(a):
    return dict(l_min=a.l_min, l_max=a.l_max, z_dim=a.z_dim.copy(), x_dim=a.x_dim.copy(), y_dim=a.y_dim.copy(),
                y_idx=a.y_idx.copy(), xz_end=a.xz_end.copy(), level_offset=a.level_offset.copy())


def rows_of(f):
    ends = f["xz_end"].astype(np.int64)
    begins = np.concatenate([[0], ends[:-1]])
    return begins, ends


def level_of_row(f, r):
    l = f["l_max"]
    while l > f["l_min"] and r < f["level_offset"][l]:
        l -= 1
    return l


def remove_particle(f, i):
    f["y_idx"] = np.delete(f["y_idx"], i)
    f["xz_end"] = np.where(f["xz_end"] > i, f["xz_end"] - 1, f["xz_end"]).astype(np.uint64)


def insert_particle(f, row, y):
    b, e = (int(f["xz_end"][row - 1]) if row else 0), int(f["xz_end"][row])
    seg = f["y_idx"][b:e]
    pos = b + int(np.searchsorted(seg, y))
    f["y_idx"] = np.insert(f["y_idx"], pos, np.uint16(y))
    f["xz_end"] = np.where(np.arange(f["xz_end"].size) >= row, f["xz_end"] + 1, f["xz_end"]).astype(np.uint64)


def mutations(base, dims, rng):
    """(name, arrays, dims) for the valid base and one of each violation."""
    out = [("valid", arrays(base), dims)]
    b0, e0 = rows_of(arrays(base))
    full = [r for r in range(len(e0)) if e0[r] - b0[r] >= 2]
    # a removed leaf: uncovered pixels
    f = arrays(base)
    i = int(rng.integers(0, f["y_idx"].size))
    remove_particle(f, i)
    out.append(("removed_leaf", f, dims))
    # a leaf added over finer leaves: double coverage
    f = arrays(base)
    fine = [r for r in range(len(e0)) if e0[r] > b0[r] and level_of_row(f, r) > f["l_min"]]
    if fine:
        r = fine[int(rng.integers(0, len(fine)))]
        l = level_of_row(f, r)
        loc = r - int(f["level_offset"][l])
        z, x = divmod(loc, int(f["x_dim"][l]))
        y = int(f["y_idx"][b0[r]])
        pr = int(f["level_offset"][l - 1]) + (z >> 1) * int(f["x_dim"][l - 1]) + (x >> 1)
        pb, pe = (int(f["xz_end"][pr - 1]) if pr else 0), int(f["xz_end"][pr])
        if (y >> 1) not in set(int(v) for v in f["y_idx"][pb:pe]):
            insert_particle(f, pr, y >> 1)
            out.append(("coarse_over_fine", f, dims))
    if full:
        # two y swapped in a row: non-increasing y
        f = arrays(base)
        r = full[int(rng.integers(0, len(full)))]
        f["y_idx"][b0[r]], f["y_idx"][b0[r] + 1] = f["y_idx"][b0[r] + 1], f["y_idx"][b0[r]]
        out.append(("swapped_y", f, dims))
        # a repeated y
        f = arrays(base)
        f["y_idx"][b0[r] + 1] = f["y_idx"][b0[r]]
        out.append(("repeated_y", f, dims))
    # the last particle of a row moved past the level grid
    f = arrays(base)
    nz_rows = [r for r in range(len(e0)) if e0[r] > b0[r]]
    r = nz_rows[-1]
    f["y_idx"][e0[r] - 1] = np.uint16(f["y_dim"][level_of_row(f, r)])
    out.append(("y_past_grid", f, dims))
    # a smaller image than the structure: cells outside the domain
    if dims[2] > 2:
        out.append(("image_too_small", arrays(base), (dims[0], dims[1], dims[2] // 2)))
    # a larger image than the structure: uncovered pixels past the cells
    out.append(("image_too_large", arrays(base), (dims[0], dims[1] + 4, dims[2])))
    # host-side structure checks
    f = arrays(base)
    f["level_offset"][f["l_max"]] += 1
    out.append(("level_offset", f, dims))
    f = arrays(base)
    f["xz_end"] = f["xz_end"][:-1].copy()
    out.append(("xz_end_length", f, dims))
    f = arrays(base)
    if len(full) and full[0] > 0:
        f["xz_end"][full[0] - 1] = f["xz_end"][full[0]] + 1
        out.append(("xz_end_decreases", f, dims))
    f = arrays(base)
    f["xz_end"][-1] -= 1
    out.append(("xz_end_last", f, dims))
    return out


def main():
    rng = np.random.default_rng(2112)
    res = {}
    k = 0
    for name in BASES:
        d = G.load(name)
        leaf = G.oracle_access(d, "leaf_")
        dims = tuple(int(v) for v in d["dims"])
        for mname, f, dm in mutations(leaf, dims, rng):
            ok, msg = R.validate_arrays(Access(**f), dm)
            key = f"c{k:03d}"
            for fk, fv in f.items():
                res[f"{key}_{fk}"] = np.asarray(fv)
            res[f"{key}_dims"] = np.array(dm, np.int32)
            res[f"{key}_ok"] = np.array([int(ok)], np.int32)
            res[f"{key}_msg"] = np.frombuffer(msg.encode(), np.uint8)
            res[f"{key}_name"] = np.frombuffer(f"{name}/{mname}".encode(), np.uint8)
            print(f"{key} {name}/{mname}: {ok} {msg}")
            k += 1
    np.savez_compressed(os.path.join(HERE, "validate.npz"), **res)


if __name__ == "__main__":
    main()
