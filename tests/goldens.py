"""Loading helpers for the committed golden vectors (tests/golden/*.npz,
produced by tests/golden/make_golden.py from the real reference)."""
from __future__ import annotations

import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names(pattern: str = "*"):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, pattern + ".npz")))


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def access_fields(d: dict, prefix: str) -> dict:
    lr = d[prefix + "l_range"]
    return dict(l_min=int(lr[0]), l_max=int(lr[1]), z_dim=d[prefix + "z_dim"], x_dim=d[prefix + "x_dim"],
                y_dim=d[prefix + "y_dim"], y_idx=d[prefix + "y_idx"], xz_end=d[prefix + "xz_end"],
                level_offset=d[prefix + "level_offset"])


def oracle_access(d: dict, prefix: str):
    from pyoracle import Access
    return Access(**access_fields(d, prefix))


def product_apr(d: dict, with_tree: bool = True):
    from paper_2112_03592_b200 import APR, LinearAccess
    leaf = LinearAccess(**access_fields(d, "leaf_"))
    tree = LinearAccess(**access_fields(d, "tree_")) if with_tree else None
    return APR(leaf, tree, tuple(int(v) for v in d["dims"]))


def conv_names(d: dict):
    return sorted(k[len("conv_"):-len("_out")] for k in d if k.startswith("conv_") and k.endswith("_out"))


def pyramid_levels(d: dict, name: str):
    k3 = d[f"conv_{name}_pyr_k3"]
    w = d[f"conv_{name}_pyr_w"]
    out, off = [], 0
    for k in k3:
        n = int(np.prod(k))
        out.append((tuple(int(v) for v in k), w[off:off + n]))
        off += n
    return out


def bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def as_oracle(a):
    """An oracle Access from a product LinearAccess."""
    from pyoracle import Access
    return Access(l_min=a.l_min, l_max=a.l_max, z_dim=np.asarray(a.z_dim, np.int32),
                  x_dim=np.asarray(a.x_dim, np.int32), y_dim=np.asarray(a.y_dim, np.int32),
                  y_idx=np.asarray(a.y_idx, np.uint16), xz_end=np.asarray(a.xz_end, np.uint64),
                  level_offset=np.asarray(a.level_offset, np.uint64))
