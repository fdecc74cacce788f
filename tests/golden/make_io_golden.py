"""Golden .apr containers (io.hpp:102-183, docs/FORMATS.md) written by the REAL
reference (oracle/_ref/libaprref.so; runs only where /root/reference is), and
the reference reader's verdict on byte-level corruptions of them.  The device
loader (aprgpu_load_apr) must read the files to the same structures and values,
write them back byte for byte (aprgpu_save_apr), and fail on each corruption
with the same exception type and message.

    python tests/golden/make_io_golden.py
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, ".."))
import goldens as G  # noqa: E402
from pyoracle import Ref  # noqa: E402

R = Ref()
OUT = os.path.join(HERE, "apr")


def corruptions(size: int, n_leaf: int, head: int, leaf):
    """(name, truncate_to or -1, [(offset, byte)]) recipes on a file of `size` bytes."""
    nl = int(leaf.l_max) + 1
    leaf_end = head + 8 + 12 * nl + 8 + 8 * nl + 8 + 8 * int(leaf.xz_end.size) + 8 + 2 * int(leaf.y_idx.size)
    last_y = leaf_end - 2  # the last leaf particle's y: 0 breaks its row's order
    return [
        ("empty", 0, []),
        ("truncated_header", 10, []),
        ("truncated_values", size - 3, []),
        ("bad_magic", -1, [(0, ord("X"))]),
        ("bad_version", -1, [(4, 2)]),
        ("zero_dim", -1, [(5, 0), (6, 0), (7, 0), (8, 0)]),
        ("bad_sigma_mode", -1, [(25, 7)]),
        ("bad_gradient_mode", -1, [(46, 3)]),
        ("bad_level_range", -1, [(head, 0xff), (head + 1, 0xff), (head + 2, 0xff), (head + 3, 0x7f)]),
        ("implausible_count", -1, [(size - 4 * n_leaf - 1, 0x7f)]),
        ("broken_structure", -1, [(last_y, 0), (last_y + 1, 0)]),
    ]


def main():
    os.makedirs(OUT, exist_ok=True)
    files = {}
    d = G.load("spheres64")
    leaf = G.oracle_access(d, "leaf_")
    apr = R.apr_from_arrays(leaf, tuple(int(v) for v in d["dims"]))
    R.save_apr(apr, d["values"], os.path.join(OUT, "spheres64.apr"))
    files["spheres64"] = (int(leaf.y_idx.size), leaf)
    built = R.build_spheres(40, 5, 3.0, 9.0, blur=2.0, seed=7, rel_error=0.1)
    R.save_apr(built, built.values(), os.path.join(OUT, "built40.apr"))
    files["built40"] = (int(built.n_particles()), built.leaf)
    res = {}
    # magic 4 + version 1 + dims 12 + rel_error 8 + sigma mode 1 + value 8 + window 4 + floor 8 + gradient 1 + passes 4
    head = 4 + 1 + 12 + 8 + 1 + 8 + 4 + 8 + 1 + 4
    for name, (n_leaf, lf) in files.items():
        raw = open(os.path.join(OUT, name + ".apr"), "rb").read()
        for cname, trunc, edits in corruptions(len(raw), n_leaf, head, lf):
            b = bytearray(raw if trunc < 0 else raw[:trunc])
            for off, v in edits:
                b[off] = v
            with tempfile.NamedTemporaryFile(suffix=".apr", delete=False) as f:
                f.write(bytes(b))
            kind, msg, h = R.load_apr(f.name)
            os.unlink(f.name)
            key = f"{name}__{cname}"
            res[key + "_trunc"] = np.array([trunc], np.int64)
            res[key + "_edits"] = np.array(edits, np.int64).reshape(-1, 2)
            res[key + "_kind"] = np.array([kind], np.int32)
            res[key + "_msg"] = np.frombuffer(msg.encode(), np.uint8)
            print(key, kind, msg)
    np.savez_compressed(os.path.join(HERE, "io.npz"), **res)


if __name__ == "__main__":
    main()
