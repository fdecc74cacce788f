"""Golden outputs of convolve_pixels (convolve.hpp:48-98) from the REAL
reference (oracle/_ref/libaprref.so; runs only where /root/reference is):
volumes x stencils x pad modes -> tests/golden/pixels.npz, checked bit for bit
against the C oracle (CPU) and the device kernel in EXACT mode (GPU).

    python tests/golden/make_pixels_golden.py
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


def main():
    rng = np.random.default_rng(48)
    recon = G.load("recon")
    vols = {
        "spheres64": np.ascontiguousarray(recon["spheres64__full"][12:52, 20:44, 8:56]),
        "random": rng.uniform(-100, 1000, (11, 17, 70)).astype(np.float32),
        "thin": rng.uniform(0, 1, (1, 3, 129)).astype(np.float32),
    }
    sts = {
        "g3": ((3, 3, 3), None),
        "g5": ((5, 5, 5), None),
        "r531": ((5, 3, 1), rng.uniform(-1, 1, 15)),
        "r7": ((7, 7, 7), rng.uniform(-1, 1, 343)),
        "r13": ((13, 13, 13), rng.uniform(-1, 1, 2197)),
        "sparse": ((3, 5, 3), np.where(rng.uniform(0, 1, 45) < 0.5, 0.0, rng.uniform(-1, 1, 45))),
    }
    res = {}
    for vn, v in vols.items():
        res[f"{vn}__vol"] = v
        for sn, (k3, w) in sts.items():
            if vn == "spheres64" and sn in ("r7", "r13", "sparse", "r531"):
                continue
            if w is None:
                w = R.gaussian_stencil(1.0, k3[0])[1]
            w = np.asarray(w, np.float32).reshape(-1)
            for pad in (0, 1):
                key = f"{vn}__{sn}__p{pad}"
                res[key + "_k3"] = np.array(k3, np.int32)
                res[key + "_w"] = w
                res[key] = R.convolve_pixels(v, w, k3, pad)
    np.savez_compressed(os.path.join(HERE, "pixels.npz"), **res)
    print(len(res), "arrays")


if __name__ == "__main__":
    main()
