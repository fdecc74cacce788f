"""Generate the committed golden vectors in tests/golden/ from the REAL reference.

Runs the unmodified aprkit headers compiled into oracle/_ref/libaprref.so
(see oracle/Makefile) -- so it only runs in the container that has
/root/reference.  The .npz files it writes are committed and travel to the GPU
box, where tests/test_parity_gpu.py compares the CUDA path against them
bit-for-bit.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from pyoracle import Ref  # noqa: E402

R = Ref()


def pack_access(prefix: str, a, out: dict):
    out[prefix + "l_range"] = np.array([a.l_min, a.l_max], np.int32)
    for k in ("z_dim", "x_dim", "y_dim", "y_idx", "xz_end", "level_offset"):
        out[prefix + k] = getattr(a, k)


def pack_pyr(prefix: str, levels, out: dict):
    out[prefix + "k3"] = np.array([list(k) for k, _ in levels], np.int32)
    out[prefix + "w"] = np.concatenate([w for _, w in levels]).astype(np.float32)


def row_index(apr, out: dict):
    leaf = apr.leaf
    zs, xs, y0s, y1s, cnt = [], [], [], [], []
    for l in range(leaf.l_min, leaf.l_max + 1):
        z, x, y0, y1 = R.nonempty_rows(apr, l)
        zs.append(z); xs.append(x); y0s.append(y0); y1s.append(y1); cnt.append(z.size)
    out["rows_count"] = np.array(cnt, np.int64)
    out["rows_z"] = np.concatenate(zs)
    out["rows_x"] = np.concatenate(xs)
    out["rows_ymin"] = np.concatenate(y0s)
    out["rows_ymax"] = np.concatenate(y1s)


def conv_case(apr, values, tree, w, k3, mode, pad, name, out: dict):
    leaf = apr.leaf
    pyr = R.make_pyramid(w, k3, leaf.l_min, leaf.l_max, mode)
    levels = pyr.levels()
    o = R.convolve(apr, values, tree, pyr, pad)
    pack_pyr(f"conv_{name}_pyr_", levels, out)
    out[f"conv_{name}_pad"] = np.array([pad], np.int32)
    out[f"conv_{name}_out"] = o


def save(name: str, d: dict):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **d)
    print(f"{name}: {os.path.getsize(path) / 1024:.1f} KiB")


def base(apr, values):
    d = {}
    pack_access("leaf_", apr.leaf, d)
    pack_access("tree_", apr.tree, d)
    d["dims"] = np.array(apr.dims, np.int32)
    d["values"] = values
    tv = R.fill_tree(apr, values)
    d["tree_values"] = tv
    row_index(apr, d)
    return d, tv


def random_aprs():
    # test_convolve.cpp:56-80 / test_tree.cpp style random APRs (helpers.hpp:23-52)
    rng = R.rng(1010)
    for i in range(10):
        apr = R.random_apr(rng, 4, 28 if i < 6 else 40)
        v = R.random_values(rng, apr.n_particles(), -100, 100)
        d, tv = base(apr, v)
        w3 = R.random_stencil(rng, 3, 3, 3)
        for pad in (0, 1):
            conv_case(apr, v, tv, w3, (3, 3, 3), 0, pad, f"r3_p{pad}", d)
        w535 = R.random_stencil(rng, 5, 3, 5)
        conv_case(apr, v, tv, w535, (5, 3, 5), 0, 1, "r535", d)
        w5 = R.random_stencil(rng, 5, 5, 5)
        conv_case(apr, v, tv, w5, (5, 5, 5), 0, 0, "r5_p0", d)
        w113 = R.random_stencil(rng, 1, 1, 3)
        conv_case(apr, v, tv, w113, (1, 1, 3), 2, 1, "u113", d)
        if i % 3 == 0:
            w13 = R.random_stencil(rng, 13, 13, 13)
            conv_case(apr, v, tv, w13, (13, 13, 13), 0, 1, "r13", d)
        k3, g = R.gaussian_stencil(1.0, 3)
        conv_case(apr, v, tv, g, k3, 1, 1, "g3_rescaled", d)
        save(f"random_apr_{i:02d}", d)


def blob_aprs():
    # acceptance.cpp criterion 3 shape: 32^3 APRs from blob targets, k in {3,5,13}
    g = np.random.default_rng(3300)
    for i in range(4):
        n = 32
        l_max = 5
        l_min = 1
        t = np.full((n, n, n), l_min, np.int32)
        zz, xx, yy = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
        for _ in range(1 + int(g.integers(0, 5))):
            level = int(g.integers(l_min, l_max + 1))
            c = g.uniform(0, n, 3)
            r = g.uniform(2.0, 0.35 * n)
            m = (zz - c[0]) ** 2 + (xx - c[1]) ** 2 + (yy - c[2]) ** 2 <= r * r
            t[m] = np.maximum(t[m], level)
        apr = R.apr_from_targets(t, l_min, l_max)
        v = g.uniform(-100, 100, apr.n_particles()).astype(np.float32)
        d, tv = base(apr, v)
        for k in (3, 5, 13):
            w = g.uniform(-1, 1, k ** 3).astype(np.float32)
            conv_case(apr, v, tv, w, (k, k, k), 0, 1, f"r{k}", d)
        save(f"blobs32_{i}", d)


def spheres64():
    # acceptance.cpp criterion 5 scene (64^3, 10 spheres, blur 1.5, seed 5500)
    apr = R.build_spheres(64, 10, 3.0, 10.0, 1.5, 0.0, 5500, 0.1)
    v = apr.values()
    d, tv = base(apr, v)
    for k in (3, 5):
        k3, w = R.gaussian_stencil(1.0, k)
        conv_case(apr, v, tv, w, k3, 0, 1, f"g{k}", d)
    save("spheres64", d)


def dense16():
    # test_convolve.cpp:82-100: dense APR (CR = 1), 5^3 Gaussian
    n = 16
    t = np.full((n, n, n), 4, np.int32)
    apr = R.apr_from_targets(t, 1, 4)
    g = np.random.default_rng(2020)
    v = g.uniform(0, 1000, apr.n_particles()).astype(np.float32)
    d, tv = base(apr, v)
    k3, w = R.gaussian_stencil(1.0, 5)
    conv_case(apr, v, tv, w, k3, 0, 1, "g5", d)
    save("dense16", d)


def restrict_vectors():
    rng = R.rng(777)
    d = {}
    idx = 0
    cases = [(1, 1, 1), (3, 3, 3), (5, 5, 5), (5, 3, 5), (1, 3, 7), (13, 13, 13)]
    for k3 in cases:
        for delta in range(0, 6 if k3 != (13, 13, 13) else 4):
            w = R.random_stencil(rng, *k3)
            ok, out = R.restrict_stencil(w, k3, delta)
            d[f"c{idx}_in"] = w
            d[f"c{idx}_meta"] = np.array(list(k3) + [delta] + list(ok), np.int32)
            d[f"c{idx}_out"] = out
            idx += 1
    for sigma, size in ((1.0, 3), (1.0, 5), (2.0, 0), (0.7, 13)):
        k3, w = R.gaussian_stencil(sigma, size)
        d[f"gauss_{idx}_meta"] = np.array([int(sigma * 1000), size, k3[0]], np.int32)
        d[f"gauss_{idx}_w"] = w
        for delta in (1, 2, 3, 4, 5):
            ok, out = R.restrict_stencil(w, k3, delta)
            d[f"c{idx}_in"] = w
            d[f"c{idx}_meta"] = np.array(list(k3) + [delta] + list(ok), np.int32)
            d[f"c{idx}_out"] = out
            idx += 1
    d["n_cases"] = np.array([idx], np.int32)
    save("restrict", d)


def rl_case():
    # rl_apr on a 64^3 sphere APR (positive values), 10 iterations, Gaussian PSFs
    apr = R.build_spheres(64, 8, 3.0, 10.0, 1.0, 0.0, 4040, 0.1)
    v = apr.values()
    d, _ = base(apr, v)
    for k in (3, 5):
        k3, w = R.gaussian_stencil(1.0, k)
        d[f"rl_g{k}_psf"] = w
        d[f"rl_g{k}_out"] = R.rl_apr(apr, v, w, k3, 10)
    save("rl_spheres64", d)


def c1():
    # 256^3, 12 spheres, r in [6,20], blur 2, seed 42, E = 0.1
    apr = R.build_spheres(256, 12, 6.0, 20.0, 2.0, 0.0, 42, 0.1)
    v = apr.values()
    d, tv = base(apr, v)
    for k in (3, 5):
        k3, w = R.gaussian_stencil(1.0, k)
        conv_case(apr, v, tv, w, k3, 0, 1, f"g{k}", d)
    save("c1_256", d)


if __name__ == "__main__":
    which = sys.argv[1:] or ["random", "blobs", "spheres64", "dense16", "restrict", "rl", "c1"]
    if "random" in which:
        random_aprs()
    if "blobs" in which:
        blob_aprs()
    if "spheres64" in which:
        spheres64()
    if "dense16" in which:
        dense16()
    if "restrict" in which:
        restrict_vectors()
    if "rl" in which:
        rl_case()
    if "c1" in which:
        c1()
