"""The C4 tiler (aprgpu_tile_apr) against a plain numpy restatement of the
tiling recipe and the reference-order oracle: structure,
rebuilt interior structure and a convolution of the tiled APR."""
import numpy as np
import pytest
import torch

import goldens as G
import paper_2112_03592_b200 as P
from paper_2112_03592_b200 import _lib as L, synth
from pyoracle import Access, Oracle

pytestmark = pytest.mark.gpu


def tile_access_numpy(a, n, tz, tx, ty):
    """Big level l = tl + sh holds in row (z, x) the source row (tl, z mod 2^tl,
    x mod 2^tl) repeated ty times along y with offsets k * 2^tl."""
    big = (n * tz, n * tx, n * ty)
    BL = 0
    while (1 << BL) < max(big):
        BL += 1
    sh = BL - a.l_max
    l_min = min(1, BL)
    zd = [-(-big[0] // (1 << (BL - l))) for l in range(BL + 1)]
    xd = [-(-big[1] // (1 << (BL - l))) for l in range(BL + 1)]
    yd = [-(-big[2] // (1 << (BL - l))) for l in range(BL + 1)]
    ends = np.concatenate([[0], np.asarray(a.xz_end, np.int64)])
    ys, counts, lo = [], [], []
    rows = 0
    for l in range(BL + 1):
        lo.append(rows if l >= l_min else 0)
        if l < l_min:
            continue
        tl = l - sh
        for z in range(zd[l]):
            for x in range(xd[l]):
                if a.l_min <= tl <= a.l_max:
                    r = int(a.level_offset[tl]) + (z % int(a.z_dim[tl])) * int(a.x_dim[tl]) + (x % int(a.x_dim[tl]))
                    row = np.asarray(a.y_idx[ends[r]:ends[r + 1]], np.int64)
                    seg = np.concatenate([row + k * int(a.y_dim[tl]) for k in range(ty)]) if row.size else row
                else:
                    seg = np.zeros(0, np.int64)
                ys.append(seg)
                counts.append(seg.size)
        rows += zd[l] * xd[l]
    y = np.concatenate(ys).astype(np.uint16) if ys else np.zeros(0, np.uint16)
    return P.LinearAccess(l_min, BL, zd, xd, yd, y, np.cumsum(counts).astype(np.uint64), lo), big


@pytest.mark.parametrize("t3", [(2, 2, 2), (4, 1, 2), (1, 3, 1)])
def test_tiler_matches_recipe_and_oracle(t3):
    d = G.load("spheres64")
    apr = G.product_apr(d)
    dev = apr.device()
    big = synth.tile_apr(dev, *t3)
    exp, dims = tile_access_numpy(apr.access, 64, *t3)
    assert big.download(L.LEAF).equals(exp)
    O = Oracle()
    tree = O.init_tree_structure(exp, dims)
    got_tree = big.download(L.TREE)
    assert np.array_equal(got_tree.y_idx, tree.y_idx) and np.array_equal(got_tree.xz_end, tree.xz_end)
    # tiled values + fill_tree + conv of the tiled APR vs the oracle
    v = torch.from_numpy(d["values"]).cuda()
    bv = torch.empty(big.n_particles, dtype=torch.float32, device="cuda")
    synth.tile_values(dev, big, *t3, v.data_ptr(), bv.data_ptr())
    torch.cuda.synchronize()
    vals = bv.cpu().numpy()
    tv = big.fill_tree(vals)
    assert np.array_equal(G.bits(tv), G.bits(O.fill_tree(exp, tree, dims, vals)))
    w = P.gaussian_stencil(1.0, 3)
    pyr = P.make_pyramid(w, exp.l_min, exp.l_max, P.PyramidMode.Restricted)
    out = big.convolve(vals, tv, pyr.device(big.ctx), 1, L.ACCUM_EXACT)
    levels = [((s.kz, s.kx, s.ky), s.weights) for s in pyr.stencils]
    ref = O.convolve(exp, tree, vals, tv, levels, exp.l_min, 1)
    assert np.array_equal(G.bits(out), G.bits(ref))
