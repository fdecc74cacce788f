"""The resident gather maps (aprgpu_map_records): after a 3^3 convolution
every particle of a 3^3 level is named by exactly one output-mask bit of one
tile record, and every active 2x2x2 block holds an output -- the map build's
bookkeeping, checked from the records themselves (record layout: MapBox<1> in
csrc/conv_tile.cu)."""
import ctypes as C

import numpy as np
import pytest

import goldens as G
import paper_2112_03592_b200 as P
from paper_2112_03592_b200 import _lib as L

pytestmark = pytest.mark.gpu

BZ = BX = 10
BY = 36  # (MapBox rows: kTY + 4 cells)
CW = BZ * BX * BY // 2  # code words; then 64 masks, 64 first indices, chunks, blocks, 2 pad, block list


def records(dapr, level, pad):
    nw, t0, nt = C.c_uint64(), C.c_uint64(), C.c_uint64()
    L.check(L.lib().aprgpu_map_records(dapr.handle, 1, pad, level, None, 0, None, C.byref(nw), C.byref(t0),
                                       C.byref(nt)))
    if nt.value == 0:
        return np.zeros((0, 0), np.uint32), 0
    buf = np.empty(nw.value, np.uint32)
    off = np.empty(nt.value + 1, np.uint32)
    L.check(L.lib().aprgpu_map_records(dapr.handle, 1, pad, level, buf.ctypes.data, buf.size, off.ctypes.data,
                                       C.byref(nw), C.byref(t0), C.byref(nt)))
    assert off[0] == 0 and off[-1] == nw.value and np.all(np.diff(off) == off[1])
    return buf.reshape(nt.value, -1), t0.value


@pytest.mark.parametrize("name", ["spheres64", "c1_256"] + G.names("random_apr_0*")[:3])
@pytest.mark.parametrize("pad", [P.PadMode.Reflect, P.PadMode.Zero])
def test_map_records_cover_every_output_once(name, pad):
    d = G.load(name)
    apr = G.product_apr(d)
    a = apr.access
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted)
    tv = P.fill_tree(apr, d["values"])
    ctx = P.default_context()
    dev = P.DeviceApr.upload(ctx, apr)
    out = dev.convolve(d["values"], tv, pyr.device(ctx), int(pad), L.ACCUM_EXACT)
    assert out.size == a.particle_count()
    lo = [int(x) for x in a.level_offset] + [a.row_count()]
    ends = np.concatenate([[0], np.asarray(a.xz_end, np.int64)])
    for lvl in range(a.l_min, a.l_max + 1):
        rec, t0 = records(dev, lvl, int(pad))
        first, nxt = int(ends[lo[lvl]]), int(ends[lo[lvl + 1]])
        n_lvl = nxt - first
        if rec.shape[0] == 0:
            assert n_lvl == 0, lvl
            continue
        masks = rec[:, CW:CW + 64]
        firsts = rec[:, CW + 64:CW + 128].astype(np.int64)
        bits = np.unpackbits(masks.view(np.uint8), bitorder="little").reshape(masks.shape[0], 64, 32)
        cnt = bits.sum(-1)
        assert int(cnt.sum()) == n_lvl, (lvl, int(cnt.sum()), n_lvl)
        # the outputs a row names are consecutive particle indices from its first
        idx = np.concatenate([firsts[t, r] + np.arange(cnt[t, r]) for t in range(rec.shape[0]) for r in range(64)
                              if cnt[t, r]])
        assert np.array_equal(np.sort(idx), np.arange(first, nxt)), lvl
        nblk = rec[:, CW + 129]
        assert np.all((nblk > 0) & (nblk <= 256)), lvl
