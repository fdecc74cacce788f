"""Host-pointer convolve_apr pipelined over z-chunks (api.cu,
convolve_host_pipelined): with page-locked buffers the copies stream per chunk
on two copy streams around per-chunk (Slab-restricted) passes; pageable
buffers (numpy arrays here, std::vector in the C++ drop-in) are staged through
pinned memory by the context's worker threads.  The result must
be bit-identical to the device-pointer call, for every chunk count, both
accumulation modes, the map and reconstruction tile paths, and the generic
row kernel (anisotropic / 13^3 stencils)."""
import numpy as np
import pytest

import goldens as G
import paper_2112_03592_b200 as P
from paper_2112_03592_b200 import _lib as L

pytestmark = pytest.mark.gpu

CASES = ["spheres64", "c1_256", "blobs32_0", "random_apr_03", "dense16"]


def _host_call(dev, values, tree, dpyr, pad, accum):
    import torch
    hv = torch.from_numpy(np.ascontiguousarray(values, np.float32)).pin_memory()
    ht = torch.from_numpy(np.ascontiguousarray(tree, np.float32) if tree.size else np.zeros(1, np.float32)).pin_memory()
    ho = torch.empty(dev.n_particles, dtype=torch.float32).pin_memory()
    L.check(L.lib().aprgpu_convolve(dev.handle, hv.data_ptr(), ht.data_ptr() if tree.size else None, dpyr.handle,
                                    int(pad), accum, ho.data_ptr(), L.HOST, None))
    return ho.numpy().copy()


def _pageable_call(dev, values, tree, dpyr, pad, accum):
    hv = np.ascontiguousarray(values, np.float32)
    ht = np.ascontiguousarray(tree, np.float32)
    ho = np.full(dev.n_particles, np.nan, np.float32)
    L.check(L.lib().aprgpu_convolve(dev.handle, hv.ctypes.data, ht.ctypes.data if ht.size else None, dpyr.handle,
                                    int(pad), accum, ho.ctypes.data, L.HOST, None))
    return ho


def _mixed_call(dev, values, tree, dpyr, pad, accum, pinned_out):
    """Per-array staging: pageable inputs with a page-locked output (the C++
    drop-in's convolve_apr), or page-locked inputs with a pageable output."""
    import torch
    if pinned_out:
        hv = np.ascontiguousarray(values, np.float32)
        ht = np.ascontiguousarray(tree, np.float32)
        vp, tp = hv.ctypes.data, (ht.ctypes.data if ht.size else None)
        ho = torch.full((dev.n_particles,), float("nan"), dtype=torch.float32).pin_memory()
        op = ho.data_ptr()
    else:
        hv = torch.from_numpy(np.ascontiguousarray(values, np.float32)).pin_memory()
        ht = torch.from_numpy(np.ascontiguousarray(tree, np.float32) if tree.size else np.zeros(1, np.float32)).pin_memory()
        vp, tp = hv.data_ptr(), (ht.data_ptr() if tree.size else None)
        ho = np.full(dev.n_particles, np.nan, np.float32)
        op = ho.ctypes.data
    L.check(L.lib().aprgpu_convolve(dev.handle, vp, tp, dpyr.handle, int(pad), accum, op, L.HOST, None))
    return ho.numpy().copy() if pinned_out else ho


def _device_call(dev, values, tree, dpyr, pad, accum):
    import torch
    v = torch.from_numpy(np.ascontiguousarray(values, np.float32)).cuda()
    t = torch.from_numpy(np.ascontiguousarray(tree, np.float32) if tree.size else np.zeros(1, np.float32)).cuda()
    o = torch.empty(dev.n_particles, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    dev.convolve_ptr(v.data_ptr(), t.data_ptr(), dpyr, int(pad), accum, o.data_ptr(), s)
    torch.cuda.synchronize()
    return o.cpu().numpy()


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("chunks", ["2", "3", "8"])
def test_pipelined_host_convolve_bit_identical(name, chunks, monkeypatch):
    monkeypatch.setenv("APRGPU_HOST_PIPELINE_MIN", "0")
    monkeypatch.setenv("APRGPU_HOST_CHUNKS", chunks)
    d = G.load(name)
    apr = G.product_apr(d)
    a = apr.access
    dev = apr.device()
    rng = np.random.default_rng(7)
    values = rng.uniform(0.0, 10.0, a.particle_count()).astype(np.float32)
    tree = P.fill_tree(apr, values)
    stencils = [P.gaussian_stencil(1.0, 3), P.gaussian_stencil(1.0, 5),
                P.Stencil(5, 3, 5, weights=rng.uniform(-1, 1, 75).astype(np.float32))]
    for w in stencils:
        pyr = P.make_pyramid(w, a.l_min, a.l_max, P.PyramidMode.Restricted)
        dpyr = pyr.device(dev.ctx)
        for accum in (L.ACCUM_EXACT, L.ACCUM_FAST):
            for pad in (P.PadMode.Reflect, P.PadMode.Zero):
                for path in ("1", "0"):
                    monkeypatch.setenv("APRGPU_TILE_MAP", path)
                    got = _host_call(dev, values, tree, dpyr, pad, accum)
                    exp = _device_call(dev, values, tree, dpyr, pad, accum)
                    assert np.array_equal(G.bits(got), G.bits(exp)), (w.kz, accum, int(pad), path)
                    got = _pageable_call(dev, values, tree, dpyr, pad, accum)
                    assert np.array_equal(G.bits(got), G.bits(exp)), ("pageable", w.kz, accum, int(pad), path)
                    for po in (True, False):
                        got = _mixed_call(dev, values, tree, dpyr, pad, accum, po)
                        assert np.array_equal(G.bits(got), G.bits(exp)), ("mixed", po, w.kz, accum, int(pad), path)


def test_pipelined_host_convolve_c3(monkeypatch):
    """C3 at full size, default chunking (8), against the device call."""
    from paper_2112_03592_b200 import synth
    apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
    dev = apr.device()
    tree = P.fill_tree(apr, values)
    for k in (3, 5):
        pyr = P.make_pyramid(P.gaussian_stencil(1.0, k), apr.access.l_min, apr.access.l_max, P.PyramidMode.Restricted)
        dpyr = pyr.device(dev.ctx)
        for accum in (L.ACCUM_FAST, L.ACCUM_EXACT):
            got = _host_call(dev, values, tree, dpyr, P.PadMode.Reflect, accum)
            exp = _device_call(dev, values, tree, dpyr, P.PadMode.Reflect, accum)
            assert np.array_equal(G.bits(got), G.bits(exp)), (k, accum)
            got = _pageable_call(dev, values, tree, dpyr, P.PadMode.Reflect, accum)
            assert np.array_equal(G.bits(got), G.bits(exp)), ("pageable", k, accum)
            got = _mixed_call(dev, values, tree, dpyr, P.PadMode.Reflect, accum, True)
            assert np.array_equal(G.bits(got), G.bits(exp)), ("mixed", k, accum)
