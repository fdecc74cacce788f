"""Concurrent calls (inputs immutable, safe for concurrent reads):
several host threads calling fill_tree / convolve_apr on ONE fresh APR (so the
lazy per-APR caches -- child links, level starts, gather maps -- are built
under contention), and pipelined host-pointer calls sharing one context.
Every result must equal the serial one bit for bit."""
import threading

import numpy as np
import pytest

import goldens as G
import paper_2112_03592_b200 as P
from paper_2112_03592_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _run_threads(fn, n):
    out, errs = [None] * n, []

    def work(i):
        try:
            out[i] = fn(i)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    return out


@pytest.mark.parametrize("name", ["spheres64", "c1_256"])
def test_concurrent_fill_and_convolve_on_one_apr(name):
    d = G.load(name)
    rng = np.random.default_rng(3)
    serial_apr = G.product_apr(d)
    values = rng.uniform(0, 100, serial_apr.access.particle_count()).astype(np.float32)
    tv0 = P.fill_tree(serial_apr, values)
    a = serial_apr.access
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted)
    out0 = P.convolve_apr(serial_apr, values, tv0, pyr)
    fresh = G.product_apr(d)  # uploaded, nothing else cached: the threads race to build the lazy caches
    fresh.device()
    pyr.device()

    def job(i):
        tv = P.fill_tree(fresh, values)
        return tv, P.convolve_apr(fresh, values, tv, pyr)

    for tv, out in _run_threads(job, 6):
        assert np.array_equal(G.bits(tv), G.bits(tv0))
        assert np.array_equal(G.bits(out), G.bits(out0))


def test_concurrent_pipelined_host_calls(monkeypatch):
    import torch
    monkeypatch.setenv("APRGPU_HOST_PIPELINE_MIN", "0")
    d = G.load("c1_256")
    apr = G.product_apr(d)
    dev = apr.device()
    a = apr.access
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted)
    pyr.device(dev.ctx)
    rng = np.random.default_rng(5)
    vals = [rng.uniform(0, 10, a.particle_count()).astype(np.float32) for _ in range(4)]
    trees = [P.fill_tree(apr, v) for v in vals]
    exp = [P.convolve_apr(apr, v, t, pyr) for v, t in zip(vals, trees)]
    # one APR handle per thread (the staging buffers are per APR), one shared context
    devs = [G.product_apr(d).device(dev.ctx) for _ in range(4)]

    def job(i):
        hv = torch.from_numpy(vals[i]).pin_memory()
        ht = torch.from_numpy(trees[i]).pin_memory()
        ho = torch.empty(a.particle_count(), dtype=torch.float32).pin_memory()
        dp = pyr.device(devs[i].ctx)
        L.check(L.lib().aprgpu_convolve(devs[i].handle, hv.data_ptr(), ht.data_ptr(), dp.handle, 1, L.ACCUM_EXACT,
                                        ho.data_ptr(), L.HOST, None))
        return ho.numpy().copy()

    for i, got in enumerate(_run_threads(job, 4)):
        assert np.array_equal(G.bits(got), G.bits(exp[i])), i


@pytest.mark.parametrize("name", ["c1_256"])
def test_concurrent_device_pointer_convolve_fresh_apr(name):
    """Device-pointer convolve_apr (no per-APR scratch, no lock on the hot
    path) from 6 threads, each on its own stream, against a FRESH APR: the
    threads race to build the gather maps; a thread must never launch on a
    map another thread has allocated but not yet built."""
    import torch
    d = G.load(name)
    rng = np.random.default_rng(11)
    ref_apr = G.product_apr(d)
    values = rng.uniform(0, 100, ref_apr.access.particle_count()).astype(np.float32)
    tv = P.fill_tree(ref_apr, values)
    a = ref_apr.access
    exp = {}
    for k in (3, 5):
        pyr = P.make_pyramid(P.gaussian_stencil(1.0, k), a.l_min, a.l_max, P.PyramidMode.Restricted)
        exp[k] = (pyr, P.convolve_apr(ref_apr, values, tv, pyr))
    fresh = G.product_apr(d).device()
    dv = torch.from_numpy(values).cuda()
    dt = torch.from_numpy(tv).cuda()
    pyrs = {k: p.device(fresh.ctx) for k, (p, _) in exp.items()}
    torch.cuda.synchronize()

    def job(i):
        k = 3 if i % 2 == 0 else 5
        st = torch.cuda.Stream()
        out = torch.full((fresh.n_particles,), float("nan"), device="cuda")
        torch.cuda.synchronize()
        fresh.convolve_ptr(dv.data_ptr(), dt.data_ptr(), pyrs[k], 1, L.ACCUM_EXACT, out.data_ptr(), st.cuda_stream)
        st.synchronize()
        return k, out.cpu().numpy()

    for k, got in _run_threads(job, 6):
        assert np.array_equal(G.bits(got), G.bits(exp[k][1])), k


@pytest.mark.parametrize("name", ["spheres64", "c1_256"])
def test_index_step_beside_fill_tree(name):
    """The paper protocol's index step (aprgpu_rebuild_index, its own scratch
    guard) on one stream while fill_tree + convolve_apr run on another, as
    bench.py's paper step does: the tree values and outputs stay bit-identical
    to the reference golden ones."""
    import torch
    d = G.load(name)
    apr = G.product_apr(d)
    a = apr.access
    dev = apr.device()
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted).device(dev.ctx)
    v = torch.from_numpy(np.ascontiguousarray(d["values"], np.float32)).cuda()
    tv = torch.empty(max(dev.n_tree, 1), dtype=torch.float32, device="cuda")
    out = torch.empty(dev.n_particles, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ref = None
    for i in range(20):
        tv.fill_(float("nan"))
        dev.rebuild_index_ptr(s2.cuda_stream)
        dev.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s1.cuda_stream)
        dev.convolve_ptr(v.data_ptr(), tv.data_ptr(), pyr, 1, L.ACCUM_EXACT, out.data_ptr(), s1.cuda_stream)
        torch.cuda.synchronize()
        t = tv.cpu().numpy()[:dev.n_tree]
        assert np.array_equal(G.bits(t), G.bits(d["tree_values"])), i
        o = out.cpu().numpy()
        if ref is None:
            ref = o.copy()
        assert np.array_equal(G.bits(o), G.bits(ref)), i
