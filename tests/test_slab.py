"""z-slab decomposition.

CPU: the slab plan's invariants, the reference-order numpy tree sums against
the reference's own fill_tree (golden vectors), and the whole slab algorithm
over torch.distributed/gloo with world_size 2 and 3 -- owned outputs and tree
nodes bit-identical to the single-domain reference results even though every
entry a rank neither owns nor receives is NaN.

GPU: the same algorithm on device state, several virtual ranks sharing one
B200 (LocalComm), bit-identical to the single-GPU convolve_apr.
"""
import os
import socket

import numpy as np
import pytest
import torch

import goldens as G
import paper_2112_03592_b200 as P
from paper_2112_03592_b200 import _lib as L
from paper_2112_03592_b200.slab import LocalComm, SlabConvolver, SlabPlan, TorchComm
from slab_cpu import CpuRankState, finalize, tree_sums

CASES = ["spheres64", "random_apr_07", "random_apr_09"]


def _plans(d, world, halo=2):
    apr = G.product_apr(d)
    return apr, [SlabPlan.make(apr.access, apr.tree_access, apr.source_dims, world, r, halo) for r in range(world)]


def _owned_mask(plan, which, n):
    m = np.zeros(n, bool)
    for b, e in plan.owned(which):
        m[b:e] = True
    b, e = plan.replicated(which)
    m[b:e] = True
    return m


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("world", [2, 3])
def test_plan_partitions_the_partitioned_levels(name, world):
    d = G.load(name)
    apr, plans = _plans(d, world)
    n = apr.access.particle_count()
    cover = np.zeros(n, np.int32)
    for p in plans:
        for b, e in p.owned("leaf"):
            cover[b:e] += 1
    rb, re_ = plans[0].replicated("leaf")
    cover[rb:re_] += 1
    assert np.all(cover == 1)  # every particle owned exactly once (replicated prefix counted once)
    for src, dst, (b, e) in plans[0].halo_transfers("leaf"):
        assert abs(src - dst) == 1 and 0 <= b < e <= n
    assert plans[0].bounds[0][0] == 0 and plans[-1].bounds[-1][1] == int(apr.source_dims[0])


@pytest.mark.parametrize("name", G.names("random_apr_*") + ["spheres64", "dense16", "c1_256"])
def test_numpy_tree_sums_are_the_reference_fill_tree(name):
    d = G.load(name)
    apr = G.product_apr(d)
    t = apr.tree_access
    vs, ws = np.zeros(t.particle_count()), np.zeros(t.particle_count())
    tree_sums(apr.access, t, apr.source_dims, d["values"], vs, ws, t.l_min, t.l_max)
    assert np.array_equal(G.bits(finalize(vs, ws)), G.bits(d["tree_values"]))


def _slab_worker(rank, world, port, name, q, halo=2):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
        d = G.load(name)
        apr = G.product_apr(d)
        plan = SlabPlan.make(apr.access, apr.tree_access, apr.source_dims, world, rank, halo=2)
        plan.halo = halo  # (a test below shrinks the exchanged halo to show it is needed)
        conv = sorted(k for k in G.conv_names(d))[0]
        levels = G.pyramid_levels(d, conv)
        st = CpuRankState(plan, apr.source_dims, levels, int(d["leaf_l_range"][0]))
        v = d["values"].copy()
        v[~_owned_mask(plan, "leaf", v.size)] = np.nan  # only owned + replicated inputs exist here
        st.values.copy_(torch.from_numpy(v))
        SlabConvolver([st], TorchComm()).convolve(None, int(d[f"conv_{conv}_pad"][0]), L.ACCUM_EXACT)
        own = _owned_mask(plan, "leaf", v.size)
        ok_out = np.array_equal(G.bits(st.out.numpy()[own]), G.bits(d[f"conv_{conv}_out"][own]))
        town = _owned_mask(plan, "tree", d["tree_values"].size)
        ok_tree = np.array_equal(G.bits(st.tree.numpy()[:town.size][town]), G.bits(d["tree_values"][town]))
        q.put((rank, bool(ok_out), bool(ok_tree), int(own.sum())))
        torch.distributed.destroy_process_group()
    except Exception as e:  # report, never hang the parent
        q.put((rank, False, False, repr(e)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_gloo(name, world, halo=2):
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, name, q, halo)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return sorted(res)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("world", [2, 3])
def test_slab_algorithm_gloo_bit_identical(name, world):
    res = _run_gloo(name, world)
    for rank, ok_out, ok_tree, n in res:
        assert ok_out and ok_tree, (rank, ok_out, ok_tree, n)
    assert sum(r[3] for r in res if isinstance(r[3], int)) >= G.load(name)["values"].size


def test_slab_without_halo_is_detected():
    # the NaN poisoning is live: with no halo rows exchanged, boundary outputs go wrong
    res = _run_gloo("spheres64", 2, halo=0)
    assert not all(ok_out for _, ok_out, _, _ in res)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES + ["c1_256"])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("accum", ["exact", "fast"])
def test_slab_gpu_virtual_ranks_bit_identical(name, world, accum):
    from paper_2112_03592_b200.slab import GpuRankState
    d = G.load(name)
    apr = G.product_apr(d)
    try:
        plans = [SlabPlan.make(apr.access, apr.tree_access, apr.source_dims, world, r, halo=2) for r in range(world)]
    except ValueError:
        pytest.skip("volume too thin for this many slabs")
    lr = d["leaf_l_range"]
    conv = "g3" if "conv_g3_out" in d else sorted(G.conv_names(d))[0]
    levels = G.pyramid_levels(d, conv)
    pyr = P.explicit_pyramid([P.Stencil(*k, weights=w) for k, w in levels], int(lr[0]), int(lr[1]))
    pad = int(d[f"conv_{conv}_pad"][0])
    acc = L.ACCUM_EXACT if accum == "exact" else L.ACCUM_FAST
    ref = P.convolve_apr(apr, d["values"], d["tree_values"], pyr, P.PadMode(pad), P.ConvolveOptions(accum=accum))
    ctx = P.default_context()
    stream = torch.cuda.Stream()  # C-ABI calls and the virtual-rank copies share one stream
    torch.cuda.set_stream(stream)
    states = []
    for p in plans:
        dev = P.DeviceApr.upload(ctx, apr)  # each virtual rank: its own handle and tree scratch
        st = GpuRankState(p, dev)
        v = d["values"].copy()
        v[~_owned_mask(p, "leaf", v.size)] = np.nan
        st.values.copy_(torch.from_numpy(v))
        states.append((st, dev))
    dpyr = pyr.device(ctx)
    SlabConvolver([s for s, _ in states], LocalComm()).convolve(dpyr, pad, acc)
    torch.cuda.synchronize()
    for st, dev in states:
        own = _owned_mask(st.plan, "leaf", ref.size)
        assert np.array_equal(G.bits(st.out.cpu().numpy()[:ref.size][own]), G.bits(ref[own])), st.rank
        # a rank's gather maps cover only the tiles its slab computes
        built, n_tiles = dev.map_tiles()
        assert 0 < built <= n_tiles, (st.rank, built, n_tiles)
        if name == "c1_256":  # (the small cases' slabs all touch every tile row)
            assert built < n_tiles, (st.rank, built, n_tiles)
        town = _owned_mask(st.plan, "tree", d["tree_values"].size)
        tv = st.tree.cpu().numpy()[:town.size]
        assert np.array_equal(G.bits(tv[town]), G.bits(d["tree_values"][town])), st.rank


class DeferredComm(LocalComm):
    """Virtual ranks whose halo exchanges only land at wait(): the interior
    pass of exchange_and_convolve runs while every halo entry is still NaN."""

    def exchange_async(self, states, attr, transfers):
        return [lambda: LocalComm.exchange(self, states, attr, transfers)]

    def wait(self, works):
        for w in works:
            w()


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("world", [2, 3])
def test_interior_bands_need_no_halo_cpu(name, world):
    """exchange_and_convolve (interior while the exchange is in flight, then
    the boundary bands) with NaN halos during the interior pass: every owned
    output still equals the reference bit for bit (CPU, C oracle ranks)."""
    d = G.load(name)
    apr, plans = _plans(d, world)
    conv = sorted(k for k in G.conv_names(d))[0]
    levels = G.pyramid_levels(d, conv)
    states = []
    for p in plans:
        st = CpuRankState(p, apr.source_dims, levels, int(d["leaf_l_range"][0]))
        v = d["values"].copy()
        v[~_owned_mask(p, "leaf", v.size)] = np.nan
        st.values.copy_(torch.from_numpy(v))
        states.append(st)
    sc = SlabConvolver(states, DeferredComm())
    sc.fill_tree()
    for st in states:  # the tree halos are NaN too until the exchange lands
        t = st.tree.numpy()
        t[~_owned_mask(st.plan, "tree", t.size)] = np.nan
    sc.exchange_and_convolve(None, int(d[f"conv_{conv}_pad"][0]), L.ACCUM_EXACT)
    for st in states:
        own = _owned_mask(st.plan, "leaf", d["values"].size)
        assert np.array_equal(G.bits(st.out.numpy()[own]), G.bits(d[f"conv_{conv}_out"][own])), st.rank


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES + ["c1_256"])
@pytest.mark.parametrize("world", [2, 4])
def test_interior_bands_need_no_halo_gpu(name, world):
    """The same on device state (aprgpu_convolve_slab_band), virtual ranks."""
    from paper_2112_03592_b200.slab import GpuRankState
    d = G.load(name)
    apr = G.product_apr(d)
    try:
        plans = [SlabPlan.make(apr.access, apr.tree_access, apr.source_dims, world, r, halo=2) for r in range(world)]
    except ValueError:
        pytest.skip("volume too thin for this many slabs")
    a = apr.access
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 5), a.l_min, a.l_max, P.PyramidMode.Restricted)
    tv = P.fill_tree(apr, d["values"])
    ref = P.convolve_apr(apr, d["values"], tv, pyr)
    ctx = P.default_context()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    states = []
    for p in plans:
        dev = P.DeviceApr.upload(ctx, apr)
        st = GpuRankState(p, dev)
        v = d["values"].copy()
        v[~_owned_mask(p, "leaf", v.size)] = np.nan
        st.values.copy_(torch.from_numpy(v))
        states.append((st, dev))
    sts = [s for s, _ in states]
    sc = SlabConvolver(sts, DeferredComm())
    sc.fill_tree()
    for st in sts:
        own_t = torch.from_numpy(_owned_mask(st.plan, "tree", st.tree.numel())).to(st.tree.device)
        st.tree[~own_t] = float("nan")
    sc.exchange_and_convolve(pyr.device(ctx), 1, L.ACCUM_EXACT)
    torch.cuda.synchronize()
    for st in sts:
        own = _owned_mask(st.plan, "leaf", ref.size)
        assert np.array_equal(G.bits(st.out.cpu().numpy()[:ref.size][own]), G.bits(ref[own])), st.rank


@pytest.mark.gpu
def test_restricted_apr_refuses_planes_outside_its_slab():
    """aprgpu_apr_restrict: the per-tile state is built for the slab's tiles
    only, so a convolution reaching outside the slab fails loudly instead of
    reading tiles that were never built; a restriction after the first
    convolution is refused."""
    d = G.load("c1_256")
    apr = G.product_apr(d)
    a = apr.access
    ctx = P.default_context()
    dev = P.DeviceApr.upload(ctx, apr)
    lc = a.l_max - 2
    dev.restrict(lc, 0, 128)
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted).device(ctx)
    tv = P.fill_tree(apr, d["values"])
    with pytest.raises(P.CapabilityError):
        dev.convolve(d["values"], tv, pyr, 1, L.ACCUM_EXACT)  # (the whole volume)
    built, n_tiles = dev.map_tiles()
    assert built < n_tiles
    fresh = P.DeviceApr.upload(ctx, apr)
    fresh.convolve(d["values"], tv, pyr, 1, L.ACCUM_EXACT)
    with pytest.raises(P.RangeError):
        fresh.restrict(lc, 0, 128)
