"""GPU parity tests: the CUDA path (through the C-ABI) against the reference.

Bars:
  * access round trip, device-built interior structure, non-empty row index,
    fill_tree and EXACT-mode convolve_apr / rl_apr: bit-identical to the
    reference (golden vectors from the real reference + the C oracle on fresh
    random inputs);
  * FAST-mode (fp32) convolution: rel <= 1e-5 with scale max(|e|,|g|,1)
    (acceptance.cpp:271-276) for non-negative stencils; rel <= 1e-4 for signed
    random stencils (fp32 accumulation of cancelling terms).
"""
import numpy as np
import pytest

import goldens as G
import paper_2112_03592_b200 as P
from paper_2112_03592_b200 import _lib as L
from pyoracle import Oracle

pytestmark = pytest.mark.gpu
ORC = Oracle()

STRUCT_CASES = G.names("random_apr_*") + G.names("blobs32_*") + ["spheres64", "dense16", "c1_256"]


def golden_pyramid(d, name):
    levels = G.pyramid_levels(d, name)
    lr = d["leaf_l_range"]
    return P.explicit_pyramid([P.Stencil(*k, weights=w) for k, w in levels], int(lr[0]), int(lr[1]))


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    s = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)
    return float(np.max(np.abs(a - b) / s)) if a.size else 0.0


@pytest.mark.parametrize("name", STRUCT_CASES)
def test_access_round_trip_and_device_tree(name):
    d = G.load(name)
    apr = G.product_apr(d, with_tree=True)
    dev = P.DeviceApr.upload(P.default_context(), apr)
    leaf = dev.download(L.LEAF)
    tree = dev.download(L.TREE)
    assert leaf.equals(apr.access)
    assert tree.equals(apr.tree_access)
    # interior structure built on the GPU == init_tree_structure (tree.hpp:26-82)
    apr2 = G.product_apr(d, with_tree=False)
    dev2 = P.DeviceApr.upload(P.default_context(), apr2)
    assert dev2.download(L.TREE).equals(apr.tree_access)


@pytest.mark.parametrize("name", STRUCT_CASES)
def test_row_index_bit_exact(name):
    d = G.load(name)
    apr = G.product_apr(d)
    dev = apr.device()
    off = 0
    for i, l in enumerate(range(apr.access.l_min, apr.access.l_max + 1)):
        z, x, y0, y1 = dev.row_index(l)
        n = int(d["rows_count"][i])
        assert z.size == n
        assert np.array_equal(z, d["rows_z"][off:off + n])
        assert np.array_equal(x, d["rows_x"][off:off + n])
        assert np.array_equal(y0, d["rows_ymin"][off:off + n])
        assert np.array_equal(y1, d["rows_ymax"][off:off + n])
        off += n


@pytest.mark.parametrize("name", STRUCT_CASES)
def test_fill_tree_bit_exact(name):
    d = G.load(name)
    apr = G.product_apr(d)
    tv = P.fill_tree(apr, d["values"])
    assert np.array_equal(G.bits(tv), G.bits(d["tree_values"]))


@pytest.fixture(params=["map", "reconstruct"])
def tile_path(request, monkeypatch):
    """Both box-tile paths: the resident gather map (default) and the per-call
    reconstruction (APRGPU_TILE_MAP=0, conv_tile.cu)."""
    monkeypatch.setenv("APRGPU_TILE_MAP", "1" if request.param == "map" else "0")
    return request.param


@pytest.mark.parametrize("name", STRUCT_CASES)
def test_convolve_exact_bit_identical_to_reference(name, tile_path):
    d = G.load(name)
    apr = G.product_apr(d)
    for c in G.conv_names(d):
        pyr = golden_pyramid(d, c)
        pad = P.PadMode(int(d[f"conv_{c}_pad"][0]))
        out = P.convolve_apr(apr, d["values"], d["tree_values"], pyr, pad)
        ref = d[f"conv_{c}_out"]
        assert np.array_equal(G.bits(out), G.bits(ref)), (c, int(np.sum(G.bits(out) != G.bits(ref))))


@pytest.mark.parametrize("name", ["spheres64", "c1_256", "dense16"] + G.names("random_apr_0*")[:4])
def test_convolve_fast_within_tolerance(name):
    d = G.load(name)
    apr = G.product_apr(d)
    for c in G.conv_names(d):
        pyr = golden_pyramid(d, c)
        pad = P.PadMode(int(d[f"conv_{c}_pad"][0]))
        out = P.convolve_apr(apr, d["values"], d["tree_values"], pyr, pad, P.ConvolveOptions(accum="fast"))
        # fp32 accumulation: 1e-5 for non-negative stencils (the reference's own
        # bound), 1e-4 for signed random stencils up to 5^3, 1e-3 for signed 13^3
        # (2197 cancelling fp32 terms)
        tol = 1e-5 if c.startswith("g") else (1e-3 if "13" in c else 1e-4)
        assert rel_err(out, d[f"conv_{c}_out"]) <= tol, c


@pytest.mark.parametrize("name", ["spheres64", "c1_256", "dense16", "blobs32_0"] + G.names("random_apr_*")[::4])
def test_map_and_reconstruction_paths_bit_identical(name, monkeypatch):
    d = G.load(name)
    apr = G.product_apr(d)
    rng = np.random.default_rng(7)
    v = rng.uniform(0, 1000, d["values"].size).astype(np.float32)
    tv = P.fill_tree(apr, v)
    for k in (3, 5):
        w = P.Stencil(k, k, k, weights=rng.uniform(0, 1, k ** 3))
        pyr = P.make_pyramid(w, apr.access.l_min, apr.access.l_max, P.PyramidMode.Restricted)
        for pad in (P.PadMode.Zero, P.PadMode.Reflect):
            for accum in ("exact", "fast"):
                out = {}
                for path in ("1", "0"):
                    monkeypatch.setenv("APRGPU_TILE_MAP", path)
                    out[path] = P.convolve_apr(apr, v, tv, pyr, pad, P.ConvolveOptions(accum=accum))
                assert np.array_equal(G.bits(out["1"]), G.bits(out["0"])), (k, pad, accum)


def _dense_apr(nz, nx, ny):
    """Every pixel a finest-level particle (CR = 1): full tiles, all 256 output
    blocks active (the acceptance criterion 4 degeneracy, at tile scale)."""
    l_max = max(int(np.ceil(np.log2(max(nz, nx, ny)))), 1)
    dims = [[-(-d // (1 << (l_max - l))) for d in (nz, nx, ny)] for l in range(l_max + 1)]
    l_min = 1
    rows = sum(dims[l][0] * dims[l][1] for l in range(l_min, l_max + 1))
    level_offset = np.zeros(l_max + 1, np.uint64)
    off = 0
    for l in range(l_min, l_max + 1):
        level_offset[l] = off
        off += dims[l][0] * dims[l][1]
    counts = np.zeros(rows, np.int64)
    counts[int(level_offset[l_max]):] = ny
    xz_end = np.cumsum(counts).astype(np.uint64)
    y = np.tile(np.arange(ny, dtype=np.uint16), nz * nx)
    z_dim, x_dim, y_dim = (np.array([d[i] for d in dims], np.int32) for i in range(3))
    return P.APR(P.LinearAccess(l_min, l_max, z_dim, x_dim, y_dim, y, xz_end, level_offset), None, (nz, nx, ny))


@pytest.mark.parametrize("shape", [(64, 64, 64), (40, 24, 70)])
def test_dense_apr_all_blocks_active(shape, tile_path):
    apr = _dense_apr(*shape)
    assert P.validate(apr).ok
    rng = np.random.default_rng(4)
    v = rng.uniform(0, 100, apr.access.particle_count()).astype(np.float32)
    tv = P.fill_tree(apr, v)
    leaf, tree = G.as_oracle(apr.access), G.as_oracle(apr.tree_access)
    for k in (3, 5):
        pyr = P.make_pyramid(P.gaussian_stencil(1.0, k), apr.access.l_min, apr.access.l_max, P.PyramidMode.Restricted)
        levels = [((s.kz, s.kx, s.ky), s.weights) for s in pyr.stencils]
        for pad in (P.PadMode.Zero, P.PadMode.Reflect):
            got = P.convolve_apr(apr, v, tv, pyr, pad)
            exp = ORC.convolve(leaf, tree, v, tv, levels, apr.access.l_min, int(pad))
            assert np.array_equal(G.bits(got), G.bits(exp)), (shape, k, pad)


@pytest.mark.parametrize("name", ["rl_spheres64"])
def test_rl_apr_bit_exact(name):
    d = G.load(name)
    apr = G.product_apr(d)
    for k in (3, 5):
        cfg = P.RLConfig(iterations=10, psf=P.Stencil(k, k, k, weights=d[f"rl_g{k}_psf"]))
        out = P.rl_apr(apr, d["values"], cfg)
        assert np.array_equal(G.bits(out), G.bits(d[f"rl_g{k}_out"])), k


def test_rl_apr_observer_bit_exact():
    """rl_apr with an observer (deconv.hpp:103-104): the device iteration is
    resumed every record_metrics_every iterations; the final estimate and every
    observed estimate equal uninterrupted runs of that many iterations."""
    d = G.load("rl_spheres64")
    apr = G.product_apr(d)
    psf = P.Stencil(3, 3, 3, weights=d["rl_g3_psf"])
    seen = []
    cfg = P.RLConfig(iterations=10, psf=psf, record_metrics_every=3)
    out = P.rl_apr(apr, d["values"], cfg, observer=lambda k, est: seen.append((k, est.copy())))
    assert [k for k, _ in seen] == [3, 6, 9]
    assert np.array_equal(G.bits(out), G.bits(d["rl_g3_out"]))
    for k, est in seen:
        ref = P.rl_apr(apr, d["values"], P.RLConfig(iterations=k, psf=psf))
        assert np.array_equal(G.bits(est), G.bits(ref)), k


def test_rl_resume_in_place_device():
    """aprgpu_rl_resume with estimate_in == out on device pointers (an in-place
    resume) continues from the running estimate: 4 + 6 iterations == 10."""
    import torch
    from paper_2112_03592_b200.aprkit import _ptr
    d = G.load("rl_spheres64")
    apr = G.product_apr(d)
    dev = apr.device()
    psf = P.Stencil(3, 3, 3, weights=d["rl_g3_psf"])
    obs = torch.from_numpy(np.ascontiguousarray(d["values"], np.float32)).cuda()
    est = torch.empty_like(obs)
    s = torch.cuda.current_stream().cuda_stream or None
    dev.rl_ptr(obs.data_ptr(), psf, 4, 0.0, L.ACCUM_EXACT, est.data_ptr(), s or 0)
    L.check(L.lib().aprgpu_rl_resume(dev.handle, obs.data_ptr(), est.data_ptr(), _ptr(psf.weights),
                                     3, 3, 3, 6, 0.0, L.ACCUM_EXACT, est.data_ptr(), L.DEVICE, s))
    torch.cuda.synchronize()
    assert np.array_equal(G.bits(est.cpu().numpy()), G.bits(d["rl_g3_out"]))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_values_and_stencils_vs_oracle(seed):
    """Fresh random values / stencils (incl. anisotropic, 7^3, 13^3, zero pad)
    on the committed structures, checked against the C oracle bit-for-bit."""
    rng = np.random.default_rng(seed)
    for name in G.names("random_apr_*")[seed::3] + ["spheres64"]:
        d = G.load(name)
        apr = G.product_apr(d)
        leaf, tree = G.oracle_access(d, "leaf_"), G.oracle_access(d, "tree_")
        dims = tuple(int(v) for v in d["dims"])
        v = rng.uniform(-1000, 1000, leaf.y_idx.size).astype(np.float32)
        tv = P.fill_tree(apr, v)
        assert np.array_equal(G.bits(tv), G.bits(ORC.fill_tree(leaf, tree, dims, v)))
        for k3 in ((3, 3, 3), (5, 5, 5), (1, 3, 5), (7, 7, 7), (3, 5, 1)):
            w = P.Stencil(*k3, weights=rng.uniform(-1, 1, int(np.prod(k3))))
            for mode in (P.PyramidMode.Restricted, P.PyramidMode.Uniform):
                pyr = P.make_pyramid(w, leaf.l_min, leaf.l_max, mode)
                levels = [((s.kz, s.kx, s.ky), s.weights) for s in pyr.stencils]
                for pad in (P.PadMode.Zero, P.PadMode.Reflect):
                    got = P.convolve_apr(apr, v, tv, pyr, pad)
                    exp = ORC.convolve(leaf, tree, v, tv, levels, leaf.l_min, int(pad))
                    assert np.array_equal(G.bits(got), G.bits(exp)), (name, k3, mode, pad)


def test_thirteen_cubed_and_determinism():
    d = G.load("random_apr_03")
    apr = G.product_apr(d)
    rng = np.random.default_rng(13)
    w = P.Stencil(13, 13, 13, weights=rng.uniform(-1, 1, 13 ** 3))
    pyr = P.make_pyramid(w, apr.access.l_min, apr.access.l_max, P.PyramidMode.Restricted)
    a = P.convolve_apr(apr, d["values"], d["tree_values"], pyr)
    b = P.convolve_apr(apr, d["values"], d["tree_values"], pyr, opt=P.ConvolveOptions(use_row_skip=False, threads=3))
    assert np.array_equal(G.bits(a), G.bits(b))
    leaf, tree = G.oracle_access(d, "leaf_"), G.oracle_access(d, "tree_")
    levels = [((s.kz, s.kx, s.ky), s.weights) for s in pyr.stencils]
    exp = ORC.convolve(leaf, tree, d["values"], d["tree_values"], levels, leaf.l_min, 1)
    assert np.array_equal(G.bits(a), G.bits(exp))


def test_errors_map_to_reference_exceptions():
    d = G.load("random_apr_00")
    apr = G.product_apr(d)
    lr = d["leaf_l_range"]
    # pyramid not covering the levels -> RangeError (convolve.hpp:224-225)
    short = P.make_pyramid(P.gaussian_stencil(1.0, 3), int(lr[0]) + 1, int(lr[1]), P.PyramidMode.Restricted)
    with pytest.raises(P.RangeError):
        P.convolve_apr(apr, d["values"], d["tree_values"], short)
    # extent 15 -> CapabilityError (convolve.hpp:226-230, test_convolve.cpp:167-178)
    big = P.make_pyramid(P.Stencil(15, 3, 3), int(lr[0]), int(lr[1]), P.PyramidMode.Uniform)
    with pytest.raises(P.CapabilityError):
        P.convolve_apr(apr, d["values"], d["tree_values"], big)
    # the C-ABI itself also refuses (no Python pre-check)
    dev = apr.device()
    with pytest.raises(P.CapabilityError):
        dev.convolve(d["values"], d["tree_values"], big.device(dev.ctx), 1, L.ACCUM_EXACT)
    # an interior structure with a missing parent -> IntegrityError (tree.hpp:98-100)
    bad = G.product_apr(d)
    t = bad.tree_access
    if t.y_idx.size:
        # the finest interior level that holds nodes
        lvl = next(l for l in range(t.l_max, t.l_min - 1, -1)
                   if (int(t.xz_end[-1]) if l == t.l_max else int(t.xz_end[int(t.level_offset[l + 1]) - 1]))
                   > (int(t.xz_end[int(t.level_offset[l]) - 1]) if int(t.level_offset[l]) else 0))
        r0 = int(t.level_offset[lvl])
        b = int(t.xz_end[r0 - 1]) if r0 else 0
        # drop the first node of that level by shifting the row ends
        ye = t.y_idx.copy()
        xz = t.xz_end.copy()
        first_row = next(r for r in range(r0, xz.size) if int(xz[r]) > b)
        ye = np.delete(ye, b)
        xz[first_row:] -= 1
        bad.tree_access = P.LinearAccess(t.l_min, t.l_max, t.z_dim, t.x_dim, t.y_dim, ye, xz, t.level_offset)
        with pytest.raises(P.IntegrityError):
            P.DeviceApr.upload(P.default_context(), bad)


def test_device_pointer_path_with_torch():
    torch = pytest.importorskip("torch")
    d = G.load("spheres64")
    apr = G.product_apr(d)
    dev = apr.device()
    pyr = golden_pyramid(d, "g3").device(dev.ctx)
    v = torch.from_numpy(d["values"]).cuda()
    tv = torch.empty(dev.n_tree, dtype=torch.float32, device="cuda")
    out = torch.empty(dev.n_particles, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    s = st.cuda_stream
    dev.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
    dev.convolve_ptr(v.data_ptr(), tv.data_ptr(), pyr, 1, L.ACCUM_EXACT, out.data_ptr(), s)
    torch.cuda.synchronize()
    assert np.array_equal(G.bits(tv.cpu().numpy()), G.bits(d["tree_values"]))
    assert np.array_equal(G.bits(out.cpu().numpy()), G.bits(d["conv_g3_out"]))
    assert dev.ctx.launch_count() > 0


def test_nonempty_row_index_and_init_tree_front_doors():
    d = G.load("random_apr_05")
    apr = G.product_apr(d)
    idx = P.nonempty_row_index(apr.access, apr.source_dims)
    off = 0
    for i, rows in enumerate(idx):
        n = int(d["rows_count"][i])
        assert len(rows) == n
        for j, r in enumerate(rows):
            assert (r.z, r.x, r.y_min, r.y_max) == (d["rows_z"][off + j], d["rows_x"][off + j],
                                                    d["rows_ymin"][off + j], d["rows_ymax"][off + j])
        off += n
    t = P.init_tree_structure(apr.access, apr.source_dims)
    assert t.equals(apr.tree_access)


@pytest.mark.parametrize("name", ["c1_256", "spheres64", "random_apr_03", "random_apr_09", "dense16", "C3"])
def test_rebuild_index_equals_upload_lists(name, monkeypatch):
    """aprgpu_rebuild_index (the paper protocol's per-call index step): the
    non-empty row lists and occupied-tile lists it recomputes equal the ones
    built at upload (APRGPU_VERIFY_INDEX=1 compares them in the library)."""
    monkeypatch.setenv("APRGPU_VERIFY_INDEX", "1")
    import subprocess
    import sys
    if name == "C3":  # (BASELINE config 3, built on the device)
        make = ("from paper_2112_03592_b200 import synth; a=synth.build_spheres_apr(1024, count=48, rmin=24.0, "
                "rmax=80.0, blur=2.0, seed=42, rel_error=0.1)[0].device(); ")
    else:
        make = "import goldens as G; a=G.product_apr(G.load(%r)).device(); " % name
    code = ("import sys; sys.path[:0]=['tests','.']; " + make +
            "a.rebuild_index_ptr(0); import torch; torch.cuda.synchronize(); print('ok')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
