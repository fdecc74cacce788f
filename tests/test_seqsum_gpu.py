"""rl_apr's observation sum replayed on the device (csrc/seqsum.cu).

The reference sums the clamped observations in one sequential double loop
(deconv.hpp:90-91), rounding after every addition.  When those partial sums
are not provably exact (C4's 548 M observations) aprgpu_rl_resume replays the
loop in parallel on the device: binade by binade, each element an increment
map in units of the running sum's ulp (round-half-even ties depend on the
running sum's parity), chunks composed in order, and the chunk where the sum
leaves its binade replayed by plain additions.  The result must equal the
sequential loop bit for bit; numpy's add.accumulate over float64 IS that loop
(a plain left-to-right accumulation, unlike np.sum's pairwise reduction).
"""
import ctypes as C

import numpy as np
import pytest

import paper_2112_03592_b200 as P
from paper_2112_03592_b200 import _lib as L
from paper_2112_03592_b200.errors import RangeError

pytestmark = pytest.mark.gpu


def seq_ref(x):
    x = np.ascontiguousarray(x, np.float32)
    # (the loop starts from +0.0: an all -0.0 input sums to +0.0)
    return float(np.add.accumulate(np.concatenate([[0.0], x.astype(np.float64)]))[-1])


def seq_dev(x, device=True):
    import torch
    ctx = P.default_context(0)
    x = np.ascontiguousarray(x, np.float32)
    out = C.c_double()
    if device and x.size:
        t = torch.from_numpy(x).cuda()
        L.check(L.lib().aprgpu_sequential_sum(ctx.handle, t.data_ptr(), x.size, L.DEVICE, C.byref(out), None))
    else:
        L.check(L.lib().aprgpu_sequential_sum(ctx.handle, x.ctypes.data if x.size else None, x.size, L.HOST,
                                              C.byref(out), None))
    return out.value


def cases():
    rng = np.random.default_rng(7)
    yield "empty", np.zeros(0, np.float32)
    yield "one", np.array([3.25], np.float32)
    yield "zeros", np.zeros(10_000, np.float32)
    yield "neg_zero", np.full(5000, -0.0, np.float32)
    yield "uniform_1e6", rng.random(1_000_000, dtype=np.float32)
    yield "ragged", rng.random(2048 * 37 + 11, dtype=np.float32) * 1000
    yield "wide_range", np.exp(rng.normal(0, 12, 3_000_000)).astype(np.float32)
    # long zero prefix, then a tiny first value, then large ones (many binades)
    z = np.zeros(300_000, np.float32)
    z[123_456] = np.float32(1e-38)
    z[200_000:] = rng.random(100_000, dtype=np.float32) * 1e6
    yield "zero_prefix_tiny_start", z
    # exact ties: 1.0 then many half-ulps of 1.0 (2^-53) and odd multiples of them
    t = np.full(200_000, np.float32(2.0 ** -53), np.float32)
    t[0] = 1.0
    t[1::7] = np.float32(3 * 2.0 ** -53)
    t[2::11] = np.float32(2.0 ** -52)
    yield "ties", t
    # ties at a larger scale, across binade changes
    k = rng.integers(0, 4, 500_000)
    yield "ties_scaled", (np.float32(2.0 ** 20) + k.astype(np.float32)) * np.float32(2.0 ** -31)
    # C4-like: 20 M observations ~ O(100) with fine low bits (the exact bound fails)
    yield "c4_like_20m", (rng.random(20_000_000, dtype=np.float32) * 300).astype(np.float32)


@pytest.mark.parametrize("name,x", list(cases()), ids=[c[0] for c in cases()])
def test_sequential_sum_bit_exact(name, x):
    ref = seq_ref(x)
    got = seq_dev(x)
    assert np.float64(got).view(np.uint64) == np.float64(ref).view(np.uint64), (name, got, ref)


def test_sequential_sum_python_loop():
    """A pure-Python left-to-right loop on a small adversarial case (independent of numpy)."""
    rng = np.random.default_rng(3)
    x = np.concatenate([np.exp(rng.normal(0, 20, 50_000)), rng.random(50_000) * 2.0 ** -40]).astype(np.float32)
    rng.shuffle(x)
    s = 0.0
    for v in x.tolist():
        s += v
    assert seq_dev(x, device=False) == s


def test_sequential_sum_rejects():
    with pytest.raises(RangeError):
        seq_dev(np.array([1.0, -1.0], np.float32))
    with pytest.raises(RangeError):
        seq_dev(np.array([1.0, np.nan], np.float32))


def test_rl_mean_replay_vs_reference():
    """rl_apr on observations whose partial sums round (values spread over 2^+-40,
    so the order-free exact sum is not provable and the device replay runs):
    bit-identical to the reference's rl_apr."""
    import goldens as G
    from pyoracle import Ref, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    d = G.load("rl_spheres64")
    apr = G.product_apr(d)
    rng = np.random.default_rng(11)
    obs = (d["values"].astype(np.float64) * np.exp2(rng.integers(-40, 40, d["values"].size))).astype(np.float32)
    R = Ref()
    rapr = R.apr_from_arrays(apr.access, apr.source_dims)
    k3, w = R.gaussian_stencil(1.0, 3)
    ref = R.rl_apr(rapr, obs, w, k3, 3)
    got = P.rl_apr(apr, obs, P.RLConfig(iterations=3, psf=P.Stencil(3, 3, 3, weights=w)))
    assert np.array_equal(np.asarray(got, np.float32).view(np.uint32), np.asarray(ref, np.float32).view(np.uint32))
