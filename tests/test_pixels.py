"""Dense pixel convolution (convolve.hpp:48-98), the pixel
baseline of the paper's APR-vs-pixels comparison.  Golden outputs from the real
reference (tests/golden/make_pixels_golden.py): 3^3 / 5^3 Gaussians, signed
5x3x1, 7^3 and 13^3 stencils, a stencil with zero weights, both pads, on a
reconstructed image, a random volume and a one-plane volume.  CPU: the C
oracle against them; GPU: the device kernel, EXACT bit-identical and FAST
within the reference's tolerance (acceptance.cpp:271-276 scale).
"""
import numpy as np
import pytest

import goldens as G
from pyoracle import Oracle

ORC = Oracle()
PIX = G.load("pixels")
KEYS = sorted(k for k in PIX if "__p" in k and not k.endswith(("_k3", "_w")))


def _case(key):
    vol = PIX[key.split("__")[0] + "__vol"]
    return vol, PIX[key + "_w"], tuple(int(v) for v in PIX[key + "_k3"]), int(key[-1])


@pytest.mark.parametrize("key", KEYS)
def test_oracle_convolve_pixels_matches_reference(key):
    vol, w, k3, pad = _case(key)
    assert np.array_equal(G.bits(ORC.convolve_pixels(vol, w, k3, pad)), G.bits(PIX[key]))


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_device_convolve_pixels(key):
    import paper_2112_03592_b200 as P
    vol, w, k3, pad = _case(key)
    st = P.Stencil(*k3, weights=w)
    got = P.convolve_pixels(vol, st, P.PadMode(pad))
    assert np.array_equal(G.bits(got), G.bits(PIX[key])), key
    fast = P.convolve_pixels(vol, st, P.PadMode(pad), accum="fast").astype(np.float64)
    ref = PIX[key].astype(np.float64)
    if key.split("__")[1].startswith("g"):
        # non-negative stencils: the reference's own bound (acceptance.cpp:271-276)
        scale = np.maximum(np.maximum(np.abs(fast), np.abs(ref)), 1.0)
        assert float(np.max(np.abs(fast - ref) / scale)) <= 1e-5, key
    else:
        # signed stencils cancel: fp32 summation's a-priori bound n * u * sum|w| max|v|
        n = int(np.count_nonzero(w))
        bound = n * 2.0 ** -24 * float(np.sum(np.abs(w), dtype=np.float64)) * float(np.max(np.abs(vol)))
        assert float(np.max(np.abs(fast - ref))) <= bound, key


@pytest.mark.gpu
def test_convolve_pixels_errors():
    import paper_2112_03592_b200 as P
    vol = np.zeros((4, 4, 4), np.float32)
    with pytest.raises(P.CapabilityError):
        P.convolve_pixels(vol, P.Stencil(15, 1, 1, weights=np.ones(15)), P.PadMode.Reflect)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(20, 100, 200), (7, 97, 198), (40, 70, 132)])
@pytest.mark.parametrize("k", [3, 5])
@pytest.mark.parametrize("pad", [0, 1])
def test_device_convolve_pixels_tiles_bit_exact(shape, k, pad):
    """Volumes with interior column tiles (x and y away from every face: the
    TMA plane loads under reflection), edge tiles (the cp.async path under
    reflection, TMA zero fill under zero padding), ragged x, and ny not a
    multiple of 4 (no tensor map): EXACT bit-identical to the C oracle."""
    import paper_2112_03592_b200 as P
    rng = np.random.default_rng(sum(shape) + k + pad)
    vol = rng.uniform(0.0, 100.0, shape).astype(np.float32)
    st = P.gaussian_stencil(1.0, k)
    got = P.convolve_pixels(vol, st, P.PadMode(pad))
    exp = ORC.convolve_pixels(vol, np.asarray(st.weights, np.float32), (k, k, k), pad)
    assert np.array_equal(G.bits(got), G.bits(exp)), (shape, k, pad)
