"""validate (apr.hpp:61-134) -- SURVEY §8f row 1's O(particles) validator.

Golden verdicts (ok + message) from the real reference on valid and broken leaf
structures (tests/golden/make_validate_golden.py): every kind of violation the
reference reports -- level offsets, xz_end, row order, level-grid range, cells
outside the image, double coverage, uncovered pixels.  CPU: the C oracle's
restatement (O(pixels) cover map) against them; GPU: the device validator
(aprgpu_validate_access, O(particles + rows)) against them -- same verdict,
same message, same first violation.
"""
import numpy as np
import pytest

import goldens as G
from pyoracle import Access, Oracle

ORC = Oracle()
VAL = G.load("validate")
KEYS = sorted({k[:4] for k in VAL if k.startswith("c")})
FIELDS = ("l_min", "l_max", "z_dim", "x_dim", "y_dim", "y_idx", "xz_end", "level_offset")


def case(key):
    f = {k: VAL[f"{key}_{k}"] for k in FIELDS}
    f["l_min"], f["l_max"] = int(f["l_min"]), int(f["l_max"])
    return (f, tuple(int(v) for v in VAL[f"{key}_dims"]), bool(VAL[f"{key}_ok"][0]),
            VAL[f"{key}_msg"].tobytes().decode(), VAL[f"{key}_name"].tobytes().decode())


def test_golden_cases_cover_every_violation():
    msgs = {case(k)[3].split(" at ")[0].split(" in ")[0] for k in KEYS}
    for m in ("", "level_offset mismatch", "xz_end length does not match level grids", "xz_end decreases",
              "non-increasing y", "y index out of level grid", "particle cell outside the image domain",
              "double coverage: overlapping particle cells", "uncovered pixel"):
        assert m in msgs, m


@pytest.mark.parametrize("key", KEYS)
def test_oracle_validate_matches_reference(key):
    f, dims, ok, msg, name = case(key)
    assert ORC.validate(Access(**f), dims) == (ok, msg), name


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_device_validate_matches_reference(key):
    import paper_2112_03592_b200 as P
    f, dims, ok, msg, name = case(key)
    rep = P.validate(P.LinearAccess(**f), dims)
    assert (rep.ok, rep.message) == (ok, msg), name


@pytest.mark.gpu
def test_device_validate_on_built_and_tiled_aprs():
    import paper_2112_03592_b200 as P
    from paper_2112_03592_b200 import synth
    apr, _ = synth.build_spheres_apr(96, count=7, rmin=4.0, rmax=14.0, blur=2.0, seed=5, rel_error=0.1)
    assert P.validate(apr).ok
    d = G.load("c1_256")
    assert P.validate(G.product_apr(d)).ok
