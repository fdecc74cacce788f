"""The .apr container (io.hpp:102-183, docs/FORMATS.md).

Fixtures written by the real reference (tests/golden/make_io_golden.py): the
device loader reads them straight into a handle -- structures, values and build
parameters equal to what the reference wrote -- writes them back byte for byte,
and fails on every byte-level corruption with the reference reader's exception
type and message (including validate's verdict on a broken structure, computed
on the device).
"""
import os
import tempfile

import numpy as np
import pytest

import goldens as G

APR_DIR = os.path.join(G.GOLDEN, "apr")
IO = G.load("io")
CORRUPT = sorted({k[: -len("_kind")] for k in IO if k.endswith("_kind")})
KINDS = {1: "IoError", 2: "BadFormatError", 3: "TruncatedFileError"}


def test_fixtures_and_verdicts_cover_the_reader():
    assert os.path.getsize(os.path.join(APR_DIR, "spheres64.apr")) > 0
    kinds = {int(IO[k + "_kind"][0]) for k in CORRUPT}
    assert kinds == {2, 3}
    msgs = " ".join(IO[k + "_msg"].tobytes().decode() for k in CORRUPT)
    for m in ("bad magic", "version", "bad source dims", "sigma mode", "gradient mode", "bad level range",
              "implausible element count", "unexpected end of file", "invalid APR structure"):
        assert m in msgs, m


@pytest.mark.gpu
def test_load_matches_the_reference_writer_and_saves_byte_identical():
    import paper_2112_03592_b200 as P
    d = G.load("spheres64")
    path = os.path.join(APR_DIR, "spheres64.apr")
    apr, values = P.load_apr(path)
    ref = G.product_apr(d)
    assert apr.access.equals(ref.access) and apr.tree_access.equals(ref.tree_access)
    assert tuple(apr.source_dims) == tuple(int(v) for v in d["dims"])
    assert np.array_equal(G.bits(values), G.bits(d["values"]))
    assert apr.params == P.BuildParams()
    for name in ("spheres64", "built40"):
        src = os.path.join(APR_DIR, name + ".apr")
        a, v = P.load_apr(src)
        with tempfile.TemporaryDirectory() as t:
            out = os.path.join(t, "x.apr")
            P.save_apr(out, a, v)
            assert open(out, "rb").read() == open(src, "rb").read(), name


@pytest.mark.gpu
def test_loaded_apr_runs_the_hot_path():
    import paper_2112_03592_b200 as P
    d = G.load("spheres64")
    apr, values = P.load_apr(os.path.join(APR_DIR, "spheres64.apr"))
    tv = P.fill_tree(apr, values)
    assert np.array_equal(G.bits(tv), G.bits(d["tree_values"]))


@pytest.mark.gpu
@pytest.mark.parametrize("key", CORRUPT)
def test_corrupt_files_fail_like_the_reference(key):
    import paper_2112_03592_b200 as P
    name = key.split("__")[0]
    raw = open(os.path.join(APR_DIR, name + ".apr"), "rb").read()
    trunc = int(IO[key + "_trunc"][0])
    b = bytearray(raw if trunc < 0 else raw[:trunc])
    for off, v in IO[key + "_edits"]:
        b[int(off)] = int(v)
    kind = KINDS[int(IO[key + "_kind"][0])]
    msg = IO[key + "_msg"].tobytes().decode()
    with tempfile.TemporaryDirectory() as t:
        p = os.path.join(t, "bad.apr")
        open(p, "wb").write(bytes(b))
        with pytest.raises(getattr(P, kind)) as e:
            P.load_apr(p)
    assert str(e.value) == msg


@pytest.mark.gpu
def test_missing_file_is_an_io_error():
    import paper_2112_03592_b200 as P
    with pytest.raises(P.IoError):
        P.load_apr("/nonexistent/x.apr")
