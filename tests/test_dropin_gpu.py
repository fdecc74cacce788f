"""The reference's OWN tests, compiled unmodified against the C++ drop-in.

tests/cpp/Makefile builds proj/tests/test_*.cpp (with the doctest shim in
tests/cpp/doctest.h) and proj/tests/acceptance.cpp from /root/reference with
include/aprkit_gpu/ ahead of the reference's include directory, so every
convolve_apr / nonempty_row_index / fill_tree / init_tree_structure / rl_apr
call in them (and validate, reconstruct_*, convolve_pixels) runs on the GPU
through libaprgpu.so: all 10 acceptance criteria.  The binaries are built in
the container that has the reference and travel to the GPU box.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "cpp", "_build")


def _run(args, timeout, env=None):
    if not os.path.exists(args[0]):
        pytest.skip(f"{os.path.basename(args[0])} not built (needs /root/reference at build time)")
    p = subprocess.run(args, capture_output=True, text=True, timeout=timeout,
                       env=dict(os.environ, **env) if env else None)
    return p.returncode, p.stdout + p.stderr


def test_reference_unit_tests_pass_on_the_dropin():
    rc, out = _run([os.path.join(BUILD, "unit_tests")], 900)
    assert rc == 0, out[-4000:]
    assert "failed: 0 | assertions" in out, out[-2000:]


@pytest.mark.parametrize("criterion", [1, 2, 3, 4, 5, 6, 7, 8, 9])
def test_reference_acceptance_criterion_on_the_dropin(criterion, tmp_path):
    rc, out = _run([os.path.join(BUILD, "acceptance"), str(tmp_path), str(criterion)], 1800)
    assert rc == 0 and "PASS" in out, out[-3000:]


def test_reference_acceptance_serialization_on_the_dropin(tmp_path):
    # criterion 10: 200 write/read/re-write round trips (read_apr validates
    # through the drop-in's device validate), then the reference's own fixtures
    # written and read back
    exe = os.path.join(BUILD, "acceptance")
    rc, out = _run([exe, str(tmp_path), "--write-fixtures", "10"], 900)
    assert rc == 0 and "PASS" in out, out[-3000:]
    rc, out = _run([exe, str(tmp_path), "10"], 900)
    assert rc == 0 and "PASS" in out, out[-3000:]


# The same unmodified reference tests with APRGPU_DEVICES=0,0: every
# convolve_apr the drop-in serves runs on two z-slabs (aprgpu_multi_*) -- two
# virtual slabs of device 0 on this one-GPU box, the N-GPU code path verbatim
# (structures too thin to cut fall back to one slab).
def test_reference_unit_tests_pass_on_two_slabs():
    rc, out = _run([os.path.join(BUILD, "unit_tests")], 900, env={"APRGPU_DEVICES": "0,0"})
    assert rc == 0, out[-4000:]
    assert "failed: 0 | assertions" in out, out[-2000:]


@pytest.mark.parametrize("criterion", [3, 4, 8, 9])
def test_reference_acceptance_on_two_slabs(criterion, tmp_path):
    rc, out = _run([os.path.join(BUILD, "acceptance"), str(tmp_path), str(criterion)], 1800,
                   env={"APRGPU_DEVICES": "0,0"})
    assert rc == 0 and "PASS" in out, out[-3000:]
