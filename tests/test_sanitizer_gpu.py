"""compute-sanitizer over the hot path: memcheck, racecheck
(shared-memory hazards: the mbarrier / bulk-copy staging and the in-place 5^3
box expansion of the map kernel, the tile scatter) and synccheck, on the C1
fixture through every kernel family (tools/sanitize_c1.py).  Zero reported
hazards is the bar."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"



def _sanitizer_usable():
    """The tool exists and runs here (some GPU pools disable it: their wrapper
    prints why and exits non-zero -- the committed profiles/r02/sanitizer_*.log
    runs stand then)."""
    if not os.path.exists(SAN):
        return False, "compute-sanitizer not found"
    try:
        r = subprocess.run([SAN, "--version"], capture_output=True, text=True, timeout=120)
    except Exception as e:  # noqa: BLE001
        return False, f"compute-sanitizer does not run: {e}"
    out = (r.stdout + r.stderr).strip()
    if r.returncode != 0 or "closed" in out.lower():
        return False, f"compute-sanitizer unavailable on this machine: {out[:200]}"
    return True, ""


_OK, _WHY = _sanitizer_usable()


@pytest.mark.skipif(not _OK, reason=_WHY or "compute-sanitizer unavailable")
@pytest.mark.parametrize("tool,workload", [("memcheck", "all"), ("racecheck", "all"), ("synccheck", "all")])
def test_compute_sanitizer_clean(tool, workload):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_c1.py"), workload]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log"), "w") as f:
        f.write(out[-20000:])
    assert "sanitize workload done" in out, out[-3000:]
    if tool == "racecheck":
        h = re.search(r"RACECHECK SUMMARY: (\d+) hazards displayed \((\d+) errors, (\d+) warnings\)", out)
        assert h and h.groups() == ("0", "0", "0"), out[-3000:]
    else:
        m = re.search(r"ERROR SUMMARY: (\d+) error", out)
        assert m and int(m.group(1)) == 0, out[-3000:]
    assert r.returncode == 0, out[-3000:]
