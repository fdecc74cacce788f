"""The bench's reference arm (bench.py --impl reference) runs only reference
code: its input comes from the C restatement of the reference build
(oracle/build_oracle.c) and the timed region is the unmodified reference
(oracle/_ref).  It must never load the product library (or torch), and its
`config` must be the same dict our arm prints."""
import json
import os
import subprocess
import sys

import pytest

from pyoracle import ref_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_reference_arm_loads_no_product_code():
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--config','c1','--steps','3','--warmup','3'];"
            "import bench; bench.main(); maps=open('/proc/self/maps').read();"
            "print(json.dumps({'aprgpu': 'libaprgpu' in maps, 'torch': 'libtorch' in maps}))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]
    res, maps = lines[0], lines[-1]
    assert not maps["aprgpu"] and not maps["torch"], maps
    assert res["impl"] == "reference" and res["value"] > 0
    assert res["e2e"]["h2d_bytes_per_step"] == 0
    sys.path.insert(0, ROOT)
    import bench
    c = res["config"]
    assert c == bench.bench_config("c1", 3, c["particles"], c["interior_nodes"], c["pixels"])
    assert c["particles"] == 278769 and c["interior_nodes"] == 39824  # SURVEY §8 C1 counts
