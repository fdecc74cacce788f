"""bench.py --csv writes the reference's bench CSV schema (bench.hpp:33-42)
from a bench line (here the committed round-2 C3 line)."""
import csv
import importlib.util
import json
import os
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_csv_rows(tmp_path):
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    res = json.load(open(os.path.join(ROOT, "profiles", "r02", "bench_c3_k3_exact.json")))
    out = tmp_path / "bench.csv"
    b.write_bench_csv(str(out), res, types.SimpleNamespace(config="c3", stencil=3, accum="exact"))
    rows = list(csv.DictReader(open(out)))
    assert list(rows[0].keys()) == ["image_id", "dims", "cr", "op", "stencil_size", "wall_time_s",
                                    "effective_throughput_Bps", "memory_bytes_apr", "memory_bytes_pixels", "threads"]
    head = rows[0]
    assert head["op"] == "conv_apr" and head["dims"] == "1024x1024x1024" and head["threads"] == "0"
    t = float(head["wall_time_s"])
    assert abs(float(head["effective_throughput_Bps"]) - 4 * 1024 ** 3 / t) / (4 * 1024 ** 3 / t) < 1e-5
    ops = {r["op"] for r in rows}
    assert {"conv_apr", "conv_apr_e2e", "conv_apr_paper", "conv_pixels"} <= ops
    assert any(r["image_id"].endswith("/reference") and r["threads"] != "0" for r in rows)
