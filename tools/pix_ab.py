"""convolve_pixels timing on a 1024^3 volume (3^3 / 5^3, EXACT / FAST), device pointers,
CUDA events, best of 3 warm runs; HBM fraction = 8 B per pixel / time / measured peak."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import _lib as L  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6377.7) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6377.7
n = 1024
ctx = P.default_context()
x = torch.rand(n ** 3, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.Stream()  # (not the legacy default stream: the C-ABI call runs on this one)
torch.cuda.set_stream(s)
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for k in (3, 5):
    w = P.gaussian_stencil(1.0, k)
    for acc_name, acc in (("exact", L.ACCUM_EXACT), ("fast", L.ACCUM_FAST)):
        ts = []
        for i in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            P.convolve_pixels_ptr(ctx, x.data_ptr(), (n, n, n), w, 1, acc, y.data_ptr(), s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = min(ts[1:])
        print(f"{tag} k{k} {acc_name}: {t:.3f} ms, hbm frac {8 * n ** 3 / (t / 1e3) / 1e9 / peak:.3f}", flush=True)
