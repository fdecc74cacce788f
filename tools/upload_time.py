import sys, time, os
sys.path[:0] = [os.getcwd()]
import numpy as np, torch
import paper_2112_03592_b200 as P
from paper_2112_03592_b200 import synth
apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
ctx = P.default_context()
h = apr.download() if hasattr(apr, "download") else apr
for i in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a2 = P.APR(apr.access, apr.tree_access, apr.source_dims)
    t1 = time.perf_counter()
    d = P.aprkit.DeviceApr.upload(ctx, a2)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"APR() {1e3*(t1-t0):.2f} ms upload {1e3*(t2-t1):.2f} ms", flush=True)
    del d
