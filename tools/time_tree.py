"""Warm timings on C3 (CUDA events): fill_tree alone, then once per KEY=VALUE
argument with that variable set (the library reads it at call time).

    python tools/time_tree.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import synth  # noqa: E402

apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
dev = apr.device()
v = torch.from_numpy(values).cuda()
tv = torch.empty(dev.n_tree, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    dev.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)


def run(tag):
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"fill_tree C3{tag}: median {ts[len(ts) // 2] * 1e3:.1f} us, min {ts[0] * 1e3:.1f} us "
          f"({dev.n_particles} leaves, {dev.n_tree} interior nodes)")


run("")
for kv in sys.argv[1:]:
    k, val = kv.split("=", 1)
    os.environ[k] = val
    for _ in range(3):
        dev.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
    run(f" [{kv}]")
    del os.environ[k]
