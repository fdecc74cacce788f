"""Dump a sample of C3's 3^3 gather-map records (EXACT, reflect) for offline
study of the apply's shared-memory access pattern (bank conflicts of the
code and value loads).  Needs a GPU:  python tools/dump_maps.py [n_sample]
Writes gpurun_out/maps_c3.npz: per sampled tile its level and record words."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import paper_2112_03592_b200 as P  # noqa: E402
from paper_2112_03592_b200 import _lib as L  # noqa: E402
from paper_2112_03592_b200 import synth  # noqa: E402

n_sample = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
apr, values = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
dapr = apr.device()
a = apr.access
pyr = P.make_pyramid(P.gaussian_stencil(1.0, 3), a.l_min, a.l_max, P.PyramidMode.Restricted).device()
v = torch.from_numpy(np.ascontiguousarray(values, np.float32)).cuda()
tv = torch.empty(max(dapr.n_tree, 1), dtype=torch.float32, device="cuda")
out = torch.empty_like(v)
s = torch.cuda.current_stream().cuda_stream
dapr.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
dapr.convolve_ptr(v.data_ptr(), tv.data_ptr(), pyr, 1, L.ACCUM_EXACT, out.data_ptr(), s)
torch.cuda.synchronize()
recs, lv, counts = [], [], {}
rng = np.random.default_rng(0)
total = 0
per = {}
for l in range(a.l_min, a.l_max + 1):
    nw, t0, nt = C.c_uint64(), C.c_uint64(), C.c_uint64()
    L.check(L.lib().aprgpu_map_records(dapr.handle, 1, 1, l, None, 0, None, C.byref(nw), C.byref(t0), C.byref(nt)))
    per[l] = (nw.value, nt.value)
    total += nt.value
for l, (nw, nt) in per.items():
    if nt == 0:
        continue
    buf = np.empty(nw, np.uint32)
    nw2, t0, nt2 = C.c_uint64(), C.c_uint64(), C.c_uint64()
    L.check(L.lib().aprgpu_map_records(dapr.handle, 1, 1, l, buf.ctypes.data, buf.size, None, C.byref(nw2),
                                       C.byref(t0), C.byref(nt2)))
    rec = buf.reshape(nt, -1)
    k = max(1, int(round(n_sample * nt / total)))
    idx = np.sort(rng.choice(nt, size=min(k, nt), replace=False))
    recs.append(rec[idx])
    lv.append(np.full(len(idx), l, np.int32))
    counts[l] = nt
    print(f"level {l}: tiles {nt}, sampled {len(idx)}", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/maps_c3.npz", rec=np.concatenate(recs), level=np.concatenate(lv),
                    levels=np.array(sorted(counts)), tiles=np.array([counts[l] for l in sorted(counts)]))
print("saved", sum(len(r) for r in recs))
