"""Build C3 on the GPU and dump its leaf/tree access structure (for offline
tile-shape analysis; not used by tests or the bench)."""
import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_03592_b200 import synth
apr, vals = synth.build_spheres_apr(1024, count=48, rmin=24.0, rmax=80.0, blur=2.0, seed=42, rel_error=0.1)
a, t = apr.access, apr.tree_access
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "c3_struct.npz"), leaf_y=a.y_idx, leaf_xz=a.xz_end,
                    leaf_lo=a.level_offset, zd=a.z_dim, xd=a.x_dim, yd=a.y_dim, l_range=np.array([a.l_min, a.l_max]),
                    tree_y=t.y_idx, tree_xz=t.xz_end, tree_lo=t.level_offset, tl_range=np.array([t.l_min, t.l_max]))
print(a.particle_count(), t.particle_count())
