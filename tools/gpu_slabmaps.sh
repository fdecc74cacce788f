mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_slab.py tests/test_multi_gpu.py tests/test_pixels.py tests/test_dropin_gpu.py -m gpu -q -x -rf 2>&1 | tail -15 > gpurun_out/slab_tests.log
python - <<'PY' >> gpurun_out/slab_tests.log 2>&1
import sys; sys.path[:0] = [".", "tests"]
import goldens as G, paper_2112_03592_b200 as P
from paper_2112_03592_b200.slab import SlabPlan
d = G.load("c1_256"); apr = G.product_apr(d)
for world in (2, 4, 8):
    for r in range(world):
        p = SlabPlan.make(apr.access, apr.tree_access, apr.source_dims, world, r, halo=2)
        print(world, r, p.lc if hasattr(p, "lc") else "", flush=True)
PY
cat gpurun_out/slab_tests.log
