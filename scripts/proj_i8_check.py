import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_1903_02153_b200 as bf
from paper_1903_02153_b200.kernel import workload_kernel
g = np.load("tests/golden/eig.npz")
pts = g["pts"]
kernel = workload_kernel("exp03")
plan = bf.FmmPlan(levels=3, order=5, scheme="chebyshev", eps=1e-7, domain_center=(0.5,0.5,0.5), domain_length=1.0)
ev = bf.FmmEvaluator(kernel, plan, cache_dir="/tmp/cc")
w = np.random.default_rng(0).standard_normal((4000, 120))
out = {}
for mode in ("fp64", "i8"):
    ev.proj_mode = mode
    out[mode] = ev.evaluate(pts, weights=w)
print("rel", np.linalg.norm(out["i8"]-out["fp64"])/np.linalg.norm(out["fp64"]))
for c in (1, 2, 3, 4, 8):
    ww = w[:, :c]
    a = {}
    for mode in ("fp64", "i8"):
        ev.proj_mode = mode
        a[mode] = ev.evaluate(pts, weights=ww)
    print(c, np.linalg.norm(a["i8"]-a["fp64"])/np.linalg.norm(a["fp64"]))
print({k: blk.rank for k, blk in ev.table.blocks.items()} if hasattr(ev.table, "blocks") else None)
