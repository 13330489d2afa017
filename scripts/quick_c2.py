"""Quick stage timing of one config on the GPU (development helper)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf
from paper_1903_02153_b200 import workloads
from paper_1903_02153_b200.kernel import workload_kernel

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wl = workloads.make(name, scale)
plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                  domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
t0 = time.time()
ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/bfmm_cache")
print("setup", time.time() - t0, "s; ranks", {k: getattr(b, "rank", None) for k, b in ev.table.blocks.items()})
X = torch.from_numpy(wl["points"]).cuda()
W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
for i in range(5):
    torch.cuda.synchronize(); t0 = time.time()
    phi = ev.evaluate(X, weights=W)
    torch.cuda.synchronize()
    print(f"iter {i}: {1e3*(time.time()-t0):.2f} ms", {k: (round(v*1e3, 3) if isinstance(v, float) else v) for k, v in ev.timings.items()})
