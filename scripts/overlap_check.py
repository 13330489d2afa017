import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf
from paper_1903_02153_b200 import workloads
from paper_1903_02153_b200.kernel import workload_kernel
wl = workloads.make("C2", 0)
plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"], domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/bfmm_cache")
X = torch.from_numpy(wl["points"]).cuda(); W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
for ov, after in ((False, False), (True, False), (True, True)):
  for S in (7,):
    ev.overlap_near = ov; ev.i8_slices = S; ev.near_after_far = after
    for _ in range(3): ev.evaluate(X, weights=W)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize(); t0 = time.perf_counter(); ev.evaluate(X, weights=W); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print("overlap", ov, "after", after, "S", S, f"{1e3*np.median(ts):.3f} ms", {k: round(v*1e3,3) for k, v in ev.timings.items() if isinstance(v, float)})
