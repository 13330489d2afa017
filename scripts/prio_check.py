"""Far-field stream priority vs the overlapped near field (C2; eager and graph)."""
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
ref = None
for graph in (False, True):
    for prio, after in ((False, False), (True, False), (True, True)):
        ev.use_graph = graph; ev.far_priority = prio; ev.near_after_far = after; ev._graphs = {}
        for _ in range(3): phi = ev.evaluate(X, weights=W)
        ts = []
        for _ in range(10):
            torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); phi = ev.evaluate(X, weights=W); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        p = phi.cpu().numpy()
        if ref is None: ref = p
        print(f"graph {graph} prio {prio} after {after}: {np.median(ts):.3f} ms  same={np.array_equal(p, ref)}", flush=True)
