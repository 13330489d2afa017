"""Does the host keep the GPU fed?  Times the C2 matvec normally and with the
GPU held by a spin kernel while every launch of the step is enqueued (the
device then runs the step back to back): the difference is launch gaps."""
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
for _ in range(3): ev.evaluate(X, weights=W, )
def run(pre_spin):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    if pre_spin:
        torch.cuda._sleep(int(30e6))  # ~15 ms of GPU spin while the host enqueues
    e0.record()
    t0 = time.perf_counter()
    ev.evaluate(X, weights=W)
    th = time.perf_counter() - t0
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1), th * 1e3
for pre in (False, True, False, True):
    r = [run(pre) for _ in range(5)]
    print("pre-spin" if pre else "normal  ", "device ms (median)", round(float(np.median([a for a, b in r])), 3), "host ms", round(float(np.median([b for a, b in r])), 3))
