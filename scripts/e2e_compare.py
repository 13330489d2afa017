"""e2e (pinned host in, pinned host out) C2 matvec time, eager vs CUDA graph,
plus the box's pinned H2D bandwidth (development helper)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf
from paper_1903_02153_b200 import workloads
from paper_1903_02153_b200.kernel import workload_kernel
x = torch.empty(32 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
d = torch.empty_like(x, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(x, non_blocking=True); torch.cuda.synchronize()
print("H2D 32 MiB %.3f ms" % ((time.perf_counter() - t0) * 1e3))
wl = workloads.make("C2", 0)
plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"], domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/bfmm_cache")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
Xh = torch.from_numpy(wl["points"]).pin_memory(); Wh = torch.from_numpy(np.ascontiguousarray(wl["weights"])).pin_memory()
X = torch.from_numpy(wl["points"]).cuda(); W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
for g, fl in ((False, False), (True, False), ("dev", True), (False, True), (True, True)):
    if g == "dev":  # bench's value loop: graph on device-resident inputs
        ev.use_graph = True
        for _ in range(13):
            flush.zero_(); ev.evaluate(X, weights=W); torch.cuda.synchronize()
        print("device-graph pass done, graphs:", len(ev._graphs))
        continue
    if g == "kt":  # bench's kernel-timing pass: eager, events, near field serialised
        ev.overlap_near, ev.profile_kernels = False, True
        for _ in range(10):
            flush.zero_(); ev.evaluate(X, weights=W); torch.cuda.synchronize()
        ev.overlap_near, ev.profile_kernels = True, False
        print("kernel-timing pass done")
        continue
    ev.use_graph = g
    for _ in range(4): phi = ev.evaluate(Xh, weights=Wh)
    ts = []
    for _ in range(10):
        if fl:
            flush.zero_()
        torch.cuda.synchronize(); t0 = time.perf_counter(); phi = ev.evaluate(Xh, weights=Wh); ts.append(time.perf_counter() - t0)
    print("graph" if g else "eager", "flush" if fl else "",  "e2e ms median %.3f min %.3f" % (1e3 * np.median(ts), 1e3 * min(ts)), "timings total", round(ev.timings["total"] * 1e3, 3))
