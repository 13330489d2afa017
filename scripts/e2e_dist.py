"""Per-call end-to-end times of the C2 matvec from pinned host buffers."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402

wl = workloads.make("C2")
plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                  domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/bfmm_cfg_cache")
Xh = torch.from_numpy(wl["points"]).pin_memory()
Wh = torch.from_numpy(np.ascontiguousarray(wl["weights"])).pin_memory()
for _ in range(3):
    ev.evaluate(Xh, weights=Wh)
ts = []
for _ in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    phi = ev.evaluate(Xh, weights=Wh)
    ts.append(1e3 * (time.perf_counter() - t0))
print(" ".join(f"{t:.2f}" for t in ts))
print("median %.3f min %.3f max %.3f" % (np.median(ts), min(ts), max(ts)))
