"""C5 step time (device-resident inputs, CUDA events, 5 steps after 2
warm-ups) for near-field scheduling variants: near_after_far False/True,
with the M2L plane kernel's smem budget from BFMM_I8_COSCHED (env)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402

wl = workloads.make("C5", 0)
plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                  domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/ovl")
X = torch.from_numpy(wl["points"]).cuda()
W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
for naf in (False, True):
    ev.near_after_far = naf
    for _ in range(2):
        ev.evaluate(X, weights=W)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ev.evaluate(X, weights=W)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(os.environ.get("BFMM_I8_COSCHED", "0"), "near_after_far", naf, "ms", sorted(ts)[2],
          flush=True)
