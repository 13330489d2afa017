"""M2L split-count sweep for one level of a config (tuning helper):
    python scripts/split_sweep.py C2 4 19 23 37 74"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402

name, lev = sys.argv[1], int(sys.argv[2])
splits = [int(a) for a in sys.argv[3:]]
wl = workloads.make(name)
plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                  domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/bfmm_cfg_cache")
ev.stream_levels = False
ev.profile_kernels = True
X = torch.from_numpy(wl["points"]).cuda()
W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
orig = ev.lib.bfmm_m2l_cheb_splits
for ns in [None] + splits:
    ev.lib.bfmm_m2l_cheb_splits = (orig if ns is None else
                                   (lambda l, m, rp, nq, ns=ns: ns if l == lev else orig(l, m, rp, nq)))
    ts = []
    for _ in range(5):
        ev.evaluate(X, weights=W)
        ts.append(ev.kernel_ms[f"m2l_l{lev}"])
    print(f"level {lev} splits {ns or 'default'}: m2l {min(ts):.4f} ms, far_field "
          f"{ev.timings['far_field'] * 1e3:.3f} ms", flush=True)
