"""int8 tensor-core M2L vs the FP64 DMMA M2L: phi agreement and kernel times
per digit count S (development helper; run on the GPU box)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402

cfgs = sys.argv[1:] or ["C1:0", "C2:1", "C2:0"]
for spec in cfgs:
    name, scale = spec.split(":")
    wl = workloads.make(name, int(scale))
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                      domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/bfmm_cache")
    X = torch.from_numpy(wl["points"]).cuda()
    W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
    res = {}
    for mode, S in [("dmma", 0), ("i8", 5), ("i8", 6), ("i8", 7), ("i8", 8)]:
        ev.m2l_mode, ev.i8_slices = mode, (S or 7)
        ev.profile_kernels = True
        ev.overlap_near = False  # kernel spans without the near field sharing the SMs
        for _ in range(3):
            phi = ev.evaluate(X, weights=W)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            phi = ev.evaluate(X, weights=W)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        res[(mode, S)] = phi.cpu().numpy() if torch.is_tensor(phi) else np.asarray(phi)
        km = {k: round(v, 4) for k, v in ev.kernel_ms.items() if k.startswith("m2l")}
        ref = res[("dmma", 0)]
        d = float(np.linalg.norm(res[(mode, S)] - ref) / np.linalg.norm(ref))
        print(f"{spec} {mode} S={S}: {1e3 * min(ts):.3f} ms  rel-L2 vs dmma {d:.3e}  "
              f"far {ev.timings.get('far_field', 0) * 1e3:.3f} ms  {km}", flush=True)
