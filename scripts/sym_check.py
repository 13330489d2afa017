"""Symmetric (register-blocked) near field vs the full P2P on C2: phi
agreement and kernel time (development helper)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402
for spec in (sys.argv[1:] or ["C2:0"]):
    name, scale = spec.split(":")
    wl = workloads.make(name, int(scale))
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                      domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/bfmm_cache")
    X = torch.from_numpy(wl["points"]).cuda()
    W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
    ev.overlap_near = False
    ev.profile_kernels = True
    res = {}
    for mode in ("full", "symmetric", "full", "symmetric"):
        ev.near_mode = mode
        ks = []
        for _ in range(6):
            phi = ev.evaluate(X, weights=W)
            torch.cuda.synchronize()
            ks.append(ev.kernel_ms.get("p2p", 0.0))
        res[mode] = phi.cpu().numpy()
        d = float(np.linalg.norm(res[mode] - res["full"]) / np.linalg.norm(res["full"]))
        print(f"{spec} {mode}: p2p {sorted(ks)[1]:.4f} ms  total {ev.timings['total']*1e3:.3f} ms  "
              f"rel vs full {d:.2e}", flush=True)
