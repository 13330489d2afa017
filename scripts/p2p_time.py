"""C2 P2P kernel time (CUDA events, near field serialised) -- development helper."""
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
ev.overlap_near = False; ev.profile_kernels = True
ks = []
for i in range(8):
    ev.evaluate(X, weights=W); torch.cuda.synchronize(); ks.append(ev.kernel_ms["p2p"])
print("p2p ms", round(sorted(ks)[1], 4), flush=True)
