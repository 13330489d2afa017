"""Time the near-field kernel of one configuration under the current
BFMM_JIT_OPTS (NVRTC options of the JIT user kernel), for tuning sweeps:

    for o in "" "-DBFMM_P2P_UNROLL=2" "-DBFMM_P2P_MINB=6"; do
        BFMM_JIT_OPTS="$o" python scripts/p2p_variants.py C2; done
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402


def main(name, scale=0, reps=5):
    wl = workloads.make(name, scale)
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                      domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/bfmm_cfg_cache")
    ev._disable_far_field = True
    ev.near_mode = os.environ.get("BFMM_NEAR_MODE", "auto")
    X = torch.from_numpy(wl["points"]).cuda()
    W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
    ev.profile_kernels = True
    ev.evaluate(X, weights=W)
    ms = []
    for _ in range(reps):
        phi = ev.evaluate(X, weights=W)
        ms.append(ev.timings["near_field"] * 1e3)
    pairs = ev.timings["near_pairs"]
    print(json.dumps({"config": name, "opts": os.environ.get("BFMM_JIT_OPTS", ""),
                      "p2p_ms": min(ms), "pairs": pairs,
                      "gpairs_per_s": pairs / min(ms) / 1e6,
                      "checksum": float(torch.linalg.norm(phi))}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2", int(sys.argv[2]) if len(sys.argv) > 2 else 0)
