"""One warm matvec of a config (for ncu launch lists / metric captures):
python scripts/one_config.py C5 [scale]  -- prints the stage timings and the
near-field pair count.  Near field and far-field levels serialised."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402

import os  # noqa: E402
if os.environ.get("BFMM_LIB"):  # a variant build of libbfmm.so (tuning sweeps)
    from paper_1903_02153_b200 import _native
    _native.load(os.environ["BFMM_LIB"])
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wl = workloads.make(name, scale)
plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                  domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/bfmm_cfg_cache")
ev.stream_levels = False  # serial levels: clean per-kernel times
ev.overlap_near = False
import os  # noqa: E402
for knob in ("i8_digits", "m2l_mode", "p2m_mode", "l2p_mode", "proj_mode", "leaf_mode",
             "near_mode"):
    if os.environ.get("BFMM_" + knob.upper()):
        setattr(ev, knob, os.environ["BFMM_" + knob.upper()])
ev.profile_kernels = bool(os.environ.get("BFMM_PROFILE"))
X = torch.from_numpy(wl["points"]).cuda()
W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
for _ in range(2):
    ev.evaluate(X, weights=W)
torch.cuda.synchronize()
print({k: round(v * 1e3, 3) if isinstance(v, float) else v for k, v in ev.timings.items()})
if ev.profile_kernels:
    print({k: round(v, 3) for k, v in ev.kernel_ms.items()})
