"""CTA-pair int8 M2L (m2l_i8p2_kernel) vs the single-CTA plane kernel:
bitwise-equal phi (the same 21 digit products land in accumulators 0..5)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402

for name, scale in (("C5", 3), ("C5", 2), ("C2", 1)):
    wl = workloads.make(name, scale)
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                      domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir="/tmp/p2c")
    out = {}
    for mode in ("pair", "1cta"):
        if mode == "1cta":
            os.environ["BFMM_I8_1CTA"] = "1"
        else:
            os.environ.pop("BFMM_I8_1CTA", None)
        out[mode] = ev.evaluate(wl["points"], weights=wl["weights"])
    torch.cuda.synchronize()
    d = np.abs(out["pair"] - out["1cta"]).max()
    print(name, scale, "bitwise" if np.array_equal(out["pair"], out["1cta"]) else f"max diff {d}",
          flush=True)
os.environ.pop("BFMM_I8_1CTA", None)
