"""Smoke-size matvecs that launch every hand-written kernel family once, for
compute-sanitizer (one tool per gpurun call, profiles/r02_sanitizer_*.txt):

  python scripts/sanitize_case.py

C2/8 (N = 125k, L = 4, gauss02 JIT functor): int8 M2L -- the plane kernel
(level 4) and the mixed-octant gather kernel (levels 2-3) -- the projections,
P2M/M2M/L2L/L2P, the P2P; the same on the FP64 DMMA engine (m2l_ws_kernel);
a clustered cloud (active-cell lists, listed-cell int8 gather, point L2P);
the symmetric P2P; the uniform FFT M2L (fft_fwd / stencil / fft_inv); the
GPU direct sum; the tree build."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402


def plan_of(wl, **kw):
    d = dict(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
             domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
    d.update(kw)
    return bf.FmmPlan(**d)


wl = workloads.make("C2", 1)
k = workload_kernel(wl["kernel"])
ev = bf.FmmEvaluator(k, plan_of(wl), cache_dir="/tmp/bfmm_san")
a = ev.evaluate(wl["points"], weights=wl["weights"])
ev.m2l_mode = "dmma"
b = ev.evaluate(wl["points"], weights=wl["weights"])
print("i8 vs dmma rel", np.linalg.norm(a - b) / np.linalg.norm(b), flush=True)
ev.m2l_mode = "i8"
ev.near_mode = "symmetric"
c = ev.evaluate(wl["points"], weights=wl["weights"])
print("symmetric P2P rel", np.linalg.norm(a - c) / np.linalg.norm(a), flush=True)

# clustered cloud: active lists + listed-cell gather + point L2P
g = np.random.default_rng(3)
pts = np.clip(0.5 + 0.05 * g.standard_normal((60000, 3)), 0.0, 1.0)
w = g.standard_normal(60000)
pl = bf.FmmPlan(levels=5, order=5, eps=1e-7, domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
evc = bf.FmmEvaluator(bf.LAPLACIAN, pl, cache_dir="/tmp/bfmm_san")
evc.far_mode = "active"
phi = evc.evaluate(pts, weights=w)
print("clustered ok", np.isfinite(phi).all(), flush=True)

# uniform FFT M2L, 3 columns
u = workloads.make("C3", 2)
evu = bf.FmmEvaluator(workload_kernel(u["kernel"]), plan_of(u), cache_dir="/tmp/bfmm_san")
phu = evu.evaluate(u["points"], weights=u["weights"][:, :3])
print("uniform ok", np.isfinite(phu).all(), flush=True)

d = bf.direct_evaluate(k, wl["points"], targets=wl["points"][:200], weights=wl["weights"])
print("direct rel", np.linalg.norm(a[:200] - d) / np.linalg.norm(d), flush=True)
torch.cuda.synchronize()
print("sanitize case done", flush=True)
