"""Throughput and accuracy of every BASELINE.json configuration at full size.

    python scripts/run_configs.py [C1 C2 C3 C4 C5] > profiles/rNN_configs.jsonl

Per config: one warm-up matvec, two timed ones (CUDA events, device-resident
inputs), stage timings, and the accuracy against the GPU direct sum on the
1,000 check targets (default_rng(1).choice(N, 1000)); where a
reference fixture exists (tests/golden) the reference's own accuracy and the
phi parity at the check targets are reported beside it.
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run(name):
    t0 = time.time()
    wl = workloads.make(name)
    kernel = workload_kernel(wl["kernel"])
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"],
                      eps=wl["eps"], domain_center=wl["center"], domain_length=wl["length"],
                      n_cols=wl["ncols"])
    ev = bf.FmmEvaluator(kernel, plan, cache_dir="/tmp/bfmm_cfg_cache")
    setup = time.time() - t0
    X = torch.from_numpy(wl["points"]).cuda()
    W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
    ev.profile_kernels = True
    ev.evaluate(X, weights=W)
    ms = []
    for _ in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        phi = ev.evaluate(X, weights=W)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    # the same matvec without per-kernel events, eager and (where the whole
    # device step is capturable) replayed from a CUDA graph
    ev.profile_kernels = False
    timings_staged = dict(ev.timings)
    kernel_ms = dict(ev.kernel_ms)
    fast = {}
    for g in (False, True):
        ev.use_graph = g
        if g and not ev._graph_ok(X, None, W, False, True):
            continue
        ev.evaluate(X, weights=W)
        t = []
        for _ in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ev.evaluate(X, weights=W)
            e1.record()
            e1.synchronize()
            t.append(e0.elapsed_time(e1))
        fast["graph" if g else "eager"] = min(t)
    ev.use_graph = False
    n = wl["points"].shape[0]
    idx = wl["check_idx"]
    phi_idx = phi[torch.from_numpy(idx).cuda()].cpu().numpy()
    t1 = time.time()
    d = bf.direct_evaluate(kernel, X, targets=X[torch.from_numpy(idx).cuda()], weights=W).cpu().numpy()
    dsec = time.time() - t1
    if phi_idx.ndim == 1:
        d = d.reshape(phi_idx.shape)
    out = {"config": name, "description": workloads.DESCRIPTION[name], "n_points": n,
           "levels": wl["levels"], "order": wl["order"], "scheme": wl["scheme"],
           "ncols": wl["ncols"], "ms_per_matvec": min(ms), "points_per_s": n / (min(ms) * 1e-3),
           "ms_per_matvec_no_kernel_events": fast.get("eager"),
           "ms_per_matvec_graph": fast.get("graph"),
           "setup_s": setup, "stages_ms": {k: (round(v * 1e3, 3) if isinstance(v, float) else v)
                                           for k, v in timings_staged.items()},
           "kernels_ms": {k: round(v, 3) for k, v in kernel_ms.items()},
           "rel_l2_vs_direct_1000": rel(phi_idx, d), "direct_seconds_gpu": dsec,
           "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}
    gp = os.path.join(GOLD, f"{name.lower()}_s0.npz")
    if not os.path.exists(gp):  # full-size C3 / C4 fixtures
        gp = os.path.join(GOLD, f"{name.lower()}_full.npz")
    if os.path.exists(gp):
        g = np.load(gp)
        out["reference_rel_l2_vs_direct"] = float(g["rel_l2_vs_direct"])
        out["rel_l2_vs_reference_phi_idx"] = rel(phi_idx, g["phi_idx"].reshape(phi_idx.shape))
        out["reference_seconds"] = float(g["seconds"])
        out["reference_threads"] = int(g["threads"])
    print(json.dumps(out), flush=True)
    del ev, X, W, phi
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]):
        run(c)
