#!/usr/bin/env python
"""FMM matvec throughput (points/s, fp64) on B200 — the BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C5] [--secondary C2|none] [--no-cpu-baseline]

Workload (N=1): C5 of BASELINE.json — Laplace 1/r, N = 64,000,000 i.i.d.
uniform in [-1,1]^3, octree L=8, Chebyshev p=5, 1 RHS — the configuration
the metric ("points/s at 1/2/4/8 B200") is quoted on: the only config
defined as a 1/2/4/8-GPU run, and the largest that fits one B200 (71 GB
peak).  Inputs are the seeded synthetic recipe of SURVEY.md §8(d) (no public
dataset is involved; the paper itself uses uniform random clouds).  A step
is one full matvec phi = K sigma: tree build, P2M, M2M, M2L, L2L, L2P, P2P,
output scatter.  ``--config C1..C5`` runs any other config the same way;
``--secondary C2`` (default) adds a short C2 measurement (the P2P-dominated
config) to the same JSON line under "secondary".

* value     device-resident inputs, CUDA-event time of K steps (barrier +
            synchronize on both sides, max over ranks); inputs are larger
            than L2 (C5: 2 GB) and L2 is flushed anyway (256 MiB write)
            between steps, outside the timed spans.
* e2e       the public API (FmmEvaluator.evaluate) on pinned host tensors:
            H2D of points + weights, the matvec, D2H of phi, every step.
  e2e_numpy the same through NumPy arrays (the reference's calling
            convention): pageable inputs staged through the evaluator's
            reusable pinned buffer.
* roofline  the dominant kernel (largest share of the step in a separate
            pass with CUDA events around every launch on its stream, the
            far-field levels and the near field serialised).  C5: the level-8
            int8 tcgen05 M2L against the measured kind::i8 peak (useful ops,
            executed ops beside); P2P against the measured DFMA peak;
            FFT M2L (C3) in Hadamard flops against the DFMA peak.
* cpu_baseline  the unmodified reference (boxfmm, installed under
            baseline/_ref by scripts/install_reference.sh) with every host
            core, on a bounded sample of the same workload: the
            density-preserving C5/512 (N = 125,000, L = 5, same kernel,
            order and points per leaf), rank 0 at N=1 only.
* --impl reference  the same reference run as the reference arm: per step
            one evaluate of that sample, all host threads, rank 0 only.
* N > 1: torchrun ranks (or ``--gpus N`` spawns them itself), NCCL; target
  cells split by Morton range (strong scaling: N = 64M in total), z of
  each level exchanged, each rank's phi range all-gathered.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FMM matvec points/sec (fp64) at 1/2/4/8 B200; P2P & M2L % of roofline"

# FP64 flops per near-field (target, source) pair -- the kernel evaluation
# plus the weight FMAs of all the config's columns -- per kernel functor:
# the FP64 thread instructions the P2P kernel executes per algorithmic pair
# (2*DFMA + DMUL + DADD, ncu smsp__sass_thread_inst_executed_op_d{fma,mul,
# add}_pred_on.sum / near_pairs), frozen once: gauss02 in round 1
# (profiles/r01_p2p_flops.txt; the kernel now executes 31.8), the others in
# round 2 (profiles/r02_p2p_flops.txt).  exp03 is C3's 16-column pair.
P2P_FLOPS_PER_PAIR = {"gauss02": 40.0, "laplacian": 18.07, "laplacianforce": 17.74,
                      "exp03": 86.0}
P2P_EXECUTED_PER_PAIR = {"gauss02": 31.8, "laplacian": 18.07, "laplacianforce": 17.74,
                         "exp03": 86.0}
NOMINAL_FP64_TF = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: DFMA/clk/SM x SMs x clock


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--secondary", default="C2", help="second config measured into the same "
                    "line ('none' to skip); N=1 only")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of CUDA-graph replay")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--balance", default="auto", choices=["auto", "cells", "work"],
                    help="N>1 shard ranges: equal cell ranges, work-weighted, or auto "
                         "(work-weighted for the clustered C4)")
    ap.add_argument("--ref-scale", type=int, default=None,
                    help="reference sample: the config scaled by 8^-k (default C5: 3, C4: 2, "
                         "C3: 2, C2: 1, C1: 0)")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
def _workloads():
    """paper_1903_02153_b200/workloads.py loaded on its own (NumPy only): the
    reference arm must not import the package (its library, its engine)."""
    spec = importlib.util.spec_from_file_location(
        "_bfmm_workloads", os.path.join(ROOT, "paper_1903_02153_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


REF_SCALE = {"C1": 0, "C2": 1, "C3": 2, "C4": 2, "C5": 3}


def config_of(name):
    W = _workloads()
    N, L, p, scheme, eps, kern, m = W.CONFIGS[name]
    return {"workload": f"{name}: {W.DESCRIPTION[name]}", "n_points": N, "levels": L,
            "order": p, "scheme": scheme, "eps": eps, "kernel": kern, "ncols": m,
            "l2": "inputs larger than L2 where the config has them; L2 flushed between "
                  "steps anyway (256 MiB write, outside the timed spans)"}


def config_dict(wl):
    return config_of(wl["name"])


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 8:
                for nm, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_threads():
    try:
        import psutil
        return max(1, psutil.cpu_count(logical=False) or os.cpu_count() or 1)
    except Exception:
        return max(1, os.cpu_count() or 1)


# ---------------------------------------------------------------------------
# the reference (unmodified boxfmm from baseline/_ref)
def _import_reference():
    path = os.environ.get("BOXFMM_SRC", os.path.join(ROOT, "baseline", "_ref"))
    if not os.path.isdir(os.path.join(path, "boxfmm")):
        return None, f"reference not installed at {path} (scripts/install_reference.sh)"
    sys.path.insert(0, path)
    import boxfmm
    return boxfmm, None


def _ref_kernel(boxfmm, key):
    if key == "gauss02":
        return boxfmm.KernelSpec("gauss02", homogen=0.0, symmetry=1,
                                 profile=lambda r: np.exp(-(r / 0.2) ** 2))
    if key == "exp03":
        return boxfmm.KernelSpec("exp03", homogen=0.0, symmetry=1,
                                 profile=lambda r: np.exp(-r / 0.3))
    return boxfmm.kernel_by_name(key)


class ReferenceSample:
    """One reference evaluate of the density-preserving scaled config (the
    bounded CPU sample), warm operator cache, `threads` host threads."""

    def __init__(self, config, scale, threads):
        boxfmm, err = _import_reference()
        if boxfmm is None:
            raise RuntimeError(err)
        self.wl = _workloads().make(config, scale)
        wl = self.wl
        plan = boxfmm.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"],
                              eps=wl["eps"], domain_center=wl["center"],
                              domain_length=wl["length"], n_cols=wl["ncols"])
        self.ev = boxfmm.FmmEvaluator(_ref_kernel(boxfmm, wl["kernel"]), plan,
                                      cache_dir="/tmp/bfmm_ref_cache", threads=threads)
        self.threads = threads
        self.n = int(wl["points"].shape[0])
        self.desc = (f"{config}/{8 ** scale} (N={self.n:,}, L={wl['levels']}, same kernel, "
                     f"order, scheme and points per leaf): one boxfmm.FmmEvaluator("
                     f"threads={threads}).evaluate per step, warm operator cache")

    def step(self):
        t0 = time.perf_counter()
        self.ev.evaluate(self.wl["points"], weights=self.wl["weights"])
        return time.perf_counter() - t0


def run_reference(args, rank, world):
    """Reference arm: the unmodified reference's CPU path, rank 0 only."""
    if rank != 0:
        return
    cfg = args.config
    scale = REF_SCALE.get(cfg, 0) if args.ref_scale is None else args.ref_scale
    threads = cpu_threads()
    try:
        ref = ReferenceSample(cfg, scale, threads)
    except RuntimeError as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}), flush=True)
        return
    for _ in range(args.warmup):
        ref.step()
    times = [ref.step() for _ in range(args.steps)]
    total = sum(times)
    value = ref.n * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SURVEY.md §8(d) recipe)",
        "config": config_of(cfg),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads,
                         "kind": "reference", "sample": ref.desc},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_timings_s": {k: round(float(v), 4) for k, v in ref.ev.timings.items()},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# algorithmic work
def level_pairs(lev):
    """P_l: (target, source) M2L cell pairs over the full level (oct:128-145)."""
    from paper_1903_02153_b200.tables import OFFSETS
    n = 1 << lev
    cnt = 0
    for t in OFFSETS:
        c = 1
        for a in range(3):
            tt = int(t[a])
            lo, hi = max(0, -tt), min(n - 1, n - 1 - tt)
            if abs(tt) == 3:
                k = len([x for x in range(lo, hi + 1) if (x % 2 == 0) == (tt > 0)])
            else:
                k = max(0, hi - lo + 1)
            c *= k
        cnt += c
    return cnt


def m2l_flops(ev, wl):
    """Algorithmic Chebyshev M2L flops per level: P_l * 2 r_l^2 * m."""
    m = wl["ncols"]
    return {lev: level_pairs(lev) * 2.0 * ev.table.block_for_level(lev).rank ** 2 * m
            for lev in range(2, wl["levels"] + 1)}


def fft_flops(wl):
    """Uniform M2L Hadamard flops per level: P_l * F * m * 8 (F = q^2 (q/2+1)
    complex bins, 8 flops per complex MAC)."""
    q = 2 * wl["order"] - 1
    F = q * q * (q // 2 + 1)
    return {lev: level_pairs(lev) * F * wl["ncols"] * 8.0 for lev in range(2, wl["levels"] + 1)}


def _valid_offsets(o):
    from paper_1903_02153_b200.tables import OFFSETS
    bits = ((o >> 2) & 1, (o >> 1) & 1, o & 1)
    out = []
    for t in OFFSETS:
        if all(not ((int(t[a]) == 3 and bits[a]) or (int(t[a]) == -3 and not bits[a]))
               for a in range(3)):
            out.append(tuple(int(x) for x in t))
    return out


def _pair_kernel(lev, S):
    """The CTA-pair plane kernel runs the level (csrc/m2l_i8p2.cuh, i8p2_ok):
    six 8-bit digits, dense level >= 5 (even z-tile count: always for whole
    levels >= 5)."""
    return S == 6 and lev >= 5 and not os.environ.get("BFMM_I8_1CTA")


def m2l_i8_ops(lev, rp, m, S):
    """int8 operations the tcgen05 M2L executes at one level: per (tile,
    offset, 32-wide k chunk, 64-wide rank tile) stage, S(S+1)/2 digit
    products of 128 x 64 x 32 (csrc/m2l_i8.cuh).  Dense levels >= 4 use the
    plane kernel, which skips offset groups whose source planes leave the
    grid; coarser levels run all 316 offsets over mixed-octant row tiles."""
    n = 1 << lev
    kc, ntn = -(-rp // 32), -(-rp // 64)
    per_stage = 2.0 * 128 * 64 * 32 * S * (S + 1) / 2
    if _pair_kernel(lev, S) and os.environ.get("BFMM_I8P2_N128") == "1":
        # unsplit m2l_i8p2_kernel: digit pairs (2k, 2k+1) per MMA, 24 products
        # (the 21 of a + b < 6 plus 3 that land in a dropped accumulator); the
        # default split variant runs those three as N = 64 MMAs: exactly 21
        per_stage = 2.0 * 128 * 64 * 32 * 24
    if lev >= 4:
        h = n // 2
        xt = 1 if lev >= 5 else 2
        yt = 16 // xt
        stages = 0
        for o in range(8):
            ox = (o >> 2) & 1
            offs = _valid_offsets(o)
            for xb in range(h // xt):
                xs = 2 * xb * xt + ox
                live = sum(1 for t in offs if xs + t[0] + 2 * (xt - 1) >= 0 and xs + t[0] < n)
                stages += live * (h // yt) * (h // 8)
        return stages * kc * ntn * m * per_stage
    stages = -(-(n ** 3 * m) // 128) * 316
    return stages * kc * ntn * per_stage


def active_level_work(cells, off, lev, rp, m, S):
    """Useful far pairs and executed int8 ops of an active-cell (sparse
    cloud) level: the valid far offsets of each listed target cell
    (octree.py:128-145), and the gather kernel's 128-row tiles per octant
    over its 189 offsets."""
    from paper_1903_02153_b200.tables import OFFSETS
    c = cells.cpu().numpy().astype(np.int64)
    n = 1 << lev

    def compact(v):
        v = v & 0x1249249249249249
        v = (v | (v >> 2)) & 0x10C30C30C30C30C3
        v = (v | (v >> 4)) & 0x100F00F00F00F00F
        v = (v | (v >> 8)) & 0x1F0000FF0000FF
        v = (v | (v >> 16)) & 0x1F00000000FFFF
        return (v | (v >> 32)) & 0x1FFFFF
    xyz = [compact(c >> 2), compact(c >> 1), compact(c)]
    pairs = 0
    for t in OFFSETS:
        ok = np.ones(len(c), bool)
        for a in range(3):
            s = xyz[a] + int(t[a])
            ok &= (s >= 0) & (s < n)
            if t[a] == 3:
                ok &= (xyz[a] & 1) == 0
            elif t[a] == -3:
                ok &= (xyz[a] & 1) == 1
        pairs += int(ok.sum())
    kc, ntn = -(-rp // 32), -(-rp // 64)
    per_stage = 2.0 * 128 * 64 * 32 * S * (S + 1) / 2
    tiles = sum(-(-(int(off[o + 1] - off[o]) * m) // 128) for o in range(8))
    return pairs, tiles * 189 * kc * ntn * per_stage


def committed_traffic(config, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu captures
    (profiles/r02_traffic.json, else r01), or None when not captured."""
    for name in ("r02_traffic.json", "r01_traffic.json"):
        path = os.path.join(ROOT, "profiles", name)
        try:
            with open(path) as f:
                rec = json.load(f).get(config, {}).get(kernel)
        except (OSError, ValueError):
            rec = None
        if rec is not None:
            return rec["bytes"]
    return None


def device_peaks(lib, stream):
    import ctypes as C
    g1, g2, g3 = C.c_double(0), C.c_double(0), C.c_double(0)
    lib.bfmm_device_fp64_probe(C.byref(g1), stream)
    lib.bfmm_device_dmma_probe(C.byref(g2), stream)
    lib.bfmm_device_i8_probe(C.byref(g3), stream)
    return {"dfma_tflops": g1.value / 1e3, "dmma_tflops": g2.value / 1e3,
            "i8_tops": g3.value}


# ---------------------------------------------------------------------------
def _evaluator(wl, device):
    import paper_1903_02153_b200 as bf
    from paper_1903_02153_b200.kernel import workload_kernel
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"],
                      eps=wl["eps"], domain_center=wl["center"], domain_length=wl["length"],
                      n_cols=wl["ncols"])
    return bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan,
                           cache_dir=os.path.join("/tmp", "bfmm_bench_cache"), device=device)


def _max_over_ranks(dist, v):
    if dist is None:
        return v
    import torch
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([v], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measure(cfg, args, rank, world, local_rank, dist, lib, peaks, steps, warmup,
            with_e2e=True):
    """Everything of one config's bench line except the CPU baseline."""
    import torch
    W = _workloads()
    wl = W.make(cfg)
    ev = _evaluator(wl, torch.device("cuda", local_rank))
    ev.use_graph = not args.no_graph
    n, m = wl["points"].shape[0], wl["ncols"]
    X = torch.from_numpy(wl["points"]).cuda()
    Wt = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
    if world > 1:
        from paper_1903_02153_b200.parallel import ShardedEvaluator
        balance = args.balance if args.balance != "auto" else ("work" if cfg == "C4" else "cells")
        runner = ShardedEvaluator(ev, dist, balance=balance)
    else:
        runner = ev
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def host_timed(make_inputs, tag):
        xs, ws = make_inputs()
        for _ in range(max(3, warmup)):
            phi = runner.evaluate(xs, weights=ws)
        barrier()
        ms = []
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            phi = runner.evaluate(xs, weights=ws)
            assert not (hasattr(phi, "is_cuda") and phi.is_cuda), tag
            ms.append(1e3 * (time.perf_counter() - t0))
        barrier()
        total = _max_over_ranks(dist, float(sum(ms)))
        del phi
        return {"value": n * steps / (total * 1e-3), "unit": "points/s",
                "ms_per_step": total / steps, "step_ms": [round(x, 3) for x in ms]}

    e2e = e2e_np = None
    if with_e2e:
        # measured before the device-resident loop (round-1 note: after it the
        # same calls ran slower on some boxes, a process-state effect)
        def pinned():
            return (torch.from_numpy(wl["points"]).pin_memory(),
                    torch.from_numpy(np.ascontiguousarray(wl["weights"])).pin_memory())
        e2e = host_timed(pinned, "e2e")
        e2e.update({"h2d_bytes_per_step": int(n * 3 * 8 + n * m * 8),
                    "d2h_bytes_per_step": int(n * m * 8),
                    "inputs": "pinned host torch tensors (points, weights) -> phi in "
                              "pinned host memory"})
        e2e_np = host_timed(lambda: (wl["points"], wl["weights"]), "e2e_numpy")
        e2e_np.update({"h2d_bytes_per_step": int(n * 3 * 8 + n * m * 8),
                       "d2h_bytes_per_step": int(n * m * 8),
                       "inputs": "NumPy arrays (pageable), as the reference's callers pass "
                                 "them; phi returned as a NumPy array"})

    # ---- device-resident timed loop ----
    for _ in range(warmup):
        runner.evaluate(X, weights=Wt)
    barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    barrier()
    launches0 = lib.bfmm_launch_count() + ev.graph_launches
    spans, stage_sum = [], {}
    for _ in range(steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        runner.evaluate(X, weights=Wt)
        e1.record()
        e1.synchronize()
        spans.append(e0.elapsed_time(e1))
        for k, v in ev.timings.items():
            if isinstance(v, float):
                stage_sum[k] = stage_sum.get(k, 0.0) + v
    barrier()
    launches = lib.bfmm_launch_count() + ev.graph_launches - launches0
    clk = clocks.stop()
    total_ms = _max_over_ranks(dist, float(sum(spans)))
    value = n * steps / (total_ms * 1e-3)

    # ---- per-kernel pass: CUDA events around every launch on its own
    # stream, far-field levels and near field serialised on one stream ----
    saved = (ev.overlap_near, ev.stream_levels, ev.profile_kernels)
    ev.overlap_near, ev.stream_levels, ev.profile_kernels = False, False, True
    kms = []
    for _ in range(max(2, min(steps, 5))):
        flush.zero_()
        runner.evaluate(X, weights=Wt)
        torch.cuda.synchronize()
        kms.append(dict(ev.kernel_ms))
        stages_serial = dict(ev.timings)
    ev.overlap_near, ev.stream_levels, ev.profile_kernels = saved
    avg = {}
    for d in kms:
        for k, v in d.items():
            avg[k] = avg.get(k, 0.0) + v / len(kms)
    step_ms = total_ms / steps
    near_pairs = int(ev.timings.get("near_pairs", 0))

    out = {"wl": wl, "ev": ev, "value": value, "total_ms": total_ms, "step_ms": step_ms,
           "launches": launches, "clocks": clk, "e2e": e2e, "e2e_numpy": e2e_np,
           "stages_ms": {k: round(1e3 * v / steps, 4) for k, v in stage_sum.items()},
           "stages_serial_ms": {k: (round(1e3 * v, 4) if isinstance(v, float) else v)
                                for k, v in stages_serial.items()},
           "kernels_ms": {k: round(v, 4) for k, v in sorted(avg.items())}}
    if rank == 0:
        share = 1.0 / world if (world == 1 or runner.shards.balance == "cells") else None
        out["roofline"], out["m2l"] = rooflines(cfg, wl, ev, avg, peaks, near_pairs, step_ms,
                                                share if share is not None else 1.0 / world)
    return out


def p2p_roofline(wl, ms, near_pairs, m, peaks):
    """The near-field kernel against the FP64 (DFMA) peak: frozen FP64 flops
    per (target, source) pair of the config's kernel functor."""
    fpp = P2P_FLOPS_PER_PAIR.get(wl["kernel"])
    pairs = near_pairs * m
    roof = {"kernel": "p2p near field (p2p_tile_kernel / p2p_kernel, FP64 pipe)", "bound": "fp64",
            "pair_interactions": pairs, "pairs_per_s": pairs / (ms * 1e-3),
            "flops_per_pair": fpp, "pair": f"(target, source) pair, all {m} column(s)"}
    if fpp is not None:
        ach = near_pairs * fpp / (ms * 1e-3) / 1e12
        ex = near_pairs * P2P_EXECUTED_PER_PAIR[wl["kernel"]] / (ms * 1e-3) / 1e12
        roof.update({"achieved": ach, "peak": peaks["dfma_tflops"], "unit": "TFLOP/s",
                     "frac": ach / peaks["dfma_tflops"],
                     "frac_of_nominal_37.2": ach / NOMINAL_FP64_TF,
                     "executed_flops_per_pair": P2P_EXECUTED_PER_PAIR[wl["kernel"]],
                     "frac_executed": ex / peaks["dfma_tflops"],
                     "peak_source": "measured live: DFMA microbenchmark "
                                    "(bfmm_device_fp64_probe); MEASURED_PEAKS.json has no "
                                    "FP64 entry"})
    return roof


def rooflines(cfg, wl, ev, avg, peaks, near_pairs, step_ms, share=1.0):
    """roofline of the dominant kernel + per-level M2L figures.  share: the
    fraction of every level's (and the near field's) work one rank does
    (1/N for the equal Morton shards of N ranks)."""
    m = wl["ncols"]
    near_pairs = near_pairs * share
    levels = {}
    if wl["scheme"] == "chebyshev":
        flops = {lev: f * share for lev, f in m2l_flops(ev, wl).items()}
        for k, v in avg.items():
            if not k.startswith("m2l_l"):
                continue
            lev = int(k.split("_l")[1])
            blk = ev._dev_block(lev)
            r, rp = ev.table.block_for_level(lev).rank, blk["rp"]
            S, bits = ev._level_digits(lev, rp, False)
            fp64 = flops[lev] / (v * 1e-3) / 1e12
            rec = {"ms": round(v, 4), "engine": ev._level_engine(lev, m, rp),
                   "rank": r, "fp64_equiv_tflops": fp64,
                   "frac_of_dmma_peak": fp64 / peaks["dmma_tflops"],
                   "traffic": committed_traffic(cfg, k)}
            executed = None
            if lev in ev.active_profile:  # sparse cloud: only the listed target cells
                cells, off = ev.active_profile[lev]
                pairs, executed = active_level_work(cells, off, lev, rp, m, S)
                flops[lev] = pairs * 2.0 * r * r * m
                fp64 = flops[lev] / (v * 1e-3) / 1e12
                rec.update({"active_cells": int(off[8]), "far_pairs": pairs,
                            "fp64_equiv_tflops": fp64,
                            "frac_of_dmma_peak": fp64 / peaks["dmma_tflops"]})
            if rec["engine"] == "i8":
                useful = flops[lev] * S * (S + 1) / 2  # digit products of the unpadded rank
                if executed is None:
                    executed = m2l_i8_ops(lev, rp, m, S) * share
                rec.update({"kernel": ("gather (active cells)" if lev in ev.active_profile
                                       else "plane pair" if _pair_kernel(lev, S)
                                       else "plane" if lev >= 4 else "gather"),
                            "digits": f"{S} x {bits}-bit",
                            "useful_int8_tops": useful / (v * 1e-3) / 1e12,
                            "executed_int8_tops": executed / (v * 1e-3) / 1e12,
                            "frac_useful": useful / (v * 1e-3) / 1e12 / peaks["i8_tops"],
                            "frac_executed": executed / (v * 1e-3) / 1e12 / peaks["i8_tops"]})
            levels[k] = rec
    else:
        flops = {lev: f * share for lev, f in fft_flops(wl).items()}
        for k, v in avg.items():
            if not k.startswith("m2lfft_l"):
                continue
            lev = int(k.split("_l")[1])
            tf = flops[lev] / (v * 1e-3) / 1e12
            levels[k] = {"ms": round(v, 4), "hadamard_tflops": tf,
                         "frac_dfma_peak": tf / peaks["dfma_tflops"],
                         "traffic": committed_traffic(cfg, k)}
    # roofline kernels: the near field and the M2L levels (the other spans --
    # p2m, m2m, projections, l2l, l2p -- are reported in kernels_ms only)
    cand = [k for k in avg if k == "p2p" or k.startswith("m2l")]
    dom = max(cand, key=avg.get) if cand else None
    if dom is None:
        return None, levels
    if dom != "p2p" and "p2p" in avg:
        # the near field's own roofline beside the dominant M2L's
        levels["p2p"] = p2p_roofline(wl, avg["p2p"], near_pairs, m, peaks)
        levels["p2p"]["traffic"] = committed_traffic(cfg, "p2p")
        levels["p2p"].update({"kernel_ms": avg["p2p"], "share_of_step": avg["p2p"] / step_ms})
    ms = avg[dom]
    share = ms / step_ms
    if dom == "p2p":
        roof = p2p_roofline(wl, ms, near_pairs, m, peaks)
    elif dom.startswith("m2lfft_l"):
        rec = levels[dom]
        roof = {"kernel": f"uniform FFT M2L level {dom.split('_l')[1]} (fft_fwd + stencil + "
                          "fft_inv)", "bound": "fp64", "achieved": rec["hadamard_tflops"],
                "peak": peaks["dfma_tflops"], "unit": "TFLOP/s",
                "frac": rec["hadamard_tflops"] / peaks["dfma_tflops"],
                "frac_of_nominal_37.2": rec["hadamard_tflops"] / NOMINAL_FP64_TF,
                "algorithmic": "Hadamard flops P_l * q^2(q/2+1) * m * 8",
                "peak_source": "measured live: DFMA microbenchmark"}
    else:
        rec = levels[dom]
        lev = dom.split("_l")[1]
        if rec["engine"] == "i8":
            kname = {"plane": "m2l_i8p_kernel", "plane pair":
                     "m2l_i8p2_kernel (CTA pair, cta_group::2)"}.get(rec["kernel"], "m2l_i8_kernel")
            roof = {"kernel": f"{kname} (M2L level {lev}, int8 tcgen05, {rec['digits']} "
                              "digits/operand)",
                    "bound": "tensor", "achieved": rec["useful_int8_tops"],
                    "peak": peaks["i8_tops"], "unit": "TFLOP/s",
                    "op_kind": "int8 tensor-core ops (1 MAC = 2), tcgen05 kind::i8",
                    "frac": rec["frac_useful"],
                    "algorithmic": "useful = P_l * 2 r^2 * m * S(S+1)/2 digit products of the "
                                   "unpadded rank",
                    "executed_int8_tops": rec["executed_int8_tops"],
                    "frac_executed": rec["frac_executed"],
                    "fp64_equiv_tflops": rec["fp64_equiv_tflops"],
                    "fp64_equiv_frac_of_dmma_peak": rec["frac_of_dmma_peak"],
                    "peak_source": "measured live: bfmm_device_i8_probe (128x256x32 kind::i8 "
                                   "MMAs back to back); MEASURED_PEAKS.json has no int8 entry"}
        else:
            roof = {"kernel": f"m2l_ws_kernel (M2L level {lev}, FP64 DMMA)", "bound": "tensor",
                    "achieved": rec["fp64_equiv_tflops"], "peak": peaks["dmma_tflops"],
                    "unit": "TFLOP/s", "frac": rec["frac_of_dmma_peak"],
                    "peak_source": "measured live: DMMA microbenchmark"}
    roof.update({"kernel_key": dom, "kernel_ms": ms, "share_of_step": share,
                 "traffic": committed_traffic(cfg, dom)})
    return roof, levels


# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import ctypes as C
    import torch

    from paper_1903_02153_b200 import _native

    # BFMM_BENCH_BACKEND=gloo with BFMM_BENCH_SHARE_GPU=1: a functional run of
    # the N-rank code path with every rank on cuda:0 and host-staged
    # exchanges (no kernel waits on another rank; its timing means nothing)
    backend = os.environ.get("BFMM_BENCH_BACKEND", "nccl")
    if os.environ.get("BFMM_BENCH_SHARE_GPU"):
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
        assert dist.get_world_size() == world == args.gpus, (dist.get_world_size(), args.gpus)
    lib = _native.load()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    peaks = device_peaks(lib, stream) if rank == 0 else None
    res = measure(args.config, args, rank, world, local_rank, dist, lib, peaks,
                  args.steps, args.warmup, with_e2e=not args.no_e2e)
    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    wl = res["wl"]
    res.pop("ev")  # free the primary config's device memory before the secondary
    torch.cuda.empty_cache()

    secondary = None
    if world == 1 and args.secondary and args.secondary.lower() != "none" \
            and args.secondary != args.config:
        s = measure(args.secondary, args, 0, 1, local_rank, None, lib, peaks,
                    min(args.steps, 10), args.warmup, with_e2e=False)
        secondary = {"config": config_dict(s["wl"]), "value": s["value"], "unit": "points/s",
                     "ms_per_step": s["step_ms"], "steps": min(args.steps, 10),
                     "roofline": s["roofline"], "kernels_ms": s["kernels_ms"],
                     "m2l_levels": s["m2l"], "clocks": s["clocks"],
                     "gpu_launches": s["launches"]}
        s.pop("ev")
        del s
        torch.cuda.empty_cache()

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        scale = REF_SCALE.get(args.config, 0) if args.ref_scale is None else args.ref_scale
        try:
            ref = ReferenceSample(args.config, scale, cpu_threads())
            ref.step()  # warm: tables and first-touch
            secs = [ref.step() for _ in range(2)]
            cpu = {"value": ref.n * len(secs) / sum(secs), "unit": "points/s",
                   "cores": ref.threads, "kind": "reference",
                   "sample": ref.desc + f"; {len(secs)} timed evaluates, "
                                        f"{sum(secs):.1f} s"}
        except RuntimeError as e:
            cpu = {"value": None, "unit": "points/s", "cores": None, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    ev_m2l = dict(res["m2l"] or {})
    p2p_roof = ev_m2l.pop("p2p", None)
    line = {
        "metric": METRIC, "value": res["value"], "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["step_ms"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SURVEY.md §8(d) recipe)",
        "config": config_dict(wl),
        "engine": {"m2l": "int8 tcgen05 (error-free digit splitting) where rank <= 256, "
                          "else FP64 DMMA" if wl["scheme"] == "chebyshev" else "FFT Hadamard",
                   "near_field": "own stream, overlaps kernel tails",
                   "parallelism": f"dp{world}: Morton-range target shards" if world > 1
                   else "single GPU"},
        "roofline": res["roofline"], "p2p_roofline": p2p_roof, "cpu_baseline": cpu,
        "e2e": res["e2e"], "e2e_numpy": res["e2e_numpy"],
        "gpu_launches": int(res["launches"]), "clocks": res["clocks"],
        "stages_ms": res["stages_ms"], "stages_serial_ms": res["stages_serial_ms"],
        "kernels_ms": res["kernels_ms"], "m2l_levels": ev_m2l,
        "peaks": dict(peaks, source="measured live in this process (libbfmm.so probes)"),
        "secondary": secondary,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def spawn(args):
    """--gpus N without a torchrun environment: launch N ranks ourselves."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        if world != args.gpus:
            raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
