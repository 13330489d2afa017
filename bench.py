#!/usr/bin/env python
"""FMM matvec throughput (points/s, fp64) on B200 — the BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2] [--no-cpu-baseline] [--no-graph]

Workload (N=1): BASELINE.json configs[1] = C2 (Gaussian exp(-(r/0.2)^2),
N = 1,000,000 uniform in [-1,1]^3, L=5, Chebyshev p=5, eps 1e-7, 1 RHS),
seeded synthetic inputs; the other configs are parity
cases (tests/).  A step is one full matvec phi = K sigma: tree build, P2M,
M2M, M2L, L2L, L2P, P2P, output scatter.

* value     device-resident inputs, CUDA-event time of K steps, L2 flushed
            (256 MiB write) between steps outside the timed spans.
* e2e       the public API on pinned host tensors: H2D of points + weights,
            the matvec, D2H of phi, every step.
* roofline  the dominant kernel (largest share of the step), timed live
            with CUDA events on its launching stream; FP64 peak measured live
            (DMMA/DFMA microbenchmarks in libbfmm.so: MEASURED_PEAKS.json has
            no FP64 entry).
* cpu_baseline  the CPU oracle (oracle/fmm_oracle.py, a NumPy restatement of
            the reference's engine with its thread pool) on the same C2
            inputs, timed on this host's cores, rank 0 at N=1 only.
* --impl reference  the same oracle as the reference arm (the reference is
            pure Python and not present on the GPU box; the oracle is pinned
            to its outputs by tests/test_oracle_golden.py).
* N > 1: target leaves are split by Morton range across ranks (one process
  per GPU, NCCL); each rank evaluates its share, phi is all-gathered.
"""

from __future__ import annotations

import argparse
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

# FP64 flops per near-field pair interaction, frozen from ncu instruction
# counts of the P2P kernel (2*DFMA + DMUL + DADD thread instructions / pair,
# profiles/r01_p2p_flops.txt); kernel-specific.
P2P_FLOPS_PER_PAIR = {"gauss02": 40.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of CUDA-graph replay")
    ap.add_argument("--balance", default="auto", choices=["auto", "cells", "work"],
                    help="N>1 shard ranges: equal cell ranges, work-weighted, or auto "
                         "(work-weighted for the clustered C4)")
    return ap.parse_args()


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


def make_workload(name):
    from paper_1903_02153_b200 import workloads
    return workloads.make(name)


def config_dict(wl):
    from paper_1903_02153_b200 import workloads
    return {"workload": f"{wl['name']}: {workloads.DESCRIPTION[wl['name']]}",
            "n_points": int(wl["points"].shape[0]), "levels": wl["levels"],
            "order": wl["order"], "scheme": wl["scheme"], "eps": wl["eps"],
            "kernel": wl["kernel"], "ncols": wl["ncols"],
            "l2": "flushed between steps (256 MiB write, outside the timed spans)"}


def oracle_step(wl, threads):
    from oracle import fmm_oracle as O
    from paper_1903_02153_b200.kernel import workload_kernel
    fmm = O.OracleFMM(workload_kernel(wl["kernel"]), wl["levels"], wl["order"],
                      wl["scheme"], wl["eps"], wl["center"], wl["length"], threads=threads)
    t0 = time.perf_counter()
    fmm.matvec(wl["points"], weights=wl["weights"])
    return time.perf_counter() - t0


def cpu_threads():
    try:
        import psutil
        return max(1, psutil.cpu_count(logical=False) or os.cpu_count() or 1)
    except Exception:
        return max(1, os.cpu_count() or 1)


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle (reference algorithm, NumPy, thread pool)
    on the host cores; rank 0 only."""
    if rank != 0:
        return
    wl = make_workload(args.config)
    threads = cpu_threads()
    for _ in range(args.warmup):
        oracle_step(wl, threads)
    times = [oracle_step(wl, threads) for _ in range(args.steps)]
    total = sum(times)
    n = wl["points"].shape[0]
    value = n * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SURVEY.md §8(d) recipe)",
        "config": config_dict(wl),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads, "kind": "port",
                         "sample": f"full {args.config} matvec per step (oracle/fmm_oracle.py)"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def fp64_peaks(lib, stream):
    import ctypes as C
    g1, g2 = C.c_double(0), C.c_double(0)
    lib.bfmm_device_fp64_probe(C.byref(g1), stream)
    lib.bfmm_device_dmma_probe(C.byref(g2), stream)
    return g1.value / 1e3, g2.value / 1e3  # TFLOP/s


def committed_traffic(config, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/r01_traffic.json), or None when that kernel was not captured."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_traffic.json")
    try:
        with open(path) as f:
            rec = json.load(f).get(config, {}).get(kernel)
    except (OSError, ValueError):
        return None
    return None if rec is None else rec["bytes"]


def m2l_flops(ev, wl):
    """Algorithmic M2L flops per level: pairs P_l * 2 r_l^2 * m."""
    from paper_1903_02153_b200.tables import OFFSETS
    out = {}
    m = wl["ncols"]
    for lev in range(2, wl["levels"] + 1):
        n = 1 << lev
        pairs = 1
        cnt = 0
        for t in OFFSETS:
            c = 1
            for a in range(3):
                tt = int(t[a])
                lo, hi = max(0, -tt), min(n - 1, n - 1 - tt)
                k = max(0, hi - lo + 1)
                if abs(tt) == 3:
                    k = len([x for x in range(lo, hi + 1) if (x % 2 == 0) == (tt > 0)])
                c *= k
            cnt += c
        blk = ev.table.block_for_level(lev)
        r = blk.rank
        out[lev] = cnt * 2.0 * r * r * m
        del pairs
    return out


def _valid_offsets(o):
    """The 189 offsets a child octant admits (octree.py:128-145 parity rule)."""
    from paper_1903_02153_b200.tables import OFFSETS
    bits = ((o >> 2) & 1, (o >> 1) & 1, o & 1)
    out = []
    for t in OFFSETS:
        if all(not ((int(t[a]) == 3 and bits[a]) or (int(t[a]) == -3 and not bits[a]))
               for a in range(3)):
            out.append(tuple(int(x) for x in t))
    return out


def m2l_i8_ops(lev, rp, m, S):
    """int8 operations the tcgen05 M2L executes at one level: per (tile,
    offset, 32-wide k chunk, 64-wide rank tile) stage, S(S+1)/2 digit
    products of 128 x 64 x 32 (csrc/m2l_i8.cuh).  Dense levels >= 4 use the
    plane kernel, which skips offset groups whose source planes leave the
    grid; coarser levels run all 316 offsets over mixed-octant row tiles
    (zero rows where the parity rule or the grid excludes a pair)."""
    n = 1 << lev
    kc, ntn = -(-rp // 32), -(-rp // 64)
    per_stage = 2.0 * 128 * 64 * 32 * S * (S + 1) / 2
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
                # a group (offsets sharing t_x) runs when any x slot's plane is inside
                live = sum(1 for t in offs if xs + t[0] + 2 * (xt - 1) >= 0 and xs + t[0] < n)
                stages += live * (h // yt) * (h // 8)
    else:  # levels <= 3: one mixed-octant row set over all 316 offsets
        stages = -(-(n ** 3 * m) // 128) * 316
    return stages * kc * ntn * (m if lev >= 4 else 1) * per_stage


def run_ours(args, rank, world, local_rank):
    import ctypes as C
    import torch

    import paper_1903_02153_b200 as bf
    from paper_1903_02153_b200 import _native
    from paper_1903_02153_b200.kernel import workload_kernel

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    wl = make_workload(args.config)
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"],
                      eps=wl["eps"], domain_center=wl["center"], domain_length=wl["length"],
                      n_cols=wl["ncols"])
    kernel = workload_kernel(wl["kernel"])
    ev = bf.FmmEvaluator(kernel, plan, cache_dir=os.path.join("/tmp", "bfmm_bench_cache"))
    # whole device step replayed from a CUDA graph (FmmEvaluator.use_graph;
    # captured during warm-up, eager path for the per-kernel timing pass)
    ev.use_graph = not args.no_graph
    lib = _native.load()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    n = wl["points"].shape[0]
    m = wl["ncols"]
    X = torch.from_numpy(wl["points"]).cuda()
    W = torch.from_numpy(np.ascontiguousarray(wl["weights"])).cuda()
    if world > 1:
        from paper_1903_02153_b200.parallel import ShardedEvaluator
        balance = args.balance if args.balance != "auto" else (
            "work" if args.config == "C4" else "cells")
        runner = ShardedEvaluator(ev, dist, balance=balance)
        step = lambda x, w: runner.evaluate(x, weights=w)  # noqa: E731
    else:
        runner = ev
        step = lambda x, w: ev.evaluate(x, weights=w)  # noqa: E731
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def measure_e2e():
        # ---- e2e through the public API with pinned host tensors ----
        Xh = torch.from_numpy(wl["points"]).pin_memory()
        Wh = torch.from_numpy(np.ascontiguousarray(wl["weights"])).pin_memory()
        phi = None
        for _ in range(max(3, args.warmup)):
            # keep the previous result alive, as in the timed loop, so both pinned
            # output blocks of the host caching allocator exist before timing
            phi = runner.evaluate(Xh, weights=Wh)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e2e_ms = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            phi = runner.evaluate(Xh, weights=Wh)
            assert phi.device.type == "cpu"
            e2e_ms.append(1e3 * (time.perf_counter() - t0))
        e2e_total = float(sum(e2e_ms))
        if dist is not None:
            t = torch.tensor([e2e_total], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_total = float(t.item())
        e2e_value = n * args.steps / (e2e_total * 1e-3)
        return Xh, Wh, e2e_ms, e2e_total, e2e_value

    # measured first: after the device-resident loop below the same calls took
    # 3.7-4.4 ms instead of 3.5 on some boxes (a process-state effect we could
    # not pin down: not the pinned-copy bandwidth, which stays at ~54 GB/s)
    Xh, Wh, e2e_ms, e2e_total, e2e_value = measure_e2e()
    for _ in range(args.warmup):
        step(X, W)
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.bfmm_launch_count() + ev.graph_launches
    spans, kms, stage_sum = [], [], {}
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        step(X, W)
        e1.record()
        e1.synchronize()
        spans.append(e0.elapsed_time(e1))
        for k, v in ev.timings.items():
            if isinstance(v, float):
                stage_sum[k] = stage_sum.get(k, 0.0) + v
    torch.cuda.synchronize()
    launches = lib.bfmm_launch_count() + ev.graph_launches - launches0
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    total_ms = float(sum(spans))
    # per-kernel times for the roofline: a separate pass with CUDA events
    # around each launch on its own stream, near field NOT overlapped (the
    # timed steps above overlap it with the far field, which would charge
    # the SM sharing to both kernels)
    ov = ev.overlap_near
    ev.overlap_near, ev.profile_kernels = False, True
    for _ in range(args.steps):
        flush.zero_()
        step(X, W)
        torch.cuda.synchronize()
        kms.append(dict(ev.kernel_ms))
    ev.overlap_near, ev.profile_kernels = ov, False
    if dist is not None:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = n * args.steps / (total_ms * 1e-3)


    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----
    dfma_tf, dmma_tf = fp64_peaks(lib, stream)
    avg = {}
    for d in kms:
        for k, v in d.items():
            avg[k] = avg.get(k, 0.0) + v / len(kms)
    dom = max(avg, key=avg.get) if avg else None
    roof = None
    if dom is not None:
        ms = avg[dom]
        if dom == "p2p":
            fpp = P2P_FLOPS_PER_PAIR.get(wl["kernel"])
            pairs = ev.timings["near_pairs"] * m
            flops = pairs * fpp
            peak = dfma_tf
            roof = {"kernel": "p2p (near field, FP64 pipe)", "bound": "fp64",
                    "flops_per_pair": fpp, "pair_interactions": pairs,
                    "pairs_per_s": pairs / (ms * 1e-3),
                    "flops_note": "frozen algorithmic figure (profiles/r01_p2p_flops.txt); "
                                  "the current kernel executes ~32 FP64 flops per pair"}
        else:
            lev = int(dom.split("_l")[1])
            flops = m2l_flops(ev, wl)[lev]
            peak = dmma_tf
            roof = {"kernel": f"m2l level {lev} ({ev.m2l_mode} implicit GEMM)",
                    "bound": "fp64-tensor"}
        achieved = flops / (ms * 1e-3) / 1e12
        roof.update({"achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": committed_traffic(args.config, dom),
                     "peak_source": "measured live: DFMA / DMMA microbenchmarks (libbfmm.so); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "kernel_ms": ms, "share_of_step": ms / (total_ms / args.steps)})
    m2l = m2l_flops(ev, wl)
    kernels = {k: round(v, 4) for k, v in sorted(avg.items())}
    m2l_frac = {k: (m2l[int(k.split("_l")[1])] / (v * 1e-3) / 1e12) / dmma_tf
                for k, v in avg.items() if k.startswith("m2l_l")}
    # the int8 tensor-core M2L against its own roofline: executed int8 ops
    # per launch / launch time vs the measured tcgen05 kind::i8 peak
    m2l_roof = None
    if ev.m2l_mode == "i8" and wl["scheme"] == "chebyshev":
        i8_peak = C.c_double(0)
        lib.bfmm_device_i8_probe(C.byref(i8_peak), stream)
        S = int(ev.i8_slices)
        m2l_roof = {"engine": f"int8 tcgen05, {S} digits per operand",
                    "peak_int8_tops": i8_peak.value,
                    "peak_source": "measured live: bfmm_device_i8_probe (128x256x32 MMAs "
                                   "back to back)", "levels": {}}
        for k, v in avg.items():
            if not k.startswith("m2l_l"):
                continue
            lev = int(k.split("_l")[1])
            rp = ev._dev_block(lev)["rp"]
            ops = m2l_i8_ops(lev, rp, m, S)
            fp64 = m2l[lev] / (v * 1e-3) / 1e12
            m2l_roof["levels"][k] = {
                "ms": round(v, 4), "kernel": "plane" if lev >= 4 else "gather",
                "int8_tops": ops / (v * 1e-3) / 1e12,
                "frac_int8_peak": ops / (v * 1e-3) / 1e12 / i8_peak.value,
                "fp64_equiv_tflops": fp64, "frac_of_dmma_peak": fp64 / dmma_tf,
                "traffic": committed_traffic(args.config, k)}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = cpu_threads()
        secs = oracle_step(wl, threads)
        cpu = {"value": n / secs, "unit": "points/s", "cores": threads, "kind": "port",
               "sample": f"one full {args.config} matvec (oracle/fmm_oracle.py, {secs:.1f} s)"}

    h2d = int(Xh.numel() * 8 + Wh.numel() * 8)
    d2h = int(n * m * 8)
    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SURVEY.md §8(d) recipe)",
        "config": config_dict(wl),
        "engine": {"m2l": (f"int8 tcgen05, {ev.i8_slices} digits" if ev.m2l_mode == "i8"
                           else "fp64 dmma"),
                   "near_field": ("own stream, overlaps kernel tails" if ev.overlap_near
                                  else "serial"),
                   "cuda_graph": bool(ev.use_graph)},
        "roofline": roof, "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_total / args.steps,
                "step_ms": [round(x, 3) for x in e2e_ms]},
        "gpu_launches": int(launches), "clocks": clk,
        "stages_ms": {k: round(1e3 * v / args.steps, 4) for k, v in stage_sum.items()},
        "kernels_ms": kernels,
        "m2l_frac_of_dmma_peak": {k: round(v, 3) for k, v in m2l_frac.items()},
        "m2l_roofline": m2l_roof,
        "fp64_peaks_tflops": {"dfma": dfma_tf, "dmma": dmma_tf},
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
