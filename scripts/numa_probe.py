"""Pinned H2D bandwidth per NUMA node / CPU affinity (diagnostic)."""
import os, subprocess, sys, time
import torch
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[-800:])
print("affinity", sorted(os.sched_getaffinity(0))[:8], "... n =", len(os.sched_getaffinity(0)))
bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip().lower()
path = f"/sys/bus/pci/devices/{bus[4:] if bus.count(':') == 2 and len(bus.split(':')[0]) == 8 else bus}"
for cand in (path, path.replace("0000", "00000000", 1)):
    for f in ("local_cpulist", "numa_node"):
        try:
            print(f, open(os.path.join(cand, f)).read().strip())
        except OSError:
            pass
def bw(tag):
    x = torch.empty(64 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
    x.fill_(1.0)
    d = torch.empty_like(x, device="cuda")
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(x, non_blocking=True); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    y = torch.empty_like(x).pin_memory()
    ts2 = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter(); y.copy_(d, non_blocking=True); torch.cuda.synchronize(); ts2.append(time.perf_counter() - t0)
    print(tag, "H2D %.1f GB/s  D2H %.1f GB/s" % (64 * 1.048576e6 / min(ts) / 1e9, 64 * 1.048576e6 / min(ts2) / 1e9), flush=True)
_dummy = torch.empty(1 << 19, dtype=torch.float64).pin_memory()  # 4 MiB, kept alive
if len(sys.argv) > 1:  # one H2D copy from the sacrificial buffer first
    _dd = torch.empty_like(_dummy, device="cuda")
    _dd.copy_(_dummy); torch.cuda.synchronize()
bw("default")
bw("default again")
bw("default third")
ncpu = os.cpu_count()
for half in (0, 1):
    cpus = set(range(half * ncpu // 2, (half + 1) * ncpu // 2))
    os.sched_setaffinity(0, cpus)
    bw(f"cpus {min(cpus)}-{max(cpus)}")
