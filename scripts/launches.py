"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch).

    python scripts/launches.py launches.csv            # per-step breakdown
    python scripts/launches.py launches.csv --all      # every launch

A matvec step starts at its tree build (the first leaf_keys_kernel); the
summary takes the median-duration complete step, so warm-up, probe and
end-to-end launches outside the step are excluded.  ncu launches are
serialised and cold-cache: compare SHARES of the step, not absolute times.
"""
import collections
import csv
import sys


def read(path):
    hdr, out = None, []
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                unit = d.get("Metric Unit", "ns")
                v = float(d["Metric Value"].replace(",", ""))
                v *= {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1.0)
                out.append((int(d["ID"]), d["Kernel Name"], v))
    return out


def short(name):
    base = name.split("(")[0]
    return base.replace("bfmm::<unnamed>::", "").replace("bfmm_nf::", "")[-70:]


def steps(launches):
    starts = [i for i, (_, k, _) in enumerate(launches) if "leaf_keys_kernel" in k]
    out = []
    for a, b in zip(starts, starts[1:]):
        out.append(launches[a:b])
    return out


def main():
    path = sys.argv[1]
    launches = read(path)
    if "--all" in sys.argv:
        for i, k, t in launches:
            print(i, f"{t / 1e3:9.1f} us", short(k))
        return
    st = steps(launches)
    if not st:
        print("no complete step found")
        return
    st.sort(key=lambda s: sum(t for _, _, t in s))
    step = st[len(st) // 2]
    tot = sum(t for _, _, t in step)
    agg = collections.defaultdict(lambda: [0.0, 0])
    for _, k, t in step:
        agg[short(k)][0] += t
        agg[short(k)][1] += 1
    print(f"# {path}: median of {len(st)} complete steps, {len(step)} launches, "
          f"{tot / 1e3:.1f} us serialised")
    print(f"{'us':>9} {'share':>6} {'n':>3}  kernel")
    for k, (t, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{t / 1e3:9.1f} {100 * t / tot:5.1f}% {n:3d}  {k}")


if __name__ == "__main__":
    main()
