import csv, subprocess, sys, io, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]; units = rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_bytes.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum"]
stall_keys = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled_") or h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("##", d.get("Kernel Name", "")[:90])
    for w in want:
        if w in d: print(f"  {w} = {d[w]} {units[hdr.index(w)]}")
    st = []
    for k in stall_keys:
        try: st.append((float(d[k]), k))
        except: pass
    st.sort(reverse=True)
    print("  stalls:", ", ".join(f"{k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')}={v:.2f}" for v, k in st[:6]))
