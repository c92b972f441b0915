"""Summarise an ncu report: key metrics + top SASS stall sites (used to write profiles/)."""
import csv, subprocess, sys, io

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.max", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__cluster_dim_x",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    for k in keys:
        if k in h:
            i = h.index(k)
            print(f"{k:60s} {r[i]} {units[i]}")
    print("stall (warps per issue-active cycle):")
    st = [(k, r[i]) for i, k in enumerate(h) if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    st = sorted(((float(v or 0), k) for k, v in st), reverse=True)[:10]
    for v, k in st:
        print(f"   {k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''):28s} {v:.2f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((r[si].strip(), int(r[wi] or 0), int(r[ei] or 0)))
    except (ValueError, IndexError):
        pass
tw = sum(d[1] for d in data) or 1
print(f"SASS: {len(data)} instructions, top stall sites:")
for s, w, e in sorted(data, key=lambda d: -d[1])[:top]:
    print(f"  {100*w/tw:5.1f}%  {s[:80]}")
