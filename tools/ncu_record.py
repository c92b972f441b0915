"""Merge one kernel's ncu --set full counters into profiles/ncu_traffic.json
(read by bench.py's roofline block: DRAM bytes per launch + limiter).

usage: python tools/ncu_record.py REPORT.ncu-rep WORKLOAD PRECISION KERNEL [SOURCE-NOTE] [--sum]
KERNEL matches the demangled kernel name by substring; launches of it in the
report are averaged, or with --sum added up (the launches one run makes of
it: C4's main launch and its tail-wave launch), percentages time-weighted."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "time": "gpu__time_duration.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_pct": "dram__bytes_read.sum.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
         "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1,
         "%": 1, "": 1}


def main():
    args = [a for a in sys.argv[1:] if a != "--sum"]
    add = "--sum" in sys.argv
    rep, workload, precision, kname = args[:4]
    note = args[4] if len(args) > 4 else os.path.basename(rep)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    sel = [r for r in rows[2:] if kname in r[ki]]
    if not sel:
        raise SystemExit(f"no launch of {kname} in {rep}")
    rec = {}
    ti = h.index(KEYS["time"])
    times = [float(r[ti].replace(",", "")) * SCALE.get(units[ti], 1) for r in sel]
    for key, metric in KEYS.items():
        if metric not in h:
            continue
        i = h.index(metric)
        vals = [float(r[i].replace(",", "")) * SCALE.get(units[i], 1) for r in sel]
        if key.endswith("_pct"):  # time-weighted over the launches
            rec[key] = sum(v * t for v, t in zip(vals, times)) / sum(times)
        else:
            rec[key] = sum(vals) if add else sum(vals) / len(vals)
    out = {"dram_bytes": int(rec.get("dram_read", 0) + rec.get("dram_write", 0)),
           "time_ms_cold": round(rec["time"] * 1e3, 4), "launches": len(sel)}
    for k in ("issue_active_pct", "l1tex_pct", "lts_pct", "dram_pct", "warps_active_pct",
              "l2_hit_pct"):
        if k in rec:
            out[k] = round(rec[k], 1)
    units_ = {"issue_active_pct": "instruction issue", "l1tex_pct": "L1/TEX (SMEM, DSMEM, LSU)",
              "lts_pct": "L2", "dram_pct": "DRAM reads"}
    top = max(units_, key=lambda k: out.get(k, 0))
    out["limiter"] = (f"{units_[top]} at {out[top]}% of peak (issue-active "
                      f"{out.get('issue_active_pct')}%, L1/TEX {out.get('l1tex_pct')}%, L2 "
                      f"{out.get('lts_pct')}%, DRAM {out.get('dram_pct')}%)")
    out["source"] = note
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    db = json.load(open(path)) if os.path.exists(path) else {}
    db.setdefault(workload, {}).setdefault(precision, {})[kname] = out
    with open(path, "w") as f:
        json.dump(db, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
