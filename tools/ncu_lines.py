"""Aggregate executed warp instructions and stall samples of an ncu report by
CUDA source line: python tools/ncu_lines.py report.ncu-rep [top]."""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
inst, samp, text = defaultdict(float), defaultdict(float), {}
fname, hdr = None, None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0].isdigit():
        continue
    key = (fname, int(row[0]))
    text[key] = row[1].strip()[:70]
    try:
        inst[key] += float(row[hdr.index("Instructions Executed")] or 0)
        samp[key] += float(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        pass
tot_i, tot_s = sum(inst.values()) or 1, sum(samp.values()) or 1
print(f"total warp instructions {tot_i:.3e}")
for k in sorted(inst, key=lambda k: -inst[k])[:top]:
    print(f"{100*inst[k]/tot_i:5.1f}% inst {100*samp[k]/tot_s:5.1f}% stall  {k[0]}:{k[1]}  {text.get(k,'')}")
