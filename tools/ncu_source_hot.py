"""Hottest CUDA source lines of a kernel capture (ncu --import-source on, -lineinfo).

    python tools/ncu_source_hot.py REPORT.ncu-rep [N]

Aggregates `ncu --page source --print-source cuda,sass` per CUDA line: warp-stall
samples and warp instructions executed, top N by samples.
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
path, hdr, recs = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr is not None and r[0].isdigit() and len(r) == len(hdr):
        d = dict(zip(hdr[4:], r[4:]))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            ins = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        if s or ins:
            recs.append((s, ins, f"{path}:{r[0]}", r[1].strip()[:90]))
tot_s = sum(r[0] for r in recs) or 1
tot_i = sum(r[1] for r in recs) or 1
print(f"samples {tot_s}, warp instructions {tot_i}")
for s, ins, where, src in sorted(recs, reverse=True)[:top]:
    print(f"{100 * s / tot_s:5.1f}% smp {100 * ins / tot_i:5.1f}% ins  {where:18s} {src}")
