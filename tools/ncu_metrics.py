"""Per-kernel ncu figures for bench.py's roofline block -> profiles/ncu_metrics.json.

    python tools/ncu_metrics.py REPORT.ncu-rep NAME=REGEX:ATOMS [...] --source TEXT

Each NAME=REGEX:ATOMS averages the launches whose kernel name matches REGEX
(one launch of ATOMS owned atoms each) and stores, per launch: duration,
DRAM bytes (read + write), L1TEX data-pipe wavefront %, FP64-pipe %, warps
active %, executed FP64 flops (2 DFMA + DADD + DMUL thread instructions).  A
NAME starting with "sum:" adds the matching kernels' per-launch figures
(e.g. the three SNAP kernels of one force evaluation) and also stores
dflop_per_atom.  Existing entries of the JSON are kept unless overwritten.
The capture needs the metrics named in METRICS (`--set full` plus
`--metrics` for the sass op counters).
"""

from __future__ import annotations

import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_metrics.json")
METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "l1tex_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dfma": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "dadd": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dmul": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "l2_sectors": "lts__t_sectors.sum",
}
SCALE = {"usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3, "us": 1.0, "ms": 1e3, "ns": 1e-3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "%": 1.0, "": 1.0, "inst": 1.0, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}


def rows(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    for v in r[2:]:
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))
        rec = {"name": d.get("Kernel Name", "")}
        for key, m in METRICS.items():
            if d.get(m, "") not in ("", "n/a"):
                rec[key] = float(d[m].replace(",", "")) * SCALE.get(u.get(m, ""), 1.0)
        yield rec


def summarize(recs, atoms):
    n = len(recs)
    avg = {k: sum(r.get(k, 0.0) for r in recs) / n for k in METRICS}
    out = {"launches": n, "n_atoms": atoms, "duration_us": avg["duration_us"],
           "dram_bytes": avg["dram_read"] + avg["dram_write"], "l1tex_wavefront_pct": avg["l1tex_wavefront_pct"],
           "fp64_pipe_pct": avg["fp64_pipe_pct"], "warps_active_pct": avg["warps_active_pct"],
           "dflop": 2 * avg["dfma"] + avg["dadd"] + avg["dmul"], "l2_bytes": 32.0 * avg["l2_sectors"]}
    return out


def main(argv):
    report, specs, source = argv[0], [], ""
    it = iter(argv[1:])
    for a in it:
        if a == "--source":
            source = next(it)
        else:
            specs.append(a)
    recs = list(rows(report))
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for spec in specs:
        name, rest = spec.split("=", 1)
        rx, atoms = rest.rsplit(":", 1)
        atoms = int(atoms)
        if name.startswith("sum:"):
            name = name[4:]
            parts = {}
            for r in recs:
                m = re.search(rx, r["name"])
                if m:
                    parts.setdefault(m.group(0), []).append(r)
            tot = {"launches": 0, "n_atoms": atoms, "duration_us": 0.0, "dram_bytes": 0.0, "dflop": 0.0,
                   "kernels": {}}
            for k, rs in parts.items():
                s = summarize(rs, atoms)
                tot["kernels"][k] = s
                for f in ("duration_us", "dram_bytes", "dflop"):
                    tot[f] += s[f]
                tot["launches"] += 1
            tot["dflop_per_atom"] = tot["dflop"] / atoms
            tot["source"] = source
            data[name] = tot
        else:
            sel = [r for r in recs if re.search(rx, r["name"])]
            if not sel:
                print(f"no launch matches {rx}", file=sys.stderr)
                continue
            s = summarize(sel, atoms)
            s["source"] = source
            data[name] = s
        print(name, json.dumps(data[name])[:300])
    with open(OUT, "w") as fh:
        json.dump(data, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
