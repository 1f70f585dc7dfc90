"""Saturation sweep (the paper's Fig. 2 claim) on one B200.

Writes profiles/<tag>_saturation_{lj,snap}.csv and prints the rates and band entries.
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2508_13523_b200.driver.bench import bench_saturation

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
sizes = [1000, 4096, 15625, 64000, 250047, 1000000, 4096000, 10077696]
out = {}
for pot in ("lj", "snap"):
    t0 = time.perf_counter()
    res = bench_saturation(pot, sizes, reps=3, csv_path=f"profiles/{tag}_saturation_{pot}.csv")
    rates = res.rates
    plateau = rates[-2:].max()
    k = int(np.argmax(rates >= 0.9 * plateau))
    out[pot] = res.sizes[k]
    print(f"{pot}: {time.perf_counter() - t0:.0f}s  band entry at n={res.sizes[k]} (plateau {plateau:.3e} atom-steps/s)")
    for n, r in res.rows:
        print(f"   {n:>9d}  {r:.4e}")
print("entry sizes:", out)
