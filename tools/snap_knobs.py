"""compute_ui / compute_yi time per schedule knob (batch_u, batch_y) on a SNAP W bcc
system, 2J=8 (CUDA events, 5 repetitions after a warm-up)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2508_13523_b200 import Box, RankedSystem, build_all
from paper_2508_13523_b200.driver.simulation import lattice_positions
from paper_2508_13523_b200.snap import SnapState, build_neighbor_map, compute_ui, compute_yi, make_coupling_tables

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 40
pos, box = lattice_positions("bcc", 3.1803, (cells,) * 3)
rng = np.random.default_rng(5)
pos = (pos + rng.normal(0.0, 0.05, pos.shape)) % box.lengths
system = RankedSystem.distribute(box, 1, pos, np.zeros_like(pos))
(nl,) = build_all(system, 4.73, 0.3, style="full", newton=False)
store = system.stores[0]
nmap = build_neighbor_map(store, nl, 4.73)
tables = make_coupling_tables(4)   # jmax = 4 (2J = 8)
beta = np.linspace(0.05, 0.1, len(tables.triples))


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


print(f"atoms {store.n_local}")
for bu in (1, 2, 4, 8):
    st = SnapState(tables, store.n_local, beta, batch_u=bu)
    print(f"batch_u={bu}: compute_ui {timed(lambda: compute_ui(nmap, st)):.3f} ms")
for by in (1, 2):
    st = SnapState(tables, store.n_local, beta, batch_y=by)
    compute_ui(nmap, st)
    print(f"batch_y={by}: compute_yi {timed(lambda: compute_yi(st)):.3f} ms")
