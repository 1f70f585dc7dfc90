"""Saturation benchmark: atom-steps/s across system sizes on the GPU (mdkk/driver/bench.py:1-148).

Same protocol as the reference: a zero-temperature simple-cubic crystal (forces
cancel by symmetry, nothing moves, lists never rebuild), so a timed step is the
steady-state cost (kick + drift + skin check, halo refresh, force, kick).  All
sizes are built first and timed round-robin, best of `reps`.  On the GPU a
step ends with the skin-check read-back, so wall time per trial is the
device-synchronised step time.
"""

from __future__ import annotations

import contextlib
import csv
import gc
import time

import numpy as np
import torch

from .simulation import LJStyle, RunConfig, RunError, Simulation, lattice_positions

_POTENTIALS = ("lj", "snap")

# the reference's setups (mdkk/driver/bench.py:24-27)
_LJ_SETUP = {"rho": 0.8, "r_c": 1.6, "skin": 0.3, "list_style": "half"}
_SNAP_SETUP = {"rho": 0.8, "r_c": 1.2, "skin": 0.25, "list_style": "full"}
_SNAP_JMAX = 1.0


class BenchResult:
    """Per-size throughput rows for one potential (mdkk/driver/bench.py:30-51)."""

    def __init__(self, potential: str, rows: list[tuple[int, float]]):
        self.potential = potential
        self.rows = rows

    @property
    def rates(self) -> np.ndarray:
        return np.array([r for _, r in self.rows])

    @property
    def sizes(self) -> np.ndarray:
        return np.array([n for n, _ in self.rows])

    def write_csv(self, path: str) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["n_atoms", "atom_steps_per_second"])
            for n, rate in self.rows:
                w.writerow([n, f"{rate:.6g}"])


def _snap_beta(jmax: float) -> np.ndarray:
    from ..snap import QuantumIndex
    return np.linspace(0.05, 0.1, len(QuantumIndex(jmax).triples()))


def _make_sim(potential: str, n_request: int, device=None) -> Simulation:
    setup = _LJ_SETUP if potential == "lj" else _SNAP_SETUP
    c = max(2, round(n_request ** (1.0 / 3.0)))
    a = (1.0 / setup["rho"]) ** (1.0 / 3.0)
    c_min = int(np.ceil(2.0 * (setup["r_c"] + setup["skin"]) / a))
    if c < c_min:
        raise RunError(f"bench size {n_request} too small: the {potential} halo "
                       f"needs at least a {c_min}^3 = {c_min ** 3} atom cube")
    sim = Simulation(RunConfig(list_style=setup["list_style"], skin=setup["skin"], device=device), log=None)
    pos, box = lattice_positions("sc", setup["rho"], (c, c, c))
    sim.box = box
    sim._positions = pos
    sim._velocities = np.zeros_like(pos)
    sim.dt = 1e-6
    if potential == "lj":
        style = LJStyle(setup["r_c"])
        style.set_coeff(1.0, 1.0)
    else:
        from ..snap.style import SnapStyle
        style = SnapStyle(setup["r_c"], _SNAP_JMAX, _snap_beta(_SNAP_JMAX), batch_u=1, tile_v=4096)
    sim.style = style
    sim._ensure_system()
    sim._forces_device()
    return sim


@contextlib.contextmanager
def _no_gc():
    was = gc.isenabled()
    gc.disable()
    try:
        yield
    finally:
        if was:
            gc.enable()


def _time_steps(sim: Simulation, n_steps: int) -> float:
    torch.cuda.synchronize(sim.device)
    t0 = time.perf_counter()
    sim.advance(n_steps)
    torch.cuda.synchronize(sim.device)
    return time.perf_counter() - t0


def bench_saturation(potential: str, sizes, reps: int = 3, csv_path: str | None = None,
                     target_time: float = 0.25, max_steps: int = 2000, device=None) -> BenchResult:
    """atom-steps/s for each requested size (rounded to a cube) (mdkk/driver/bench.py:105-148)."""
    if potential not in _POTENTIALS:
        raise RunError(f"unknown bench potential {potential!r}; choose from {_POTENTIALS}")
    if reps < 1:
        raise RunError("reps must be at least 1")
    sims, n_atoms, warms = [], [], []
    for n_request in sizes:
        sim = _make_sim(potential, int(n_request), device)
        sims.append(sim)
        n_atoms.append(len(sim._positions))
        warms.append(max(_time_steps(sim, 1), 1e-9))
    trial_time = max(target_time, max(warms))
    n_steps = [int(np.clip(round(trial_time / w), 1, max_steps)) for w in warms]
    best = [0.0] * len(sims)
    extra = 2
    gc.collect()
    with _no_gc():
        for rnd in range(reps + extra):
            for i, sim in enumerate(sims):
                expected = n_steps[i] * n_atoms[i] / max(best[i], 1e-9)
                if rnd >= reps and expected >= 0.5:
                    continue
                elapsed = _time_steps(sim, n_steps[i])
                best[i] = max(best[i], n_atoms[i] * n_steps[i] / elapsed)
    rows = list(zip(n_atoms, best))
    del sims
    gc.collect()
    result = BenchResult(potential, rows)
    if csv_path:
        result.write_csv(csv_path)
    return result
