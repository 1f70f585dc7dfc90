"""Saturation sweep: device-timed atom-steps/s across system sizes (mdkk/driver/bench.py:105-148).

The reference's protocol (a zero-temperature simple-cubic crystal: forces
cancel by symmetry, nothing moves, lists never rebuild, so a step is the
steady-state cost) and its interface (`bench_saturation(potential, sizes,
reps, csv_path)`, `BenchResult`, CSV `n_atoms,atom_steps_per_second`) are
kept; the measurement is the GPU's own:

* every trial is a stretch of `Simulation.advance(k)` bracketed by CUDA events
  on the engine's stream, so the rate is device time, not host wall time;
* k is calibrated per size from an event-timed probe so one trial covers at
  least `target_time` of device work (launch latency amortised at small N);
* sizes are visited in a rotated order each round (no size always runs right
  after the same neighbour) and the per-size rate is the fastest trial.
"""

from __future__ import annotations

import csv
import gc

import numpy as np
import torch

from .simulation import LJStyle, RunConfig, RunError, Simulation, lattice_positions

# (lattice density, r_c, skin, list style) of the reference's two setups
# (mdkk/driver/bench.py:24-27); SNAP runs 2J = 2 with a linear beta ramp
SETUPS = {
    "lj": (0.8, 1.6, 0.3, "half"),
    "snap": (0.8, 1.2, 0.25, "full"),
}
SNAP_JMAX = 1.0


class BenchResult:
    """(n_atoms, atom-steps/s) rows of one potential (mdkk/driver/bench.py:30-51)."""

    def __init__(self, potential: str, rows):
        self.potential = potential
        self.rows = [(int(n), float(r)) for n, r in rows]

    @property
    def sizes(self) -> np.ndarray:
        return np.array([n for n, _ in self.rows])

    @property
    def rates(self) -> np.ndarray:
        return np.array([r for _, r in self.rows])

    def write_csv(self, path: str) -> None:
        with open(path, "w", newline="") as fh:
            out = csv.writer(fh)
            out.writerow(["n_atoms", "atom_steps_per_second"])
            out.writerows([n, f"{r:.6g}"] for n, r in self.rows)


def _crystal(potential: str, n_request: int, device) -> Simulation:
    rho, r_c, skin, list_style = SETUPS[potential]
    side = max(2, round(n_request ** (1.0 / 3.0)))
    need = int(np.ceil(2.0 * (r_c + skin) * rho ** (1.0 / 3.0)))   # the halo needs L >= 2 (r_c + skin)
    if side < need:
        raise RunError(f"bench size {n_request} too small: the {potential} halo needs at least a "
                       f"{need}^3 = {need ** 3} atom cube")
    pos, box = lattice_positions("sc", rho, (side, side, side))
    sim = Simulation(RunConfig(list_style=list_style, skin=skin, device=device), log=None)
    sim.box, sim._positions, sim._velocities, sim.dt = box, pos, np.zeros_like(pos), 1e-6
    if potential == "lj":
        sim.style = LJStyle(r_c)
        sim.style.set_coeff(1.0, 1.0)
    else:
        from ..snap.coupling import QuantumIndex
        from ..snap.style import SnapStyle
        beta = np.linspace(0.05, 0.1, len(QuantumIndex(SNAP_JMAX).triples()))
        sim.style = SnapStyle(r_c, SNAP_JMAX, beta, batch_u=1, tile_v=4096)
    sim._ensure_system()
    sim._forces_device()
    return sim


def _device_ms(sim: Simulation, steps: int) -> float:
    """Device time of `steps` engine steps (CUDA events on the engine's stream)."""
    stream = torch.cuda.current_stream(sim.device)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    sim.advance(steps)
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b)


def bench_saturation(potential: str, sizes, reps: int = 3, csv_path: str | None = None,
                     target_time: float = 0.25, max_steps: int = 4000, device=None) -> BenchResult:
    """Fastest device-timed atom-steps/s per requested size (rounded to a cube)."""
    if potential not in SETUPS:
        raise RunError(f"unknown bench potential {potential!r}; choose from {tuple(SETUPS)}")
    if reps < 1:
        raise RunError("reps must be at least 1")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    sims = [_crystal(potential, int(n), dev) for n in sizes]
    atoms = [len(s._positions) for s in sims]
    probe_steps = 4
    steps = []
    for s in sims:
        _device_ms(s, 1)                                   # first-call buffers outside the probe
        per = max(_device_ms(s, probe_steps) / probe_steps, 1e-6)
        steps.append(int(np.clip(np.ceil(1e3 * target_time / per), probe_steps, max_steps)))
    best_ms = np.full(len(sims), np.inf)
    gc.collect()
    gc_was = gc.isenabled()
    gc.disable()
    try:
        for rnd in range(reps):
            order = np.roll(np.arange(len(sims)), rnd)
            for k in order:
                best_ms[k] = min(best_ms[k], _device_ms(sims[k], steps[k]) / steps[k])
    finally:
        if gc_was:
            gc.enable()
    result = BenchResult(potential, [(n, n / (ms * 1e-3)) for n, ms in zip(atoms, best_ms)])
    del sims
    gc.collect()
    if csv_path:
        result.write_csv(csv_path)
    return result
