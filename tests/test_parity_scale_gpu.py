"""Parity at the benchmarked configurations (BASELINE.json configs[0..4]).

The headline numbers are measured on C2 (2,048,000 atoms), C3 (16.4M) and C5
(1M SNAP).  These tests pin the kernels there, not only on small systems:

* C1 32k and C2 2M: the exact directed neighbour set (SHA-256 of the sorted
  canonical keys, `tests/golden/make_golden.py:canonical_keys`), per-gid row
  counts, capacity, ghost count, step-0 E / W / max|F| / sum F and a force
  subsample against the UNMODIFIED reference (`lj_c1_sets.npz`,
  `lj_c2_sets.npz`), full/newton-off and half/newton-on lists, 1 and 8 ranks;
* C4: the reference's own 100-step SNAP NVE trajectory at 2J=8 (`snap_run.npz`);
* C3 / C5: 8 in-process ranks against 1 rank on the same GPU (the reference's
  rank-invariance tests, mdkk tests/test_driver.py:252-260,
  tests/test_pair_lj.py:115-121), E at 1e-12 and F at 1e-10·max|F|.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden
from oracle import md

pytestmark = pytest.mark.gpu


def _device_keys(system, lists, n_atoms):
    """Sorted int64 keys ((gid_i·n + gid_j)·27 + shift code) of every directed entry,
    formed on the device from the list tables (same encoding as make_golden.canonical_keys)."""
    import torch
    keys, counts = [], torch.zeros(n_atoms, dtype=torch.int64, device=system.device)
    for store, nl in zip(system.stores, lists):
        n = nl.n_local
        if n == 0:
            continue
        t = nl.expanded(nl.max_neighbors)[:, :n]
        code = torch.full((store.n_total,), 13, dtype=torch.int64, device=system.device)
        for ln in store._lanes_in:
            code[ln.start:ln.start + ln.count] = ln.code.long()
        valid = t >= 0
        rows = torch.arange(n, device=t.device).expand_as(t)[valid]
        cols = t[valid].long()
        gid = store.gid[: store.n_total].long()
        gi = gid[rows]
        keys.append((gi * n_atoms + gid[cols]) * 27 + code[cols])
        counts.index_add_(0, gi, torch.ones_like(gi))
        del t, valid, rows, cols
    k = torch.sort(torch.cat(keys))[0]
    return k.cpu().numpy(), counts.cpu().numpy()


def _check_sets_and_forces(g, tag, style, newton, n_ranks, sub, counts_every=1):
    import torch
    from paper_2508_13523_b200 import Box, LJCut, PairParams, RankedSystem, build_all, compute_pair
    n = int(g["n"])
    cells = round((n / 4) ** (1 / 3))
    pos, lengths = md.lattice("fcc", 0.8442, (cells,) * 3)
    pos = md.jittered(pos, 0.02, 1)
    system = RankedSystem.distribute(Box(lengths), n_ranks, pos, np.zeros_like(pos))
    lists = build_all(system, 2.5, 0.3, style=style, newton=newton)
    k = f"{style}_{n_ranks}"
    assert [nl.max_neighbors for nl in lists] == g[f"cap_{k}"].tolist()
    assert [s.n_ghost for s in system.stores] == g[f"nghost_{k}"].tolist()
    keys, counts = _device_keys(system, lists, n)
    assert len(keys) == int(g[f"nentries_{k}"])
    assert np.array_equal(counts[::counts_every], g[f"counts_{k}"].astype(np.int64))
    assert hashlib.sha256(counts.astype(np.uint8).tobytes()).hexdigest() == str(g[f"counts_sha_{k}"])
    assert hashlib.sha256(keys.astype("<i8").tobytes()).hexdigest() == str(g[f"sha_{k}"]), \
        f"{tag} {k}: directed neighbour set differs from the reference"
    del keys
    torch.cuda.empty_cache()
    res = compute_pair(LJCut(PairParams(1.0, 1.0, 2.5)), system, lists)
    assert res.energy == pytest.approx(float(g[f"E_{k}"]), rel=1e-12)
    assert np.allclose(res.virial, g[f"W_{k}"], rtol=1e-12)
    f = res.forces
    fmax = float(g[f"Fmax_{k}"])
    assert abs(float(np.abs(f).max()) - fmax) <= 1e-10 * fmax
    assert np.abs(f[::sub] - g[f"F_sub_{k}"]).max() <= 1e-10 * fmax
    assert np.abs(f.sum(axis=0) - g[f"Fsum_{k}"]).max() <= 1e-9 * fmax * np.sqrt(n)


@pytest.mark.parametrize("n_ranks", [1, 8])
@pytest.mark.parametrize("style,newton", [("full", False), ("half", True)])
def test_c1_exact_sets_and_step0(gpu, style, newton, n_ranks):
    """C1 32k jittered fcc: exact directed sets and step-0 E/W/F vs the reference."""
    _check_sets_and_forces(golden("lj_c1_sets.npz"), "C1", style, newton, n_ranks, sub=37)


@pytest.mark.parametrize("style,newton", [("full", False), ("half", True)])
def test_c2_2m_exact_sets_and_step0(gpu, style, newton):
    """C2 (the headline config) 2,048,000 atoms: exact directed sets and step-0 E/W/F."""
    _check_sets_and_forces(golden("lj_c2_sets.npz"), "C2", style, newton, 1, sub=997, counts_every=97)


def test_c4_snap_100_step_trajectory_matches_reference(gpu):
    """C4: the reference's 100-step NVE run (2,000 bcc, 2J=8, rc 4.73, dt 0.001, T 0.01),
    thermo every 10 steps, through the device engine."""
    from paper_2508_13523_b200 import Box
    from paper_2508_13523_b200.driver import RunConfig
    from paper_2508_13523_b200.driver.simulation import Simulation, seeded_velocities
    from paper_2508_13523_b200.snap.style import SnapStyle
    g = golden("snap_run.npz")
    pos, lengths = md.lattice("bcc", 3.1803, (10, 10, 10))
    sim = Simulation(RunConfig(list_style="full", newton=False), log=None)
    sim.box = Box(lengths)
    sim._positions = pos
    sim._velocities = seeded_velocities(len(pos), 0.01, 1.0, 4928459)
    sim.style = SnapStyle(4.73, 4.0, np.linspace(0.05, 0.1, 55))
    sim.dt = 0.001
    sim.thermo_every = 10
    rows = np.array(sim.run_nve(100).rows)
    ref = g["rows"]
    assert rows.shape == ref.shape
    assert rows[0, 1] == pytest.approx(ref[0, 1], rel=1e-12)
    assert np.allclose(rows[:, 1:], ref[:, 1:], rtol=1e-10, atol=1e-12)
    snap = sim.results[-1].snapshots[100][::7]
    assert np.abs(snap - g["final_pos_sub"]).max() < 1e-10


def _rank_invariance(pos, lengths, compute, n_ranks=8):
    from paper_2508_13523_b200 import Box, RankedSystem
    out = []
    for r in (1, n_ranks):
        system = RankedSystem.distribute(Box(lengths), r, pos, np.zeros_like(pos))
        out.append(compute(system))
        del system
    (e1, f1), (e8, f8) = out
    assert e8 == pytest.approx(e1, rel=1e-12)
    assert np.abs(f8 - f1).max() <= 1e-10 * np.abs(f1).max()
    return e1


@pytest.mark.parametrize("style,newton", [("full", False), ("half", True)])
def test_c3_16m_eight_ranks_equal_one(gpu, style, newton):
    """C3 16,384,000 atoms: 8 bricks (2,2,2) vs 1 brick, step-0 E and F."""
    from paper_2508_13523_b200 import LJCut, PairParams, build_all, compute_pair
    pos, lengths = md.lattice("fcc", 0.8442, (160, 160, 160))
    pos = md.jittered(pos, 0.02, 7)

    def lj(system):
        lists = build_all(system, 2.5, 0.3, style=style, newton=newton)
        res = compute_pair(LJCut(PairParams(1.0, 1.0, 2.5)), system, lists)
        assert sum(int(nl.counts_dev[: nl.n_local].sum()) for nl in lists) > 0
        return res.energy, res.forces
    _rank_invariance(pos, lengths, lj)


def test_c5_snap_1m_eight_ranks_equal_one(gpu):
    """C5 1,024,000 bcc atoms, 2J=8: 8 bricks vs 1 brick, E and F (ghost forces folded back)."""
    from paper_2508_13523_b200 import build_all
    from paper_2508_13523_b200.driver import RunConfig
    from paper_2508_13523_b200.snap.style import SnapStyle
    pos, lengths = md.lattice("bcc", 3.1803, (80, 80, 80))
    pos = md.jittered(pos, 0.05, 1)
    style = SnapStyle(4.73, 4.0, np.linspace(0.05, 0.1, 55))

    def snap(system):
        lists = build_all(system, 4.73, 0.3, style="full", newton=False)
        style._states = {}
        res = style.compute(system, lists, RunConfig(list_style="full", newton=False))
        return res.energy, res.forces
    e = _rank_invariance(pos, lengths, snap)
    # extensive: the 1M energy per atom sits next to the C4 2k KAT's (same lattice, jitter)
    assert e / len(pos) == pytest.approx(65509.51457722162 / 2000, rel=2e-3)
