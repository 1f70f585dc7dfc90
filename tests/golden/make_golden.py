"""Generate golden vectors by running the UNMODIFIED reference `mdkk` engine.

Run in the build container (the reference is importable there, not on the GPU
box):  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture records the reference's own outputs on seeded inputs so the
oracle (oracle/) and the CUDA path can be pinned to them.  Outputs are small
compressed npz files committed next to this script.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_PKG = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

from mdkk.domain import Box, RankedSystem  # noqa: E402
from mdkk.neighbor import build_all  # noqa: E402
from mdkk.pair_lj import LJCut, PairParams, compute_pair  # noqa: E402
from mdkk.driver.simulation import RunConfig, run_script, lattice_positions  # noqa: E402
from mdkk.snap import (  # noqa: E402
    SnapState, build_neighbor_map, compute_bi, compute_fused_deidrj, compute_ui,
    compute_yi, make_coupling_tables, QuantumIndex,
)


def random_config(n, rho, seed, min_sep=0.85):
    """Same construction as the reference tests/conftest.py:16-31."""
    rng = np.random.default_rng(seed)
    cells = int(np.ceil(n ** (1.0 / 3.0)))
    a = (1.0 / rho) ** (1.0 / 3.0)
    lo = np.stack(np.meshgrid(*[np.arange(cells)] * 3, indexing="ij"), axis=-1).reshape(-1, 3)
    order = rng.permutation(len(lo))[:n]
    jitter = rng.uniform(-0.5, 0.5, (n, 3)) * (a - min_sep)
    return (lo[order] + 0.5) * a + jitter, Box((a * cells,) * 3)


def directed_set(system, lists):
    """Directed (gid_i, gid_j, shift_x, shift_y, shift_z) entries of every rank."""
    out = []
    for store, nl in zip(system.stores, lists):
        rows, cols, w, wj = nl.pairs()
        sh = np.rint(store.ghost_shift[cols] / system.box.lengths).astype(np.int64)
        out.append(np.column_stack([store.global_ids[rows], store.global_ids[cols], sh,
                                    np.full(len(rows), store.rank), (w * 2).astype(np.int64),
                                    wj.astype(np.int64)]))
    return np.concatenate(out) if out else np.zeros((0, 8), np.int64)


def lj_small():
    pos, box = random_config(120, 0.7, seed=2)
    out = {"pos": pos, "lengths": box.lengths, "rc": 2.5, "skin": 0.3}
    for style, newton in (("full", False), ("half", True), ("half", False)):
        for n_ranks in (1, 2, 4):
            system = RankedSystem.distribute(box, n_ranks, pos, np.zeros_like(pos))
            lists = build_all(system, 2.5, 0.3, style=style, newton=newton)
            res = compute_pair(LJCut(PairParams(1.0, 1.0, 2.5)), system, lists)
            tag = f"{style}_{int(newton)}_{n_ranks}"
            out[f"E_{tag}"] = res.energy
            out[f"F_{tag}"] = res.forces
            out[f"W_{tag}"] = res.virial
            out[f"pairs_{tag}"] = directed_set(system, lists)
            out[f"cap_{tag}"] = np.array([nl.max_neighbors for nl in lists])
            out[f"nghost_{tag}"] = np.array([s.n_ghost for s in system.stores])
    np.savez_compressed(os.path.join(HERE, "lj_small.npz"), **out)


def lj_32k():
    pos, box = lattice_positions("fcc", 0.8442, (20, 20, 20))
    pos = pos + np.random.default_rng(1).normal(0.0, 0.02, pos.shape)
    out = {"lengths": box.lengths}
    for style, newton in (("full", False), ("half", True)):
        system = RankedSystem.distribute(box, 1, pos, np.zeros_like(pos))
        lists = build_all(system, 2.5, 0.3, style=style, newton=newton)
        res = compute_pair(LJCut(PairParams(1.0, 1.0, 2.5)), system, lists)
        out[f"E_{style}"] = res.energy
        out[f"W_{style}"] = res.virial
        out[f"F_{style}_sub"] = res.forces[::37]
        out[f"Fmax_{style}"] = float(np.abs(res.forces).max())
        out[f"nentries_{style}"] = int(sum(len(nl.pairs()[0]) for nl in lists))
        out[f"cap_{style}"] = int(lists[0].max_neighbors)
        out[f"nghost_{style}"] = int(system.stores[0].n_ghost)
    np.savez_compressed(os.path.join(HERE, "lj_32k_jitter.npz"), **out)


def melt_runs():
    silent = lambda *_: None  # noqa: E731
    with open(os.path.join(REF_PKG, "scripts/melt.in")) as fh:
        text = fh.read()
    out = {}
    sim = run_script(text, RunConfig(), log=silent)
    out["melt500_rows"] = np.array(sim.results[-1].rows)
    # C1: 32k fcc rho 0.8442, rc 2.5, T 1.44 seed 87287, dt 0.005, 100 steps.
    c1 = ("units lj\nboundary p p p\nlattice fcc 0.8442\ncreate_box 20 20 20\ncreate_atoms\n"
          "mass 1.0\nvelocity 1.44 87287\npair_style lj/cut 2.5\npair_coeff 1.0 1.0\n"
          "timestep 0.005\nthermo 10\nrun 100\n")
    for style in ("half", "full"):
        t0 = time.time()
        sim = run_script(c1, RunConfig(list_style=style, newton=(style == "half")), log=silent)
        out[f"c1_{style}_rows"] = np.array(sim.results[-1].rows)
        out[f"c1_{style}_final_pos_sub"] = sim.results[-1].snapshots[100][::97]
        print(f"C1 {style}: {time.time() - t0:.1f}s")
    np.savez_compressed(os.path.join(HERE, "lj_runs.npz"), **out)


def _cluster(n, seed, spread=2.6, min_sep=0.8, box_l=12.0):
    rng = np.random.default_rng(seed)
    pts = [rng.uniform(-spread, spread, 3)]
    while len(pts) < n:
        cand = rng.uniform(-spread, spread, 3)
        if min(np.linalg.norm(cand - p) for p in pts) >= min_sep:
            pts.append(cand)
    return np.asarray(pts) + box_l / 2.0


def _snap_pipeline(pos, box, jmax, beta, r_c, skin):
    system = RankedSystem.distribute(box, 1, pos, np.zeros_like(pos))
    lists = build_all(system, cutoff=r_c, skin=skin, style="full", newton=False)
    tables = make_coupling_tables(jmax)
    store, nl = system.stores[0], lists[0]
    nmap = build_neighbor_map(store, nl, r_c)
    state = SnapState(tables, store.n_local, beta)
    compute_ui(nmap, state)
    energy = float(np.sum(compute_bi(state) @ state.beta))
    compute_yi(state)
    f = compute_fused_deidrj(nmap, state, store.n_total)
    fr = store.force.read("a")
    fr[: store.n_total] = f
    store.force.mark_modified("a")
    system.reverse_comm()
    gid = store.global_ids[: store.n_local]
    o = np.argsort(gid)
    return energy, system.gather_forces(), state.u_view()[o], state.y_view()[o], nmap.n_pairs


def snap_fixtures():
    out = {}
    for jmax, seed in ((1, 39), (2, 40), (4, 43)):
        n = 10 if jmax < 4 else 6
        pos = _cluster(n, seed)
        beta = np.random.default_rng(11).uniform(-0.5, 0.5, len(QuantumIndex(jmax).triples()))
        e, f, u, y, npairs = _snap_pipeline(pos, Box((12.0,) * 3), jmax, beta, 1.9, 0.2)
        tag = f"j{int(2 * jmax)}"
        out.update({f"{tag}_pos": pos, f"{tag}_beta": beta, f"{tag}_E": e, f"{tag}_F": f,
                    f"{tag}_U": u, f"{tag}_Y": y})
    # periodic 40-atom system, 2J=4, rc 1.4 (reference tests/test_snap.py:457-462 geometry)
    pos = np.random.default_rng(53).uniform(0, 6.0, (40, 3))
    beta = np.random.default_rng(11).uniform(-0.5, 0.5, len(QuantumIndex(2).triples()))
    e, f, u, y, _ = _snap_pipeline(pos, Box((6.0,) * 3), 2, beta, 1.4, 0.3)
    out.update({"per_pos": pos, "per_beta": beta, "per_E": e, "per_F": f, "per_U": u, "per_Y": y})
    # C4: 2,000 bcc tungsten-like, 2J=8, rc 4.73, skin 0.3, N(0,0.05) jitter seed 1
    a = 3.1803
    grid = np.stack(np.meshgrid(*[np.arange(10)] * 3, indexing="ij"), -1).reshape(-1, 3).astype(float)
    basis = np.array([[0, 0, 0], [0.5, 0.5, 0.5]])
    lat = (grid[:, None, :] + basis[None]).reshape(-1, 3) * a
    pos = lat + np.random.default_rng(1).normal(0.0, 0.05, lat.shape)
    beta = np.linspace(0.05, 0.1, 55)
    t0 = time.time()
    e, f, u, y, npairs = _snap_pipeline(pos, Box((10 * a,) * 3), 4, beta, 4.73, 0.3)
    print(f"SNAP 2k: {time.time() - t0:.1f}s, pairs {npairs}")
    out.update({"c4_E": e, "c4_F": f, "c4_U_sub": u[:16], "c4_Y_sub": y[:16], "c4_npairs": npairs})
    # perfect lattice energy (SURVEY §8(c) KAT 64610.777035472027)
    e0, f0, _, _, _ = _snap_pipeline(lat, Box((10 * a,) * 3), 4, beta, 4.73, 0.3)
    out.update({"c4_lattice_E": e0, "c4_lattice_Fmax": float(np.abs(f0).max())})
    np.savez_compressed(os.path.join(HERE, "snap.npz"), **out)


def qeq_fixtures():
    """Reference QEq on the reference tests' configuration (mdkk tests/test_qeq.py:17-40)."""
    from mdkk.qeq import QeqParams, QeqSystem, build_matrix, qeq_energy, solve_qeq
    out = {}
    for tag, n, rho, seed in (("a", 60, 0.5, 12), ("b", 200, 0.6, 5)):
        pos, box = random_config(n, rho, seed)
        L = box.lengths
        params = QeqParams(gamma=0.8, eta=20.0, chi=-0.35, cutoff=2.0)
        system = RankedSystem.distribute(box, 1, pos, np.zeros((n, 3)))
        lists = build_all(system, params.cutoff, 0.3, style="full", newton=False)
        H = build_matrix(system.stores[0], lists[0], params)
        # uniform chi (the reference's setup) gives q = 0; a seeded spread makes the charges non-trivial
        chi = params.chi + 0.1 * np.random.default_rng(seed + 1).normal(size=n)
        qs = QeqSystem(H, chi, tol=1e-10)
        out[f"{tag}_chi"] = chi
        q = solve_qeq(qs)
        gathered = system.gather()[0]
        out[f"{tag}_pos"] = gathered
        out[f"{tag}_L"] = np.asarray(L, dtype=np.float64)
        out[f"{tag}_H"] = H.to_dense()
        out[f"{tag}_q"] = q
        out[f"{tag}_E"] = qeq_energy(qs)
        out[f"{tag}_iters"] = np.array(qs.iterations)
    np.savez_compressed(os.path.join(HERE, "qeq.npz"), **out)


def canonical_keys(pairs, n_atoms):
    """Directed entries -> sorted int64 keys ((gid_i·n + gid_j)·27 + shift code).

    `pairs` is `directed_set`'s (gid_i, gid_j, sx, sy, sz, rank, 2w, wj) array.
    The test side (tests/test_parity_scale_gpu.py) encodes its own lists the
    same way, so a SHA-256 of the sorted key bytes pins the exact directed set.
    """
    code = (pairs[:, 2] + 1) * 9 + (pairs[:, 3] + 1) * 3 + (pairs[:, 4] + 1)
    keys = (pairs[:, 0] * n_atoms + pairs[:, 1]) * 27 + code
    keys.sort()
    return keys


def _set_digest(system, lists, n_atoms):
    import hashlib
    pairs = directed_set(system, lists)
    keys = canonical_keys(pairs, n_atoms)
    counts = np.zeros(n_atoms, np.int64)
    np.add.at(counts, pairs[:, 0], 1)
    return (hashlib.sha256(keys.astype("<i8").tobytes()).hexdigest(), len(keys),
            counts.astype(np.uint8))


def lj_sets(cells, tag, n_ranks_list=(1,), sub=997, counts_every=1):
    """Exact directed neighbour sets at the benchmarked LJ configs (C1 32k / C2 2M).

    fcc rho* 0.8442 + N(0, 0.02) jitter from default_rng(1), rc 2.5, skin 0.3;
    full/newton-off and half/newton-on lists; the set's SHA-256 and per-gid row
    counts, plus the step-0 E, W, max|F|, sum F and a 1/`sub` force subsample.
    """
    import hashlib
    pos, box = lattice_positions("fcc", 0.8442, cells)
    pos = pos + np.random.default_rng(1).normal(0.0, 0.02, pos.shape)
    n = len(pos)
    out = {"lengths": box.lengths, "n": n}
    for style, newton in (("full", False), ("half", True)):
        for n_ranks in n_ranks_list:
            t0 = time.time()
            system = RankedSystem.distribute(box, n_ranks, pos, np.zeros_like(pos))
            lists = build_all(system, 2.5, 0.3, style=style, newton=newton)
            t1 = time.time()
            digest, n_entries, counts = _set_digest(system, lists, n)
            res = compute_pair(LJCut(PairParams(1.0, 1.0, 2.5)), system, lists)
            k = f"{style}_{n_ranks}"
            out[f"sha_{k}"] = digest
            out[f"nentries_{k}"] = n_entries
            out[f"counts_{k}"] = counts[::counts_every]
            out[f"counts_sha_{k}"] = hashlib.sha256(counts.tobytes()).hexdigest()
            out[f"cap_{k}"] = np.array([nl.max_neighbors for nl in lists])
            out[f"nghost_{k}"] = np.array([s.n_ghost for s in system.stores])
            out[f"E_{k}"] = res.energy
            out[f"W_{k}"] = res.virial
            out[f"Fmax_{k}"] = float(np.abs(res.forces).max())
            out[f"Fsum_{k}"] = res.forces.sum(axis=0)
            out[f"F_sub_{k}"] = res.forces[::sub]
            print(f"{tag} {k}: build {t1 - t0:.1f}s total {time.time() - t0:.1f}s "
                  f"entries {n_entries} E {res.energy!r}", flush=True)
            del system, lists, res
    np.savez_compressed(os.path.join(HERE, f"{tag}.npz"), **out)


def snap_c4_run():
    """C4: 2,000 bcc, 2J=8, rc 4.73, skin 0.3, beta linspace(0.05, 0.1, 55),
    m 1, T 0.01 seed 4928459, dt 0.001, 100 NVE steps through the reference's own
    Simulation (bcc sites built here in the reference's cell-major x basis order,
    mdkk/driver/simulation.py:156-178, because mdkk has no bcc lattice)."""
    from mdkk.driver.simulation import Simulation, SnapStyle, seeded_velocities
    a = 3.1803
    grid = np.stack(np.meshgrid(*[np.arange(10)] * 3, indexing="ij"), -1).reshape(-1, 3).astype(float)
    basis = np.array([[0, 0, 0], [0.5, 0.5, 0.5]])
    pos = (grid[:, None, :] + basis[None]).reshape(-1, 3) * a
    sim = Simulation(RunConfig(list_style="full", newton=False), log=lambda *_: None)
    sim.box = Box((10 * a,) * 3)
    sim._positions = pos
    sim._velocities = seeded_velocities(len(pos), 0.01, 1.0, 4928459)
    sim.style = SnapStyle(4.73, 4.0, np.linspace(0.05, 0.1, 55))
    sim.dt = 0.001
    sim.thermo_every = 10
    t0 = time.time()
    res = sim.run_nve(100)
    print(f"C4 run: {time.time() - t0:.1f}s", flush=True)
    out = {"rows": np.array(res.rows), "final_pos_sub": res.snapshots[100][::7],
           "pos10_sub": res.snapshots[10][::7]}
    np.savez_compressed(os.path.join(HERE, "snap_run.npz"), **out)


def c1_drift():
    """C1 1000-step NVE thermo (every 100 steps) from the reference, full and half lists: the
    drift bound of the north star ("no worse than the reference's")."""
    silent = lambda *_: None  # noqa: E731
    c1 = ("units lj\nboundary p p p\nlattice fcc 0.8442\ncreate_box 20 20 20\ncreate_atoms\n"
          "mass 1.0\nvelocity 1.44 87287\npair_style lj/cut 2.5\npair_coeff 1.0 1.0\n"
          "timestep 0.005\nthermo 100\nrun 1000\n")
    out = {}
    for style in ("full", "half"):
        t0 = time.time()
        sim = run_script(c1, RunConfig(list_style=style, newton=(style == "half")), log=silent)
        out[f"c1_{style}_rows1000"] = np.array(sim.results[-1].rows)
        print(f"C1 1000 {style}: {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "lj_drift.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["lj_small", "lj_32k", "snap", "runs", "qeq"]
    if "c1_drift" in which:
        c1_drift()
    if "lj_sets_c1" in which:
        lj_sets((20, 20, 20), "lj_c1_sets", n_ranks_list=(1, 8), sub=37)
    if "lj_sets_c2" in which:
        lj_sets((80, 80, 80), "lj_c2_sets", sub=997, counts_every=97)
    if "snap_run" in which:
        snap_c4_run()
    if "lj_small" in which:
        lj_small()
    if "lj_32k" in which:
        lj_32k()
    if "snap" in which:
        snap_fixtures()
    if "runs" in which:
        melt_runs()
    if "qeq" in which:
        qeq_fixtures()
