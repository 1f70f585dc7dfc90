"""The reference's SNAP unit tests for the hot path, run against the GPU drop-in.

Mirrors mdkk tests/test_snap.py case by case (same inputs, assertions and
tolerances): pair levels unitary (:247-258), level 1 the seed matrix
(:261-269), forces vs central finite differences of the energy (:436-454),
periodic force balance (:457-462), atom relabelling bit-exact per atom
(:502-520), map validation (:288-307), rotation / translation invariance
(:398-418), state validation (:523-531).  Energies take the descriptor route E = sum beta . B like the
reference's helper (mdkk tests/test_snap.py:93-115).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

R_C = 1.9
BOX_L = 12.0


def _cluster(n, seed, spread=2.6, min_sep=0.8):
    rng = np.random.default_rng(seed)
    pts = [rng.uniform(-spread, spread, 3)]
    while len(pts) < n:
        cand = rng.uniform(-spread, spread, 3)
        if min(np.linalg.norm(cand - p) for p in pts) >= min_sep:
            pts.append(cand)
    return np.asarray(pts) + BOX_L / 2.0


def _beta_for(jmax, seed=11):
    from paper_2508_13523_b200.snap import QuantumIndex
    rng = np.random.default_rng(seed)
    return rng.uniform(-0.5, 0.5, len(QuantumIndex(jmax).triples()))


def _pipeline(pos, box_l, jmax, beta, r_c=R_C, tables=None, global_ids=None, **knobs):
    from paper_2508_13523_b200 import Box, RankedSystem, build_all
    from paper_2508_13523_b200.snap import (SnapState, build_neighbor_map, compute_bi, compute_fused_deidrj,
                                            compute_ui, compute_yi, make_coupling_tables)
    pos = np.asarray(pos, dtype=np.float64)
    system = RankedSystem.distribute(Box((box_l,) * 3), 1, pos, np.zeros_like(pos), global_ids=global_ids)
    lists = build_all(system, r_c, 0.2, style="full", newton=False)
    tables = tables or make_coupling_tables(jmax)
    energy, states = 0.0, []
    for store, nlist in zip(system.stores, lists):
        nmap = build_neighbor_map(store, nlist, r_c)
        state = SnapState(tables, store.n_local, beta, **knobs)
        compute_ui(nmap, state)
        energy += float(np.sum(compute_bi(state) @ state.beta))
        compute_yi(state)
        f = compute_fused_deidrj(nmap, state, store.n_total)
        fr = store.force.read("a")
        fr[: store.n_total] = f
        store.force.mark_modified("a")
        states.append(state)
    system.reverse_comm()
    return energy, system.gather_forces(), states, system


def _pair_u(a_dir, r, jmax):
    """U of atom 0 in a two-atom system = f_c(r) u(a, b) (plus the j=0 slot): the levels
    of one pair, read back through compute_ui."""
    pos = np.array([[6.0, 6.0, 6.0], 6.0 + r * np.asarray(a_dir, dtype=np.float64)])
    _, _, states, system = _pipeline(pos, BOX_L, jmax, _beta_for(jmax), r_c=R_C)
    g = system.stores[0].global_ids[: system.stores[0].n_local]
    u = states[0].u_view()[np.argsort(g)][0]
    fc = 0.5 * (1.0 + np.cos(np.pi * r / R_C))
    return u / fc, states[0].index


def test_pair_levels_are_unitary(gpu):
    rng = np.random.default_rng(7)
    for _ in range(4):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        u, qi = _pair_u(d, rng.uniform(0.6, 1.7), 4)
        for tj in range(qi.twojmax + 1):
            blk = u[qi.block(tj)].reshape(tj + 1, tj + 1)
            assert np.allclose(blk @ np.conj(blk).T, np.eye(tj + 1), atol=1e-12)


def test_pair_level_one_is_the_seed_matrix(gpu):
    """Level 1 = [[conj a, -conj b], [b, a]] with a = (z0 - i z)/r0, b = (y - i x)/r0
    (mdkk/snap/compute.py:35-45, :125-147)."""
    d = np.array([0.3, -0.5, 0.8])
    d /= np.linalg.norm(d)
    r = 1.1
    u, qi = _pair_u(d, r, 1)
    x, y, z = d * r
    z0 = r / np.tan(0.99 * np.pi * r / R_C)
    r0 = np.sqrt(r * r + z0 * z0)
    a, b = (z0 - 1j * z) / r0, (y - 1j * x) / r0
    lvl1 = u[qi.block(1)].reshape(2, 2)
    assert np.allclose(lvl1, np.array([[np.conj(a), -np.conj(b)], [b, a]]), rtol=0, atol=1e-14)
    assert u[0] == pytest.approx(1.0, abs=1e-15)


def _fd_forces(pos, jmax, beta, h=1e-6, atoms=None):
    from paper_2508_13523_b200.snap import make_coupling_tables
    tables = make_coupling_tables(jmax)
    atoms = range(len(pos)) if atoms is None else atoms
    grad = np.zeros((len(pos), 3))
    for i in atoms:
        for d in range(3):
            pp = np.array(pos, dtype=np.float64)
            pp[i, d] += h
            ep = _pipeline(pp, BOX_L, jmax, beta, tables=tables)[0]
            pp[i, d] -= 2 * h
            em = _pipeline(pp, BOX_L, jmax, beta, tables=tables)[0]
            grad[i, d] = (ep - em) / (2 * h)
    return grad


@pytest.mark.parametrize("jmax", [1, 2])
def test_forces_match_finite_differences(gpu, jmax):
    pos = _cluster(8, 37 + jmax)
    beta = _beta_for(jmax, seed=41)
    _, forces, _, _ = _pipeline(pos, BOX_L, jmax, beta)
    grad = _fd_forces(pos, jmax, beta)
    scale = max(1.0, np.abs(forces).max())
    assert np.abs(forces + grad).max() / scale < 1e-6


def test_forces_match_finite_differences_high_order_spot(gpu):
    pos = _cluster(3, 43, spread=1.0)
    beta = _beta_for(4, seed=47)
    _, forces, _, _ = _pipeline(pos, BOX_L, 4, beta)
    grad = _fd_forces(pos, 4, beta, atoms=[0])
    scale = max(1.0, np.abs(forces).max())
    assert np.abs(forces[0] + grad[0]).max() / scale < 1e-6


def test_forces_sum_to_zero_periodic(gpu):
    pos = np.random.default_rng(53).uniform(0, 6.0, (40, 3))
    _, forces, _, _ = _pipeline(pos, 6.0, 2, _beta_for(2), r_c=1.4)
    assert np.abs(forces.sum(axis=0)).max() < 1e-10


def test_atom_relabeling_is_bit_exact_per_atom(gpu):
    """U and B per atom do not depend on labels (geometric accumulation order);
    E and F to 1e-12 (mdkk tests/test_snap.py:502-520)."""
    from paper_2508_13523_b200.snap import compute_bi, make_coupling_tables
    pos = _cluster(20, 71)
    beta = _beta_for(1, seed=73)
    tables = make_coupling_tables(1)
    e0, f0, states0, sys0 = _pipeline(pos, BOX_L, 1, beta, tables=tables, batch_u=1)
    perm = np.random.default_rng(79).permutation(len(pos))
    e1, f1, states1, sys1 = _pipeline(pos[perm], BOX_L, 1, beta, tables=tables, global_ids=perm, batch_u=1)
    g0 = np.argsort(sys0.stores[0].global_ids[: sys0.stores[0].n_local])
    g1 = np.argsort(sys1.stores[0].global_ids[: sys1.stores[0].n_local])
    assert np.array_equal(states0[0].u_view()[g0], states1[0].u_view()[g1])
    assert np.array_equal(compute_bi(states0[0])[g0], compute_bi(states1[0])[g1])
    assert e1 == pytest.approx(e0, rel=1e-12)
    assert np.allclose(f1, f0, rtol=1e-12, atol=1e-12)


def test_neighbor_map_requires_full_list_and_reach(gpu):
    """mdkk tests/test_snap.py:288-307."""
    from paper_2508_13523_b200 import Box, RankedSystem, build, build_all
    from paper_2508_13523_b200.snap import SnapError, build_neighbor_map
    pos = _cluster(6, 3)
    box = Box((BOX_L,) * 3)
    system = RankedSystem.distribute(box, 1, pos, np.zeros_like(pos))
    system.exchange_ghosts(R_C + 0.2)
    half = build(system.stores[0], box, R_C, 0.2, style="half", newton=True)
    with pytest.raises(SnapError):
        build_neighbor_map(system.stores[0], half, R_C)
    full = build(system.stores[0], box, R_C, 0.2, style="full", newton=False)
    with pytest.raises(SnapError):
        build_neighbor_map(system.stores[0], full, R_C + 1.0)
    z = RankedSystem.distribute(box, 1, np.full((2, 3), 5.0), np.zeros((2, 3)))
    (zl,) = build_all(z, R_C, 0.2, style="full", newton=False)
    with pytest.raises(SnapError):
        build_neighbor_map(z.stores[0], zl, R_C).n_pairs


def test_rotation_and_translation_invariance(gpu):
    """mdkk tests/test_snap.py:398-418: E and B invariant under rotations (1e-8) and
    translations (1e-12)."""
    from paper_2508_13523_b200.snap import compute_bi
    pos = _cluster(10, 29)
    beta = _beta_for(2)
    e0, _, states, sys0 = _pipeline(pos, BOX_L, 2, beta)
    g0 = np.argsort(sys0.stores[0].global_ids[: sys0.stores[0].n_local])
    b0 = compute_bi(states[0])[g0]
    rng = np.random.default_rng(31)
    center = pos.mean(axis=0)
    for _ in range(3):
        q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        if np.linalg.det(q) < 0:
            q[:, 0] = -q[:, 0]
        e1, _, states1, sys1 = _pipeline((pos - center) @ q.T + center, BOX_L, 2, beta)
        g1 = np.argsort(sys1.stores[0].global_ids[: sys1.stores[0].n_local])
        assert e1 == pytest.approx(e0, rel=1e-8)
        assert np.allclose(compute_bi(states1[0])[g1], b0, rtol=1e-8, atol=1e-10)
    e2 = _pipeline(pos + np.array([0.4, -0.9, 1.7]), BOX_L, 2, beta)[0]
    assert e2 == pytest.approx(e0, rel=1e-12)


def test_state_validation(gpu):
    """mdkk tests/test_snap.py:523-531."""
    from paper_2508_13523_b200.snap import SnapError, SnapState, compute_energy, make_coupling_tables
    tables = make_coupling_tables(1)
    with pytest.raises(SnapError):
        SnapState(tables, 4, np.zeros(3))
    with pytest.raises(SnapError):
        SnapState(tables, 4, np.zeros(5), layout="c")
    assert compute_energy(SnapState(tables, 0, np.zeros(5))) == 0.0
