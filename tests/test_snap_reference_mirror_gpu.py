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


# ------------------------------------------- exported helpers (mdkk/snap/__init__.py:3-21)
def test_pair_u_flat_unitary_seed_and_oracle(gpu):
    """pair_u_flat: unitary blocks for unit (a, b) (mdkk tests/test_snap.py:247-258), the seed
    matrix at level 1 (:261-269), and the four-term recursion for arbitrary (a, b)."""
    from oracle import snap as osnap
    from paper_2508_13523_b200.snap import QuantumIndex, pair_u_flat
    rng = np.random.default_rng(7)
    n = 6
    th = rng.uniform(0, np.pi, n)
    a = np.cos(th / 2) * np.exp(1j * rng.uniform(0, 2 * np.pi, n))
    b = np.sin(th / 2) * np.exp(1j * rng.uniform(0, 2 * np.pi, n))
    qi = QuantumIndex(4)
    flat = pair_u_flat(a, b, qi.twojmax)
    for tj in range(qi.twojmax + 1):
        blk = flat[:, qi.block(tj)].reshape(n, tj + 1, tj + 1)
        assert np.allclose(np.einsum("npq,nrq->npr", blk, np.conj(blk)), np.eye(tj + 1), atol=1e-12)
    a1, b1 = np.array([0.6 + 0.3j]), np.array([0.2 - 0.7j])
    lvl = pair_u_flat(a1, b1, 2)
    assert np.array_equal(lvl[0, 1:5].reshape(2, 2), np.array([[np.conj(a1[0]), -np.conj(b1[0])], [b1[0], a1[0]]]))
    assert lvl[0, 0] == 1.0 + 0.0j
    a2 = rng.normal(size=50) + 1j * rng.normal(size=50)
    b2 = rng.normal(size=50) + 1j * rng.normal(size=50)
    ref, _ = osnap.pair_levels(a2, b2, 8)
    got = pair_u_flat(a2, b2, 8)
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


def test_cutoff_switch_endpoints_and_slope(gpu):
    """mdkk tests/test_snap.py:272-284."""
    from paper_2508_13523_b200.snap import cutoff_switch
    fc, dfc = cutoff_switch(np.array([0.0, 1.5, 3.0]), 3.0)
    assert fc[0] == pytest.approx(1.0) and fc[1] == pytest.approx(0.5) and fc[2] == pytest.approx(0.0, abs=1e-16)
    assert dfc[0] == pytest.approx(0.0, abs=1e-16) and dfc[2] == pytest.approx(0.0, abs=1e-15)
    r, h = np.linspace(0.3, 2.7, 9), 1e-6
    fp, _ = cutoff_switch(r + h, 3.0)
    fm, _ = cutoff_switch(r - h, 3.0)
    _, d = cutoff_switch(r, 3.0)
    assert np.allclose((fp - fm) / (2 * h), d, atol=1e-8)


def test_zi_route_consistent_with_descriptors(gpu):
    """compute_zi: Re sum Z conj(U) per triple == B (mdkk tests/test_snap.py:348-361)."""
    from paper_2508_13523_b200.snap import compute_bi, compute_zi
    for layout in ("a", "b"):
        _, _, states, _ = _pipeline(_cluster(8, 17), BOX_L, 1, _beta_for(1), layout=layout)
        state = states[0]
        bi = compute_bi(state)
        u = state.u_view()
        qi = state.index
        for it, (tj, _, _) in enumerate(state.tables.triples):
            z = compute_zi(state, it)
            ublk = u[:, qi.block(tj)].reshape(len(u), tj + 1, tj + 1)
            via_z = np.einsum("npq,npq->n", z, np.conj(ublk)).real
            assert np.allclose(via_z, bi[:, it], rtol=1e-12, atol=1e-13)


def test_triple_terms_groupings(gpu):
    """TripleTerms (mdkk/snap/coupling.py:69-91): the grouping orders reproduce the terms."""
    from paper_2508_13523_b200.snap import TripleTerms, make_coupling_tables
    tables = make_coupling_tables(2)
    for tt in tables.terms:
        assert isinstance(tt, TripleTerms) and tt.n_terms == len(tt.coeff)
        for key in ("iz", "iu1", "iu2"):
            idx = getattr(tt, key)
            srt = idx[getattr(tt, f"order_{key}")]
            assert np.all(np.diff(srt) >= 0)
            assert np.array_equal(srt[getattr(tt, f"starts_{key}")], getattr(tt, f"unique_{key}"))
        assert tables.cg[(tt.tj1, tt.tj2, tt.tj)].shape == (tt.tj1 + 1, tt.tj2 + 1)


def test_neighbor_map_deriv_params_match_oracle(gpu):
    """NeighborMap.deriv_params (mdkk/snap/compute.py:98-102) vs the analytic gradients."""
    from oracle import snap as osnap
    from paper_2508_13523_b200 import Box, RankedSystem, build_all
    from paper_2508_13523_b200.snap import build_neighbor_map
    pos = _cluster(12, 5)
    system = RankedSystem.distribute(Box((BOX_L,) * 3), 1, pos, np.zeros_like(pos))
    (nl,) = build_all(system, R_C, 0.2, style="full", newton=False)
    nmap = build_neighbor_map(system.stores[0], nl, R_C)
    sel = slice(1, nmap.n_pairs - 1)
    da, db = nmap.deriv_params(sel)
    dr = nmap.dr[sel]
    r, a, b, _, _, z0, r0 = osnap.pair_params(dr, R_C)
    rda, rdb = osnap.pair_grads(dr, r, R_C, a, b, z0, r0)
    assert np.allclose(da, rda, rtol=1e-12, atol=1e-13) and np.allclose(db, rdb, rtol=1e-12, atol=1e-13)


def test_brute_force_pairs_matches_oracle(gpu):
    """brute_force_pairs (mdkk/neighbor.py:234-245; mdkk tests/test_neighbor.py:126-128)."""
    from oracle import md
    from paper_2508_13523_b200 import Box, brute_force_pairs
    pos, lengths = md.random_config(300, 0.8, seed=9)
    assert brute_force_pairs(pos, Box(lengths), 1.6) == md.pair_set_brute(pos, lengths, 1.6)
