"""The reference's own unit tests for the hot path, run against the GPU drop-in.

Mirrors mdkk tests/test_pair_lj.py, test_domain.py and test_neighbor.py case by
case (same inputs, same assertions, same tolerances); the checker is the
O(N^2) oracle (oracle/md.py, the reference's conftest lj_reference) or a
brute-force pair set.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import md

pytestmark = pytest.mark.gpu


def _box(lengths):
    from paper_2508_13523_b200 import Box
    return Box(lengths)


def _compute(pos, lengths, r_c=2.5, n_ranks=1, style="half", newton=True, mode="atom", strategy=None,
             n_workers=None, skin=0.3):
    from paper_2508_13523_b200 import LJCut, PairParams, RankedSystem, build_all, compute_pair
    system = RankedSystem.distribute(_box(lengths), n_ranks, pos, np.zeros_like(pos))
    lists = build_all(system, r_c, skin, style=style, newton=newton)
    return compute_pair(LJCut(PairParams(1.0, 1.0, r_c)), system, lists, mode=mode, strategy=strategy,
                        n_workers=n_workers)


# ------------------------------------------------------------- test_pair_lj
def test_energy_forces_virial_match_reference(gpu):
    pos, L = md.random_config(120, 0.7, seed=2)
    e_ref, f_ref, w_ref = md.lj_reference_n2(pos, L, 1.0, 1.0, 2.5)
    res = _compute(pos, L)
    assert res.energy == pytest.approx(e_ref, rel=1e-12)
    assert np.allclose(res.forces, f_ref, rtol=1e-12, atol=1e-10)
    assert np.allclose(res.virial, w_ref, rtol=1e-12, atol=1e-9)


def test_pressure_matches_virial_trace(gpu):
    pos, L = md.random_config(90, 0.5, seed=8)
    res = _compute(pos, L)
    vol = float(np.prod(L))
    assert res.pressure(vol) == pytest.approx(res.virial[:3].sum() / (3 * vol), rel=1e-15)


def test_forces_sum_to_zero(gpu):
    pos, L = md.random_config(150, 0.7, seed=13)
    for style, newton in (("half", True), ("full", False)):
        assert np.all(np.abs(_compute(pos, L, style=style, newton=newton).forces.sum(axis=0)) < 1e-10)


def test_two_body_closed_form_through_the_kernel(gpu):
    """U(2 sigma) = 4 (2^-12 - 2^-6); at r_min the energy is -eps and the force vanishes; just inside
    the cutoff the pair energy is the unshifted value (mdkk tests/test_pair_lj.py:28-50)."""
    for r, e_want in ((2.0, 4.0 * (2.0 ** -12 - 2.0 ** -6)), (2.0 ** (1.0 / 6.0), -1.0),
                      (2.5 - 1e-9, 4.0 * ((2.5 - 1e-9) ** -12 - (2.5 - 1e-9) ** -6))):
        pos = np.array([[5.0, 5.0, 5.0], [5.0 + r, 5.0, 5.0]])
        for style, newton in (("half", True), ("full", False)):
            res = _compute(pos, np.array([12.0, 12.0, 12.0]), style=style, newton=newton)
            assert res.energy == pytest.approx(e_want, rel=1e-12)
    pos = np.array([[5.0, 5.0, 5.0], [5.0 + 2.0 ** (1.0 / 6.0), 5.0, 5.0]])
    assert np.abs(_compute(pos, np.array([12.0] * 3)).forces).max() < 1e-12
    pos = np.array([[5.0, 5.0, 5.0], [7.5 + 1e-9, 5.0, 5.0]])     # just outside: truncated to zero
    assert _compute(pos, np.array([12.0] * 3)).energy == 0.0


@pytest.mark.parametrize("strategy_name", ["serial", "duplicate", "atomic"])
def test_strategies_agree(gpu, strategy_name):
    from paper_2508_13523_b200.memspace import Atomic, Duplicate, Serial
    strategy = {"serial": Serial(), "duplicate": Duplicate(copies=3), "atomic": Atomic()}[strategy_name]
    pos, L = md.random_config(70, 0.7, seed=6)
    ref = _compute(pos, L)
    got = _compute(pos, L, strategy=strategy, n_workers=3, mode="neighbor")
    assert got.energy == pytest.approx(ref.energy, rel=1e-12)
    assert np.allclose(got.forces, ref.forces, rtol=1e-12, atol=1e-10)


def test_unknown_mode_rejected(gpu):
    from paper_2508_13523_b200 import PairError
    pos, L = md.random_config(125, 0.5, seed=3)
    with pytest.raises(PairError):
        _compute(pos, L, mode="warp")


# ------------------------------------------------------------- test_domain
def _system(n=60, n_ranks=4, halo=1.5, seed=3):
    from paper_2508_13523_b200 import RankedSystem
    pos, L = md.random_config(n, 0.5, seed=seed)
    vel = np.random.default_rng(seed).normal(size=pos.shape)
    system = RankedSystem.distribute(_box(L), n_ranks, pos, vel)
    system.exchange_ghosts(halo)
    return system, pos, vel, L


def test_distribute_partitions_all_atoms(gpu):
    from paper_2508_13523_b200.domain import wrap_positions
    system, pos, vel, L = _system()
    assert sum(s.n_local for s in system.stores) == len(pos)
    gp, gv, gids = system.gather()
    assert np.array_equal(gids, np.arange(len(pos)))
    assert np.allclose(gp, wrap_positions(pos, _box(L)), atol=1e-15)
    assert np.array_equal(gv, vel)


def test_ghosts_cover_halo_sphere(gpu):
    """Every pair within the halo is resolvable rank-locally (mdkk tests/test_domain.py:77-100)."""
    system, pos, _, L = _system(n=48, n_ranks=2, halo=1.2)
    brute = set()
    for i in range(len(pos)):
        d = pos[i + 1:] - pos[i]
        d -= L * np.round(d / L)
        for j in np.flatnonzero((d * d).sum(axis=1) < 1.2 * 1.2):
            brute.add((i, i + 1 + int(j)))
    seen = set()
    for store in system.stores:
        p, ids = store.positions(), store.global_ids
        for a in range(store.n_local):
            r2 = ((p - p[a]) ** 2).sum(axis=1)
            for b in np.flatnonzero((r2 > 0) & (r2 < 1.2 * 1.2)):
                seen.add(tuple(sorted((int(ids[a]), int(ids[b])))))
    assert brute <= seen


def test_halo_wider_than_half_box_rejected(gpu):
    from paper_2508_13523_b200 import DomainError
    system, _, _, L = _system(n_ranks=1)
    with pytest.raises(DomainError):
        system.exchange_ghosts(0.51 * float(L.min()))


def test_single_rank_still_builds_periodic_ghosts(gpu):
    system, *_ = _system(n_ranks=1, halo=1.0)
    assert system.stores[0].n_ghost > 0


def test_forward_comm_bit_exact_after_position_update(gpu):
    system, *_ = _system(n_ranks=4)
    rng = np.random.default_rng(0)
    for store in system.stores:
        p = store.pos.read("a")
        p[: store.n_local] += 0.01 * rng.normal(size=(store.n_local, 3))
        store.pos.mark_modified("a")
    system.forward_comm()
    for store in system.stores:
        pos = store.positions()
        for g in range(store.n_ghost):
            row = store.n_local + g
            owner = system.stores[store.owner_rank[row]]
            src = owner.positions()[store.owner_index[row]]
            assert np.array_equal(pos[row], src + store.ghost_shift[row])


def test_reverse_comm_folds_ghost_forces_to_owners(gpu):
    system, *_ = _system(n_ranks=4)
    rng = np.random.default_rng(1)
    expect = {}
    for store in system.stores:
        f = store.force.read("a")
        f[: store.n_total] = rng.normal(size=(store.n_total, 3))
        store.force.mark_modified("a")
    for store in system.stores:
        f = store.forces()
        for a in range(store.n_local):
            expect[int(store.global_ids[a])] = expect.get(int(store.global_ids[a]), 0) + f[a]
        for g in range(store.n_ghost):
            row = store.n_local + g
            gid = int(system.stores[store.owner_rank[row]].global_ids[store.owner_index[row]])
            expect[gid] = expect.get(gid, 0) + f[row]
    system.reverse_comm()
    for store in system.stores:
        f = store.forces()
        assert np.all(f[store.n_local:] == 0.0)
        for a in range(store.n_local):
            assert np.allclose(f[a], expect[int(store.global_ids[a])], rtol=1e-14, atol=1e-14)


def test_migrate_reassigns_moved_atoms(gpu):
    from paper_2508_13523_b200.domain import wrap_positions
    system, pos, vel, L = _system(n=60, n_ranks=4, halo=1.0)
    rng = np.random.default_rng(9)
    for store in system.stores:
        p = store.pos.read("a")
        p[: store.n_local] += rng.normal(scale=0.8, size=(store.n_local, 3))
        store.pos.mark_modified("a")
    moved = {int(g): system.stores[r].positions()[i].copy() for r in range(system.n_ranks)
             for i, g in enumerate(system.stores[r].global_ids[: system.stores[r].n_local])}
    system.migrate(1.0)
    gp, _, gids = system.gather()
    assert np.array_equal(gids, np.arange(60))
    for gid in range(60):
        assert np.allclose(gp[gid], wrap_positions(moved[gid][None], _box(L))[0], atol=1e-12)
    for store in system.stores:   # every atom sits in its owner's brick
        p = store.positions()[: store.n_local]
        assert np.all(system.rankset.rank_of(p) == store.rank)


def test_zero_forces_clears_all_rows(gpu):
    system, *_ = _system(n_ranks=2)
    for store in system.stores:
        f = store.force.read("a")
        f[: store.n_total] = 1.0
        store.force.mark_modified("a")
    system.zero_forces()
    for store in system.stores:
        assert np.all(store.forces() == 0.0)


# ----------------------------------------------------------- test_neighbor
def test_full_style_stores_each_pair_twice_and_half_once(gpu):
    from paper_2508_13523_b200 import RankedSystem, build_all
    pos, L = md.random_config(100, 0.6, seed=21)
    system = RankedSystem.distribute(_box(L), 1, pos, np.zeros_like(pos))
    (full,) = build_all(system, 2.0, 0.3, style="full", newton=False)
    rows, cols, w, wj = full.pairs()
    assert np.all(w == 0.5) and not wj.any()
    (half,) = build_all(system, 2.0, 0.3, style="half", newton=True)
    hr, hc, hw, hwj = half.pairs()
    assert np.all(hw == 1.0) and hwj.all()
    assert 2 * len(hr) == len(rows)


def test_canonical_order_invariant_under_input_permutation(gpu):
    """Per-atom rows in (gid, z, y, x) order regardless of input order (mdkk tests/test_neighbor.py:74-103)."""
    from paper_2508_13523_b200 import RankedSystem, build_all
    pos, L = md.random_config(90, 0.6, seed=23)

    def directed(p, gids):
        system = RankedSystem.distribute(_box(L), 1, p, np.zeros_like(p), global_ids=gids)
        (nl,) = build_all(system, 2.0, 0.3, style="full", newton=False)
        rows, cols, _, _ = nl.pairs()
        g = system.stores[0].global_ids
        out = {}
        for r, c in zip(rows, cols):
            out.setdefault(int(g[r]), []).append(int(g[c]))
        return out
    a = directed(pos, None)
    perm = np.random.default_rng(5).permutation(len(pos))
    b = directed(pos[perm], perm)
    assert a == b


def test_build_rejects_oversized_halo(gpu):
    from paper_2508_13523_b200 import NeighborError, RankedSystem, build
    pos, L = md.random_config(40, 0.6, seed=2)
    system = RankedSystem.distribute(_box(L), 1, pos, np.zeros_like(pos))
    with pytest.raises(NeighborError):
        build(system.stores[0], system.box, 0.5 * float(L.min()), 0.3)
