"""Edge cases of the LJ hot path against the oracle.

- Ragged partitions: ranks that own no atoms but hold ghosts.
- Empty pair sets.
- A lone atom.
- Pairs exactly at the cutoff and at cutoff + skin. Both tests are strict:
  r^2 < rc^2 for the force (oracle/md.py lj_reference_n2, mdkk tests/conftest.py:38-64)
  and r^2 < bc^2 for list membership (mdkk/neighbor.py).
- A last cluster that fills only part of a warp.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import md

pytestmark = pytest.mark.gpu


def _forces(pos, lengths, rc, skin, n_ranks, style, newton, eps=1.0, sigma=1.0):
    from paper_2508_13523_b200 import Box, LJCut, PairParams, RankedSystem, build_all, compute_pair
    system = RankedSystem.distribute(Box(lengths), n_ranks, pos, np.zeros_like(pos))
    lists = build_all(system, rc, skin, style=style, newton=newton)
    return system, lists, compute_pair(LJCut(PairParams(eps, sigma, rc)), system, lists)


def _check(res, pos, lengths, rc, eps=1.0, sigma=1.0):
    e_ref, f_ref, w_ref = md.lj_reference_n2(pos, lengths, eps, sigma, rc)
    assert res.energy == pytest.approx(e_ref, rel=1e-12, abs=1e-300)
    scale = max(np.abs(f_ref).max(), 1e-300)
    assert np.abs(res.forces - f_ref).max() <= 1e-10 * scale
    assert np.allclose(res.virial, w_ref, rtol=1e-12, atol=1e-10)


@pytest.mark.parametrize("style,newton", [("full", False), ("half", True), ("half", False)])
@pytest.mark.parametrize("n_ranks", [2, 8])
def test_ranks_without_owned_atoms(gpu, style, newton, n_ranks):
    """All atoms in one corner brick; the other ranks own nothing but receive ghosts."""
    rng = np.random.default_rng(5 + n_ranks)
    g = np.arange(5) * 1.1 + 0.4
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    pos = pos + rng.uniform(-0.05, 0.05, pos.shape)
    lengths = np.array([12.0, 12.0, 12.0])
    system, _, res = _forces(pos, lengths, 2.5, 0.3, n_ranks, style, newton)
    owned = [s.n_local for s in system.stores]
    assert sum(owned) == len(pos) and owned.count(0) >= 1
    _check(res, pos, lengths, 2.5)


@pytest.mark.parametrize("style,newton", [("full", False), ("half", True)])
def test_empty_pair_set_and_lone_atom(gpu, style, newton):
    lengths = np.array([10.0, 10.0, 10.0])
    for pos in (np.array([[1.0, 1.0, 1.0], [6.0, 6.0, 6.0]]), np.array([[2.0, 3.0, 4.0]])):
        _, lists, res = _forces(pos, lengths, 2.5, 0.3, 1, style, newton)
        assert sum(len(nl.pairs()[0]) for nl in lists) == 0
        assert res.energy == 0.0 and not np.any(res.forces) and not np.any(res.virial)


@pytest.mark.parametrize("style,newton", [("full", False), ("half", True)])
def test_pairs_exactly_at_cutoff_and_list_radius(gpu, style, newton):
    """rc = 2.5, skin = 0.5: bc = 3.0 exactly. The partners sit at r = 2.5 (listed, no
    force), 3.0 (not listed), 2.999 (listed, no force) and 2.4 (the one interaction)."""
    lengths = np.array([10.0, 10.0, 10.0])
    pos = np.array([[1.0, 1.0, 1.0],
                    [3.5, 1.0, 1.0],      # r = 2.5 exactly (all values exact in binary)
                    [1.0, 4.0, 1.0],      # r = 3.0 = bc exactly
                    [1.0, 1.0, 3.999],    # just inside bc
                    [8.0, 8.0, 8.0],
                    [8.0, 8.0, 5.6]])     # r = 2.4 from the atom above
    _, lists, res = _forces(pos, lengths, 2.5, 0.5, 1, style, newton)
    rows, cols, _, _ = lists[0].pairs()
    n_pairs = len(rows) if style == "half" else len(rows) // 2
    # listed unordered pairs: (0,1) at 2.5, (0,3) at 2.999, (4,5) at 2.4, plus (1,3) at
    # |(-2.5, 0, 2.999)| = 3.905 > bc and (2,3) at |(0,-3,2.999)| > bc: three in all
    assert n_pairs == 3
    _check(res, pos, lengths, 2.5)
    e24 = 4.0 * ((1 / 2.4) ** 12 - (1 / 2.4) ** 6)
    assert res.energy == pytest.approx(e24, rel=1e-12)
    assert not np.any(res.forces[:4])


@pytest.mark.parametrize("n", [31, 33, 65, 97])
def test_partial_last_cluster(gpu, n):
    """Atom counts off multiples of the 32-atom cluster: the tail lanes of the last warp
    are masked in both the build and the force launch."""
    pos, lengths = md.random_config(n, 0.7, seed=300 + n)
    for style, newton in (("full", False), ("half", True)):
        _, _, res = _forces(pos, lengths, 1.8, 0.3, 1, style, newton)
        _check(res, pos, lengths, 1.8)


def test_host_position_write_after_sort_drops_stale_cell_order(gpu):
    """sort_local() leaves the owned rows cell-sorted and the halo selection scans
    only the boundary-layer rows of that order; a host-side position write through
    the DualArray protocol afterwards must invalidate it, or an atom moved into
    the halo layer would be missed as a ghost (mdkk/domain.py:246-293)."""
    from paper_2508_13523_b200 import Box, RankedSystem
    pos, lengths = md.lattice("fcc", 0.8442, (6, 6, 6))
    pos = md.jittered(pos, 0.02, 3)
    system = RankedSystem.distribute(Box(lengths), 1, pos, np.zeros_like(pos))
    system.sort_local(2.8)
    s = system.stores[0]
    a = s.pos.read("a")
    gids = s.gid[: s.n_local].cpu().numpy()
    k = int(np.argmin(np.abs(a[: s.n_local] - 0.5 * np.asarray(lengths)).sum(axis=1)))  # the most interior atom
    a[k] = (0.05, 0.5 * lengths[1], 0.5 * lengths[2])   # now within the halo of the x = 0 face
    s.pos.mark_modified("a")
    system.exchange_ghosts(2.8)
    by_gid = np.empty_like(pos)
    by_gid[gids] = a[: s.n_local]
    ref = md.Ranked(lengths, 1, by_gid, np.zeros_like(by_gid))
    ref.exchange_ghosts(2.8)
    r0 = ref.ranks[0]
    ours = np.sort(s.gid[s.n_local: s.n_total].cpu().numpy())
    assert s.n_ghost == len(r0.gid) - r0.n_local
    assert np.array_equal(ours, np.sort(r0.gid[r0.n_local:]))
    assert gids[k] in ours
