"""SNAP edge cases against the CPU oracle (oracle/snap.py, pinned to the reference's
goldens in tests/test_oracle.py).

- Ranks that own no atoms.
- A partner exactly at r = rc: it is outside the strict r < rc map of the reference
  (mdkk/snap/compute.py neighbour map), and f_c(rc) = 0 anyway.
- An isolated atom with no partners: U is the j = 0 identity only.
- Atom counts that are not a multiple of the kernels' per-CTA batch.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import md, snap as osnap

pytestmark = pytest.mark.gpu


def _gpu(pos, lengths, jmax, beta, rc, skin, n_ranks):
    from paper_2508_13523_b200 import Box, RankedSystem, build_all
    from paper_2508_13523_b200.snap import (SnapState, build_neighbor_map, compute_fused_deidrj, compute_ui,
                                            compute_yi, energy_from_y, make_coupling_tables)
    system = RankedSystem.distribute(Box(lengths), n_ranks, pos, np.zeros_like(pos))
    lists = build_all(system, rc, skin, style="full", newton=False)
    tables = make_coupling_tables(jmax)
    e = 0.0
    for store, nl in zip(system.stores, lists):
        nmap = build_neighbor_map(store, nl, rc)
        state = SnapState(tables, store.n_local, beta)
        compute_ui(nmap, state)
        compute_yi(state)
        e += energy_from_y(state)
        f = compute_fused_deidrj(nmap, state, store.n_total)
        fr = store.force.read("a")
        fr[: store.n_total] = f
        store.force.mark_modified("a")
    system.reverse_comm()
    return e, system.gather_forces(), system


def _oracle(pos, lengths, jmax, beta, rc, skin):
    sys_ = md.Ranked(lengths, 1, pos, np.zeros_like(pos))
    lists = md.build_all(sys_, rc, skin, "full", False)
    e, _ = osnap.snap_compute(sys_, lists, osnap.SnapOracle(2 * jmax, beta, rc))
    return e, sys_.gather_forces()


def _beta(jmax, seed=3):
    return np.random.default_rng(seed).uniform(-0.5, 0.5, len(osnap.triples(2 * jmax)))


def _same(gpu_out, ref):
    (e, f, _), (e_ref, f_ref) = gpu_out, ref
    assert e == pytest.approx(e_ref, rel=1e-12)
    assert np.abs(f - f_ref).max() <= 1e-10 * max(1.0, np.abs(f_ref).max())


@pytest.mark.parametrize("n_ranks", [2, 8])
def test_ranks_without_owned_atoms(gpu, n_ranks):
    g = np.arange(4) * 1.05 + 0.5
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    pos = pos + np.random.default_rng(n_ranks).uniform(-0.05, 0.05, pos.shape)
    lengths = np.array([12.0] * 3)
    out = _gpu(pos, lengths, 2, _beta(2), 1.9, 0.2, n_ranks)
    assert [s.n_local for s in out[2].stores].count(0) >= 1
    _same(out, _oracle(pos, lengths, 2, _beta(2), 1.9, 0.2))


def test_partner_exactly_at_cutoff_and_isolated_atom(gpu):
    lengths = np.array([12.0] * 3)
    pos = np.array([[2.0, 2.0, 2.0], [3.5, 2.0, 2.0],      # r = 1.5 = rc exactly
                    [2.0, 3.25, 2.0],                      # r = 1.25 from atom 0
                    [8.0, 8.0, 8.0]])                      # alone
    beta = _beta(2, seed=9)
    out = _gpu(pos, lengths, 2, beta, 1.5, 0.3, 1)
    _same(out, _oracle(pos, lengths, 2, beta, 1.5, 0.3))
    assert not np.any(out[1][3])


@pytest.mark.parametrize("n", [1, 7, 33, 129])
def test_odd_atom_counts(gpu, n):
    rng = np.random.default_rng(100 + n)
    lengths = np.array([9.0] * 3)
    pts = [rng.uniform(0, 9.0, 3)]
    while len(pts) < n:
        c = rng.uniform(0, 9.0, 3)
        d = np.array(pts) - c
        d -= lengths * np.round(d / lengths)
        if np.sqrt((d * d).sum(1)).min() > 0.9:
            pts.append(c)
    pos = np.array(pts)
    beta = _beta(1, seed=n)
    _same(_gpu(pos, lengths, 1, beta, 1.7, 0.3, 1), _oracle(pos, lengths, 1, beta, 1.7, 0.3))
