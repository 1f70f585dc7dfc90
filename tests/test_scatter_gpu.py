"""ScatterAccumulator strategies on the device (mdkk/memspace.py:165-257) and
compute_pair's `strategy` on half lists (mdkk/pair_lj.py:114-179).

Mirrors the reference's tests/test_memspace.py:160-210 with the CUDA path
under test; Serial is additionally pinned bit-for-bit to sequential np.add.at
and Duplicate to the reference's per-copy staging + np.add.reduce.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import md

pytestmark = pytest.mark.gpu


def _contribs(rng, n_target, n_contrib, width=3):
    idx = rng.integers(0, n_target, n_contrib)
    vals = rng.normal(size=(n_contrib, width))
    return idx, vals


def test_serial_is_sequential_add_at_bit_for_bit(gpu):
    from paper_2508_13523_b200.memspace import ScatterAccumulator, Serial
    rng = np.random.default_rng(3)
    idx, vals = _contribs(rng, 16, 4000)
    acc = ScatterAccumulator((16, 3), Serial())
    acc.add(idx[:1500], vals[:1500])
    acc.add(idx[1500:], vals[1500:])
    ref = np.zeros((16, 3))
    np.add.at(ref, idx, vals)
    assert np.array_equal(acc.finalize(), ref)


def test_duplicate_matches_reference_staging_bit_for_bit(gpu):
    from paper_2508_13523_b200.memspace import Duplicate, ScatterAccumulator, scatter_accumulate
    rng = np.random.default_rng(4)
    idx, vals = _contribs(rng, 32, 1000)
    got = scatter_accumulate(ScatterAccumulator((32, 3), Duplicate(copies=4)), list(zip(idx, vals)))
    staging = np.zeros((4, 32, 3))
    bounds = np.linspace(0, 1000, 5).astype(int)
    for w in range(4):
        np.add.at(staging[w], idx[bounds[w]:bounds[w + 1]], vals[bounds[w]:bounds[w + 1]])
    assert np.array_equal(got, np.add.reduce(staging, axis=0))


@pytest.mark.parametrize("name", ["duplicate", "atomic"])
def test_strategies_match_serial_within_reassociation(gpu, name):
    from paper_2508_13523_b200.memspace import Atomic, Duplicate, ScatterAccumulator, Serial, scatter_accumulate
    rng = np.random.default_rng(5)
    idx, vals = _contribs(rng, 32, 1000)
    contribs = list(zip(idx, vals))
    strategy = Duplicate(copies=4) if name == "duplicate" else Atomic()
    serial = scatter_accumulate(ScatterAccumulator((32, 3), Serial()), contribs)
    other = scatter_accumulate(ScatterAccumulator((32, 3), strategy), contribs)
    assert np.allclose(other, serial, rtol=1e-12, atol=1e-12)


def test_duplicate_worker_buffers_are_independent(gpu):
    from paper_2508_13523_b200.memspace import Duplicate, ScatterAccumulator
    acc = ScatterAccumulator((4,), Duplicate(copies=3))
    acc.add([0], [1.0], worker=0)
    acc.add([0], [10.0], worker=1)
    acc.add([0], [100.0], worker=2)
    assert acc.finalize()[0] == 111.0


def test_finalize_is_a_barrier_and_indices_are_checked(gpu):
    from paper_2508_13523_b200.memspace import MemspaceError, ScatterAccumulator, Serial
    acc = ScatterAccumulator((4,), Serial())
    acc.add([1], [2.0])
    acc.finalize()
    with pytest.raises(MemspaceError):
        acc.add([1], [2.0])
    with pytest.raises(MemspaceError):
        acc.finalize()
    acc = ScatterAccumulator((4,), Serial())
    with pytest.raises(IndexError):
        acc.add([4], [1.0])
    with pytest.raises(IndexError):
        acc.add([-1], [1.0])


@pytest.mark.parametrize("newton", [True, False])
@pytest.mark.parametrize("n_ranks", [1, 2])
def test_compute_pair_strategies_on_half_lists(gpu, newton, n_ranks):
    """Every strategy agrees with the O(N^2) oracle at 1e-12; Serial is run-to-run
    bit-identical (no atomics anywhere on its path)."""
    from paper_2508_13523_b200 import Box, LJCut, PairParams, RankedSystem, build_all, compute_pair
    from paper_2508_13523_b200.memspace import Atomic, Duplicate, Serial
    pos, lengths = md.random_config(900, 0.75, seed=77)
    e_ref, f_ref, w_ref = md.lj_reference_n2(pos, lengths, 1.0, 1.0, 2.0)
    system = RankedSystem.distribute(Box(lengths), n_ranks, pos, np.zeros_like(pos))
    lists = build_all(system, 2.0, 0.3, style="half", newton=newton)
    forces = {}
    for name, strat in (("serial", Serial()), ("serial2", Serial()), ("duplicate", Duplicate(copies=5)),
                        ("atomic", Atomic()), ("default", None)):
        res = compute_pair(LJCut(PairParams(1.0, 1.0, 2.0)), system, lists, strategy=strat)
        assert res.energy == pytest.approx(e_ref, rel=1e-12), name
        assert np.allclose(res.forces, f_ref, rtol=1e-12, atol=1e-10), name
        assert np.allclose(res.virial, w_ref, rtol=1e-12, atol=1e-10), name
        forces[name] = res.forces
    assert np.array_equal(forces["serial"], forces["serial2"])


def test_unknown_strategy_is_rejected(gpu):
    from paper_2508_13523_b200 import Box, LJCut, PairError, PairParams, RankedSystem, build_all, compute_pair
    pos, lengths = md.random_config(100, 0.7, seed=1)
    system = RankedSystem.distribute(Box(lengths), 1, pos, np.zeros_like(pos))
    lists = build_all(system, 2.0, 0.3, style="half", newton=True)
    with pytest.raises(PairError):
        compute_pair(LJCut(PairParams(1.0, 1.0, 2.0)), system, lists, strategy="atomic")


def test_pair_energy_force_closed_form(gpu):
    """LJCut.pair_energy_force (mdkk/pair_lj.py:81-91) on host arrays and device tensors."""
    import torch
    from paper_2508_13523_b200 import LJCut, PairError, PairParams
    k = LJCut(PairParams(1.0, 1.0, 2.5))
    r2 = np.array([4.0, 2 ** (1 / 3), 1.5])
    e, fp = k.pair_energy_force(r2)
    assert e[0] == pytest.approx(4 * (2.0 ** -12 - 2.0 ** -6), rel=1e-15)
    assert e[1] == pytest.approx(-1.0, rel=1e-14) and abs(fp[1]) < 1e-13
    ed, fd = k.pair_energy_force(torch.tensor(r2, device="cuda"))
    assert np.array_equal(ed.cpu().numpy(), e) and np.array_equal(fd.cpu().numpy(), fp)
    with pytest.raises(PairError):
        k.pair_energy_force(np.array([0.0, 1.0]))
