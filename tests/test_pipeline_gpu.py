"""The engine's speculative launches give exactly the unpipelined results.

`Simulation.step_device` queues the force launch before the host has read the
step's skin test (mdkk_lj_force_gated skips it on the device when the step
rebuilds) and, on rebuild steps, before the build's capacity check
(`build(..., defer=True)` + `NeighborList.settle`).  Both must be invisible:
same trajectory bit for bit as the synchronous path, including a table
overflow that forces the regrow-and-relaunch branch.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MELT = """\
units lj
boundary p p p
lattice fcc 0.8442
create_box 8 8 8
create_atoms
mass 1.0
velocity 1.44 87287
pair_style lj/cut 2.5
pair_coeff 1.0 1.0
timestep 0.005
thermo 10
"""


def _sim(style="full"):
    from paper_2508_13523_b200.driver import RunConfig, Simulation
    sim = Simulation(RunConfig(list_style=style, newton=(style == "half")), log=None)
    sim.execute(MELT)
    return sim


@pytest.mark.parametrize("style", ["full", "half"])
def test_speculative_loop_matches_synchronous_loop(gpu, style):
    a, b = _sim(style), _sim(style)
    b.style.supports_gate = False          # the plain synchronous step
    ra, rb = a.run_nve(60), b.run_nve(60)
    assert ra.n_rebuilds == rb.n_rebuilds and ra.n_rebuilds >= 3
    if style == "full":   # owner writes: bit-identical
        assert ra.lines == rb.lines
        assert np.array_equal(a.system.gather_positions(), b.system.gather_positions())
    else:                 # FP64 atomics: summation order may differ
        for (s0, *r0), (s1, *r1) in zip(ra.rows, rb.rows):
            assert s0 == s1 and np.allclose(r0, r1, rtol=1e-12, atol=1e-12)


def test_gated_launch_is_a_no_op_when_the_step_rebuilds(gpu):
    import torch
    from paper_2508_13523_b200.pair_lj import lj_force_rank
    sim = _sim()
    sim.run_nve(0)
    s, nl = sim.system.stores[0], sim.lists[0]
    before = s.f.clone()
    ev = torch.zeros(7, dtype=torch.float64, device=s.device)
    flags = torch.zeros(1, dtype=torch.int32, device=s.device)
    d2 = torch.tensor([0.2 ** 2], dtype=torch.float64, device=s.device)   # sqrt = 0.2 > skin/2
    s.f.fill_(7.0)
    lj_force_rank(s, nl, sim.style.kernel.params, ev, flags, virial=False, gate=d2, gate_limit=0.15)
    assert bool((s.f == 7.0).all())
    d2.fill_(0.1 ** 2)                                                     # 0.1 <= skin/2: runs
    s.f.copy_(before)
    lj_force_rank(s, nl, sim.style.kernel.params, ev, flags, virial=False, gate=d2, gate_limit=0.15)
    assert torch.equal(s.f[: s.n_local], before[: s.n_local])


def test_deferred_build_overflow_regrows_and_relaunches(gpu):
    sim = _sim()
    sim.run_nve(5)
    sim._rebuild_lists()                       # reference: synchronous build
    e_ref = float(sim._forces_device().item())
    f_ref = sim.system.gather_forces()
    cap_ref = sim.lists[0].max_neighbors
    for hint, expect_ok in ((sim._cap_hint, True), (8, False)):
        sim._cap_hint = hint
        sim._rebuild_lists(defer=True)
        assert sim.lists[0].pending
        sim._forces_device()
        ok = sim._settle_lists()
        assert ok is expect_ok and not sim.lists[0].pending
        e = float(sim._forces_device().item()) if not ok else float(sim._e_dev.item())
        assert e == e_ref
        assert np.array_equal(sim.system.gather_forces(), f_ref)
        assert sim.lists[0].max_neighbors == cap_ref          # the reference growth sequence
        assert sim.lists[0].alloc_cap >= sim.lists[0].max_count


def test_fused_loop_overflow_relaunch_matches_synchronous(gpu):
    """The fused advance loop's regrow-and-relaunch branch (a rebuild whose table outgrows
    the capacity hint) keeps the trajectory bit-identical to the synchronous loop."""
    a, b = _sim("full"), _sim("full")
    b.style.supports_gate = False
    a.run_nve(0)
    b.run_nve(0)
    for sim in (a, b):
        sim._cap_hint = 8            # the next deferred rebuild overflows and regrows
    assert a._fusable() and not b._fusable()
    ra, rb = a.run_nve(40), b.run_nve(40)
    assert ra.n_rebuilds == rb.n_rebuilds and ra.n_rebuilds >= 2
    assert ra.lines == rb.lines
    assert np.array_equal(a.system.gather_positions(), b.system.gather_positions())
    assert np.array_equal(a.system.gather()[1], b.system.gather()[1])     # velocities


def test_overlapped_snapshots_match_synchronous_reads(gpu):
    """run_nve's thermo snapshots whose read-back overlaps the next stretch (pinned DMA on
    a copy stream, large enough for the staged path) equal positions read synchronously at
    the same steps."""
    from paper_2508_13523_b200.driver import RunConfig, Simulation
    big = MELT.replace("create_box 8 8 8", "create_box 23 23 23")
    a = Simulation(RunConfig(list_style="full", newton=False), log=None)
    b = Simulation(RunConfig(list_style="full", newton=False), log=None)
    a.execute(big)
    b.execute(big)
    assert a.snapshots and 4 * 23 ** 3 * 3 * 8 > (1 << 20)
    ra = a.run_nve(30)
    ref = {0: b.run_nve(0).snapshots[0]}       # the last snapshot of a run is read synchronously
    for k in range(1, 4):
        ref[10 * k] = b.run_nve(10).snapshots[10]
    assert sorted(ra.snapshots) == [0, 10, 20, 30]
    for step, snap in ra.snapshots.items():
        assert np.array_equal(snap, ref[step]), step
    # each snapshot owns its (pinned) block: later steps and later snapshots leave it alone
    snaps = list(ra.snapshots.values())
    assert not any(np.shares_memory(p, q) for i, p in enumerate(snaps) for q in snaps[i + 1:])
    keep = {k: v.copy() for k, v in ra.snapshots.items()}
    a.run_nve(20)
    assert all(np.array_equal(ra.snapshots[k], keep[k]) for k in keep)


@pytest.mark.parametrize("style", ["full", "half"])
@pytest.mark.parametrize("at", [3, 7])
def test_blow_up_aborts_at_the_first_bad_step(gpu, style, at):
    """Atom 0 moved exactly onto atom 1 right before step `at`'s force launch: that step's
    energy and forces are not finite, and the run stops there -- between thermo steps --
    with the reference's error (its kernel raises PairError on r = 0, mdkk/pair_lj.py:83-84,
    checked every step), not at the next thermo step."""
    from paper_2508_13523_b200 import PairError
    sim = _sim(style)
    sim.thermo_every = 100
    orig = sim.style.compute_device
    state = {"done": False}

    def poisoned(system, lists, config, *a, **kw):
        if sim._run_step == at and not state["done"]:
            s = system.stores[0]
            s.x[0, :3] = s.x[1, :3]
            state["done"] = True
        return orig(system, lists, config, *a, **kw)
    sim.style.compute_device = poisoned
    with pytest.raises(PairError, match="coincident"):
        sim.run_nve(40)
    assert sim._run_step == at + 1      # stopped at the next step's check, not at thermo 40


def test_nonfinite_energy_is_named_with_its_step(gpu):
    """Non-finite energy without coincidence (a NaN-poisoned epsilon from step 4 on): the run
    stops right after step 4 with "non-finite potential energy at step 4"."""
    from paper_2508_13523_b200.driver import RunError
    sim = _sim("full")
    sim.thermo_every = 100
    orig = sim.style.compute_device

    def poisoned(system, lists, config, *a, **kw):
        if sim._run_step == 4:
            sim.style.kernel.params.epsilon = float("nan")
        return orig(system, lists, config, *a, **kw)
    sim.style.compute_device = poisoned
    with pytest.raises(RunError, match="non-finite potential energy at step 4$"):
        sim.run_nve(40)


def test_single_rank_migrate_fast_path_matches_general_path(gpu):
    """RankedSystem.migrate's one-rank fast path (mdkk_rebuild1_select: wrap, cell sort,
    boundary rows, halo count in one call; the sort's gather also fills a skin-test
    reference) gives bit for bit the rows, ghosts and bins of the general path."""
    import torch
    from oracle import md
    from paper_2508_13523_b200 import Box, RankedSystem
    from paper_2508_13523_b200.domain import shell_grid_args

    pos, lengths = md.lattice("fcc", 0.8442, (10, 10, 10))
    pos = md.jittered(pos, 0.3, 7) + 0.37 * lengths   # drifted past the box: wrap has work
    vel = md.jittered(np.zeros_like(pos), 1.0, 8)
    out = {}
    for fast in (True, False):
        system = RankedSystem.distribute(Box(lengths), 1, pos, vel)
        system.sort_width = 2.8
        if not fast:
            system._migrate_single = lambda *a, **k: 0   # force the general path
        ref = torch.zeros_like(system.stores[0].x)
        wrote = system.migrate(2.8, zero_forces=False, ref_out=ref)
        s = system.stores[0]
        nt = s.n_total
        ncell = shell_grid_args(s.lo, s.hi, 2.8)[4]
        out[fast] = (s.x[:nt].cpu(), s.v[: s.n_local].cpu(), s.gid[:nt].cpu(), s.oidx[nt - s.n_ghost:nt].cpu(),
                     s._bins[2][: ncell + 1].cpu(), s.n_ghost, wrote, ref[: s.n_local].cpu())
    a, b = out[True], out[False]
    assert a[5] == b[5] and a[5] > 0
    for k in range(5):
        assert torch.equal(a[k], b[k]), k
    assert a[6] is True and b[6] is False
    assert torch.equal(a[7], a[0][: a[7].shape[0]])   # the reference rows are the sorted owned rows


def test_generated_inputs_are_pinned_and_upload_directly(gpu):
    """The engine keeps the positions / velocities it generates in pinned host memory
    (memspace.pinned_array), so the run's upload is a single DMA; values are unchanged."""
    import torch
    from paper_2508_13523_b200 import memspace
    from paper_2508_13523_b200.driver import RunConfig, Simulation
    a = np.random.default_rng(3).random((100_000, 3))
    p = memspace.pinned_array(a)
    assert torch.from_numpy(p).is_pinned() and np.array_equal(p, a) and not np.shares_memory(p, a)
    assert np.array_equal(memspace.upload(p, torch.device("cuda", 0)).cpu().numpy(), a)
    small = np.arange(6.0).reshape(2, 3)
    assert memspace.pinned_array(small) is small or np.array_equal(memspace.pinned_array(small), small)
    sim = Simulation(RunConfig(list_style="full", newton=False), log=None)
    sim.execute(MELT.replace("create_box 8 8 8", "create_box 23 23 23"))
    assert torch.from_numpy(sim._positions).is_pinned() and torch.from_numpy(sim._velocities).is_pinned()
