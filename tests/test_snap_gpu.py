"""GPU parity for the SNAP pipeline vs the reference goldens and the CPU oracle.

Mirrors mdkk tests/test_snap.py (closed forms, cluster invariants, periodic
force balance) and SURVEY §8(c)'s C4 KAT.  Tolerances: energy 1e-12
relative, forces 1e-10 * max|F|, U / Y 1e-12 relative.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import md, snap as osnap

pytestmark = pytest.mark.gpu


def _pipeline(pos, lengths, jmax, beta, rc, skin):
    from paper_2508_13523_b200 import Box, RankedSystem, build_all
    from paper_2508_13523_b200.snap import (SnapState, build_neighbor_map, compute_fused_deidrj, compute_ui,
                                            compute_yi, energy_from_y, make_coupling_tables)
    system = RankedSystem.distribute(Box(lengths), 1, pos, np.zeros_like(pos))
    (nl,) = build_all(system, rc, skin, style="full", newton=False)
    store = system.stores[0]
    nmap = build_neighbor_map(store, nl, rc)
    state = SnapState(make_coupling_tables(jmax), store.n_local, beta)
    compute_ui(nmap, state)
    compute_yi(state)
    f = compute_fused_deidrj(nmap, state, store.n_total)
    fr = store.force.read("a")
    fr[: store.n_total] = f
    store.force.mark_modified("a")
    system.reverse_comm()
    o = np.argsort(store.global_ids[: store.n_local])
    return energy_from_y(state), system.gather_forces(), state.u_view()[o], state.y_view()[o]


@pytest.mark.parametrize("tag,jmax", [("j2", 1), ("j4", 2), ("j8", 4)])
def test_cluster_matches_reference(gpu, tag, jmax):
    g = golden("snap.npz")
    e, f, u, y = _pipeline(g[f"{tag}_pos"], np.array([12.0] * 3), jmax, g[f"{tag}_beta"], 1.9, 0.2)
    assert e == pytest.approx(float(g[f"{tag}_E"]), rel=1e-12)
    assert np.allclose(u, g[f"{tag}_U"], rtol=1e-12, atol=1e-14)
    assert np.allclose(y, g[f"{tag}_Y"], rtol=1e-11, atol=1e-13)
    scale = max(1.0, np.abs(g[f"{tag}_F"]).max())
    assert np.abs(f - g[f"{tag}_F"]).max() / scale < 1e-10


def test_periodic_matches_reference_and_balances(gpu):
    g = golden("snap.npz")
    e, f, _, _ = _pipeline(g["per_pos"], np.array([6.0] * 3), 2, g["per_beta"], 1.4, 0.3)
    assert e == pytest.approx(float(g["per_E"]), rel=1e-12)
    assert np.abs(f - g["per_F"]).max() < 1e-10 * max(1.0, np.abs(g["per_F"]).max())
    assert np.abs(f.sum(axis=0)).max() < 1e-10


def test_c4_2000_bcc_matches_reference(gpu):
    """SURVEY §8(c) KAT (3): E = 65509.51457722162 on jittered 2k bcc, 2J=8, rc 4.73."""
    g = golden("snap.npz")
    pos, lengths = md.lattice("bcc", 3.1803, (10, 10, 10))
    pos = md.jittered(pos, 0.05, 1)
    e, f, u, y = _pipeline(pos, lengths, 4, np.linspace(0.05, 0.1, 55), 4.73, 0.3)
    assert e == pytest.approx(float(g["c4_E"]), rel=1e-12)
    assert e == pytest.approx(65509.51457722162, rel=1e-12)
    assert np.abs(f - g["c4_F"]).max() <= 1e-10 * np.abs(g["c4_F"]).max()
    assert np.allclose(u[:16], g["c4_U_sub"], rtol=1e-12, atol=1e-12)
    assert np.allclose(y[:16], g["c4_Y_sub"], rtol=1e-11, atol=1e-11)


def test_c4_perfect_lattice_energy(gpu):
    g = golden("snap.npz")
    pos, lengths = md.lattice("bcc", 3.1803, (10, 10, 10))
    e, f, _, _ = _pipeline(pos, lengths, 4, np.linspace(0.05, 0.1, 55), 4.73, 0.3)
    assert e == pytest.approx(float(g["c4_lattice_E"]), rel=1e-12)
    assert e == pytest.approx(64610.777035472027, rel=1e-12)
    assert np.abs(f).max() < 1e-9


def test_single_pair_closed_form(gpu):
    """mdkk tests/test_snap.py:375-395 (jmax 1/2: B = (fc^3, 2 fc^3))."""
    d, rc = 1.3, 1.9
    pos = np.array([[5.0, 5.0, 5.0], [5.0 + d, 5.0, 5.0]])
    beta = np.array([0.37, -0.21])
    e, f, u, y = _pipeline(pos, np.array([12.0] * 3), 0.5, beta, rc, 0.2)
    fc = 0.5 * (1 + np.cos(np.pi * d / rc))
    dfc = -np.pi / (2 * rc) * np.sin(np.pi * d / rc)
    assert e == pytest.approx(2 * (beta[0] + 2 * beta[1]) * fc ** 3, rel=1e-12)
    assert u[0, 0] == pytest.approx(fc, rel=1e-14)
    assert y[0, 0] == pytest.approx(3 * beta[0] * fc ** 2 + 2 * beta[1] * fc ** 2, rel=1e-12)
    assert f[0] == pytest.approx([2 * (beta[0] + 2 * beta[1]) * 3 * fc ** 2 * dfc, 0.0, 0.0], abs=1e-12)


def test_zero_distance_raises(gpu):
    from paper_2508_13523_b200.snap import SnapError
    with pytest.raises(SnapError):
        from paper_2508_13523_b200 import Box, RankedSystem, build_all
        from paper_2508_13523_b200.snap import (SnapState, build_neighbor_map, compute_ui, make_coupling_tables)
        from paper_2508_13523_b200.snap.compute import check_flags
        system = RankedSystem.distribute(Box((12.0,) * 3), 1, np.full((2, 3), 5.0), np.zeros((2, 3)))
        (nl,) = build_all(system, 1.9, 0.2, style="full", newton=False)
        st = SnapState(make_coupling_tables(1), 2, np.zeros(5))
        compute_ui(build_neighbor_map(system.stores[0], nl, 1.9), st)
        check_flags(st)


def test_snap_style_nve_matches_oracle(gpu, tmp_path):
    """snap/kk through run_script vs the oracle's SNAP NVE (same lattice, velocities, dt)."""
    from paper_2508_13523_b200.driver import RunConfig, run_script
    coeff = tmp_path / "w.coeff"
    beta = np.linspace(0.05, 0.1, 14)
    coeff.write_text("2\n" + "\n".join(repr(float(b)) for b in beta) + "\n")
    script = (f"units lj\nboundary p p p\nlattice bcc 3.1803\ncreate_box 4 4 4\ncreate_atoms\nmass 1.0\n"
              f"velocity 0.5 4928459\nsuffix kk\npair_style snap 4.73 {coeff}\ntimestep 0.001\nthermo 5\nrun 10\n")
    sim = run_script(script, RunConfig(), log=None)
    rows = np.array(sim.results[-1].rows)
    # oracle: same physics through oracle/snap.py
    pos, L = md.lattice("bcc", 3.1803, (4, 4, 4))
    vel = md.seeded_velocities(len(pos), 0.5, 1.0, 4928459)
    so = osnap.SnapOracle(4, beta, 4.73)
    sys_ = md.Ranked(L, 1, pos, vel)
    lists = md.build_all(sys_, 4.73, 0.3, "full", False)
    e0, _ = osnap.snap_compute(sys_, lists, so)
    ref = [e0]
    h = 0.5 * 0.001
    for step in range(1, 11):
        for r in sys_.ranks:
            r.v += h * r.f[: r.n_local]
            r.x[: r.n_local] += 0.001 * r.v
        if any(nl.needs_rebuild() for nl in lists):
            sys_.migrate(5.03)
            lists = [md.build(r, L, 4.73, 0.3, "full", False) for r in sys_.ranks]
        else:
            sys_.forward()
        e, _ = osnap.snap_compute(sys_, lists, so)
        for r in sys_.ranks:
            r.v += h * r.f[: r.n_local]
        if step % 5 == 0:
            ref.append(e)
    assert np.allclose(rows[:, 1], ref, rtol=1e-10)


# ---------------------------------------------------------------- API-parity stages
def _state_for(pos, lengths, jmax, beta, rc, skin):
    from paper_2508_13523_b200 import Box, RankedSystem, build_all
    from paper_2508_13523_b200.snap import SnapState, build_neighbor_map, compute_ui, compute_yi, make_coupling_tables
    system = RankedSystem.distribute(Box(lengths), 1, pos, np.zeros_like(pos))
    (nl,) = build_all(system, rc, skin, style="full", newton=False)
    store = system.stores[0]
    nmap = build_neighbor_map(store, nl, rc)
    state = SnapState(make_coupling_tables(jmax), store.n_local, beta)
    compute_ui(nmap, state)
    compute_yi(state)
    return system, store, nmap, state


def test_neighbor_map_arrays_match_reference_order(gpu):
    """Pairs within r_c in (row, dz, dy, dx) order with unit-sphere a, b (mdkk tests/test_snap.py:305-323)."""
    g = golden("snap.npz")
    pos = g["j4_pos"]
    system, store, nmap, _ = _state_for(pos, np.array([12.0] * 3), 2, g["j4_beta"], 1.9, 0.2)
    o = osnap.SnapOracle(4, g["j4_beta"], 1.9)
    rows, cols, _, _ = nmap.nlist.pairs()
    x = store.positions()
    r_rows, r_cols, r_dr = o.pairs_from_list(x, rows, cols)
    assert nmap.n_pairs == len(r_rows)
    assert np.array_equal(nmap.rows, r_rows) and np.array_equal(nmap.cols, r_cols)
    assert np.array_equal(nmap.dr, r_dr)
    assert np.all(nmap.r <= 1.9) and np.all(nmap.r > 0)
    assert np.allclose(np.abs(nmap.a) ** 2 + np.abs(nmap.b) ** 2, 1.0, atol=1e-12)
    r, a, b, fc, dfc, _, _ = osnap.pair_params(r_dr, 1.9)
    assert np.allclose(nmap.a, a, rtol=0, atol=1e-14) and np.allclose(nmap.b, b, rtol=0, atol=1e-14)
    assert np.allclose(nmap.fc, fc, rtol=1e-13, atol=1e-15) and np.allclose(nmap.dfc, dfc, rtol=1e-13, atol=1e-15)


def test_staged_path_matches_oracle_and_fused(gpu):
    """compute_duidrj == the reference's per-pair d(f_c u)/dr; staged == fused forces (mdkk tests/test_snap.py:465-478)."""
    from paper_2508_13523_b200.snap import compute_deidrj, compute_duidrj, compute_fused_deidrj
    g = golden("snap.npz")
    bcc, L = md.lattice("bcc", 3.1803, (4, 4, 4))
    cases = ((g["j4_pos"], np.array([12.0] * 3), 2, g["j4_beta"], 1.9, 0.2),
             (md.jittered(bcc, 0.05, 2), L, 4, np.linspace(0.05, 0.1, 55), 4.73, 0.3))
    for pos, lengths, jmax, beta, rc, skin in cases:
        system, store, nmap, state = _state_for(pos, lengths, jmax, beta, rc, skin)
        assert nmap.n_pairs > 0
        du = compute_duidrj(nmap, state)
        dr = nmap.dr
        r, a, b, fc, dfc, z0, r0 = osnap.pair_params(dr, rc)
        da, db = osnap.pair_grads(dr, r, rc, a, b, z0, r0)
        u, dun = osnap.pair_levels(a, b, 2 * jmax, da, db)
        wdu = fc[:, None, None] * dun + (dfc[:, None] * dr / r[:, None])[:, :, None] * u[:, None, :]
        assert np.abs(du - wdu).max() <= 1e-12 * np.abs(wdu).max()
        fused = compute_fused_deidrj(nmap, state, store.n_total)
        staged = compute_deidrj(nmap, state, du, store.n_total)
        assert np.abs(staged - fused).max() <= 1e-12 * max(1.0, np.abs(fused).max())


def test_descriptors_and_energy_routes(gpu):
    """compute_bi_complex vs the oracle's invariants; descriptor and adjoint energies agree
    (mdkk tests/test_snap.py:328-372); imaginary residue negligible."""
    from paper_2508_13523_b200.snap import compute_bi, compute_bi_complex, compute_energy, energy_from_y
    pos, lengths = md.lattice("bcc", 3.1803, (10, 10, 10))
    pos = md.jittered(pos, 0.05, 1)
    beta = np.linspace(0.05, 0.1, 55)
    system, store, nmap, state = _state_for(pos, lengths, 4, beta, 4.73, 0.3)
    bc = compute_bi_complex(state)
    o = osnap.SnapOracle(8, beta, 4.73)
    U = state.u_view()
    ref = np.stack([((c * U[:, i1]) * U[:, i2] * np.conj(U[:, iz])).sum(axis=1) for (iz, i1, i2, c) in o.terms], 1)
    assert np.abs(bc - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
    assert np.abs(bc.imag).max() < 1e-10 * max(1.0, np.abs(bc.real).max())
    assert np.array_equal(compute_bi(state), bc.real)
    assert compute_energy(state) == pytest.approx(energy_from_y(state), rel=1e-12)
    assert compute_energy(state) == pytest.approx(65509.51457722162, rel=1e-12)   # SURVEY §8(c) KAT (3)


def test_knobs_do_not_change_results(gpu):
    """mdkk tests/test_snap.py:482-499: layout / tile_v / batch knobs leave E and F unchanged (1e-12)."""
    from paper_2508_13523_b200 import Box, RankedSystem, build_all
    from paper_2508_13523_b200.snap import (SnapState, build_neighbor_map, compute_bi, compute_energy,
                                            compute_fused_deidrj, compute_ui, compute_yi, energy_from_y,
                                            make_coupling_tables)
    pos, lengths = md.lattice("bcc", 3.1803, (5, 5, 5))
    pos = md.jittered(pos, 0.05, 5)
    beta = np.random.default_rng(67).uniform(-0.1, 0.1, 55)
    tables = make_coupling_tables(4)
    system = RankedSystem.distribute(Box(lengths), 1, pos, np.zeros_like(pos))
    (nl,) = build_all(system, 4.73, 0.3, style="full", newton=False)
    store = system.stores[0]
    nmap = build_neighbor_map(store, nl, 4.73)

    def run(**knobs):
        st = SnapState(tables, store.n_local, beta, **knobs)
        compute_ui(nmap, st)
        compute_yi(st)
        f = compute_fused_deidrj(nmap, st, store.n_total)
        return energy_from_y(st), f, st.u_view().copy(), st.y_view().copy(), compute_bi(st), compute_energy(st)

    e0, f0, u0, y0, b0, eb0 = run()
    fscale = max(1.0, np.abs(f0).max())
    for knobs in ({"batch_u": 1}, {"batch_u": 2}, {"batch_u": 16}, {"batch_y": 3}, {"batch_y": 2, "batch_u": 1},
                  {"tile_v": 1}, {"tile_v": 37},
                  {"layout": "b"}, {"batch_u": 2, "batch_y": 4, "tile_v": 64, "layout": "b"}):
        e1, f1, u1, y1, b1, eb1 = run(**knobs)
        assert e1 == pytest.approx(e0, rel=1e-12), knobs
        assert eb1 == pytest.approx(eb0, rel=1e-12), knobs
        assert np.abs(f1 - f0).max() / fscale < 1e-12, knobs
        # batch_u regroups the per-warp pair sums of U (rounding only); the reference asserts E and F
        assert np.allclose(u1, u0, rtol=1e-13, atol=1e-14) and np.allclose(y1, y0, rtol=1e-13, atol=1e-14), knobs
        assert np.allclose(b1, b0, rtol=1e-13, atol=1e-13), knobs


def test_one_call_pipeline_bit_identical(gpu):
    """mdkk_snap_compute (handle workspace and caller dumps) == ui -> yi -> fused deidrj: U, Y and E bit
    for bit; F up to the order of the FP64 atomics that fold f_k."""
    import torch
    from paper_2508_13523_b200 import _lib
    from paper_2508_13523_b200.snap import compute_fused_deidrj, energy_from_y
    bcc, L = md.lattice("bcc", 3.1803, (4, 4, 4))
    system, store, nmap, state = _state_for(md.jittered(bcc, 0.05, 5), L, 4, np.linspace(0.05, 0.1, 55), 4.73, 0.3)
    f_ref = compute_fused_deidrj(nmap, state, store.n_total)
    e_ref = energy_from_y(state)
    nl, dev, n = nmap.nlist, state.device, store.n_local
    for dumps in (False, True):
        f = torch.zeros((store.n_total, 4), dtype=torch.float64, device=dev)
        e = torch.zeros(1, dtype=torch.float64, device=dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        U = torch.zeros((n, state.index.n_flat), dtype=torch.complex128, device=dev) if dumps else None
        Yh = torch.zeros((145, n), dtype=torch.complex128, device=dev) if dumps else None
        for _ in range(2):      # the second call reuses the grown workspace
            f.zero_()
            _lib.check(_lib.lib().mdkk_snap_compute(
                _lib.ctx(dev), state.handle().ptr, store.x.data_ptr(), n, nl.table_dev.data_ptr(),
                nl.counts_dev.data_ptr(), nl.alloc_cap, 4.73, U.data_ptr() if dumps else None,
                Yh.data_ptr() if dumps else None, f.data_ptr(), e.data_ptr(), flags.data_ptr(),
                _lib.stream(dev)), "mdkk_snap_compute")
        assert int(flags.item()) == 0
        assert float(e.item()) == e_ref
        assert np.abs(f[:, :3].cpu().numpy() - f_ref).max() <= 1e-13 * np.abs(f_ref).max()
        if dumps:   # default layout "a": U rows are atoms, as the handle writes them
            assert state._lay == 0
            assert np.array_equal(U.cpu().numpy(), state.U_dev[:n].cpu().numpy())
            assert np.array_equal(Yh.cpu().numpy(), state.Yh_dev[:, :n].cpu().numpy())
