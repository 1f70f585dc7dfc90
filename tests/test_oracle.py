"""Pin the CPU oracle against the reference's golden vectors and KATs (CPU only)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import md, snap


def _directed(sys, lists):
    out = []
    for rk, nl in zip(sys.ranks, lists):
        sh = np.rint(rk.shift[nl.cols] / sys.lengths).astype(np.int64)
        out.append(np.column_stack([rk.gid[nl.rows], rk.gid[nl.cols], sh,
                                    np.full(len(nl.rows), rk.rank), (nl.weight * 2).astype(np.int64),
                                    nl.write_j.astype(np.int64)]))
    return np.concatenate(out)


def _rowset(a):
    return set(map(tuple, np.asarray(a).tolist()))


@pytest.mark.parametrize("style,newton", [("full", False), ("half", True), ("half", False)])
@pytest.mark.parametrize("n_ranks", [1, 2, 4])
def test_lj_small_matches_reference(style, newton, n_ranks):
    g = golden("lj_small.npz")
    tag = f"{style}_{int(newton)}_{n_ranks}"
    sys = md.Ranked(g["lengths"], n_ranks, g["pos"], np.zeros_like(g["pos"]))
    lists = md.build_all(sys, 2.5, 0.3, style, newton)
    assert _rowset(_directed(sys, lists)) == _rowset(g[f"pairs_{tag}"])
    assert [nl.cap for nl in lists] == g[f"cap_{tag}"].tolist()
    assert [r.n_ghost for r in sys.ranks] == g[f"nghost_{tag}"].tolist()
    e, f, w = md.lj_compute(sys, lists, 1.0, 1.0, 2.5)
    assert e == pytest.approx(float(g[f"E_{tag}"]), rel=1e-13)
    assert np.abs(f - g[f"F_{tag}"]).max() <= 1e-12 * np.abs(g[f"F_{tag}"]).max()
    assert np.allclose(w, g[f"W_{tag}"], rtol=1e-12, atol=1e-10)


def test_lj_small_matches_n2_reference():
    g = golden("lj_small.npz")
    e, f, w = md.lj_reference_n2(g["pos"], g["lengths"], 1.0, 1.0, 2.5)
    assert e == pytest.approx(float(g["E_half_1_1"]), rel=1e-12)
    assert np.allclose(f, g["F_half_1_1"], rtol=1e-12, atol=1e-10)


@pytest.mark.parametrize("style,newton", [("full", False), ("half", True)])
def test_lj_32k_kat(style, newton):
    """SURVEY §8(c) KAT (2): E = -215477.76387663497 (full) on jittered 32k fcc."""
    g = golden("lj_32k_jitter.npz")
    pos, lengths = md.lattice("fcc", 0.8442, (20, 20, 20))
    pos = md.jittered(pos, 0.02, 1)
    sys = md.Ranked(lengths, 1, pos, np.zeros_like(pos))
    lists = md.build_all(sys, 2.5, 0.3, style, newton)
    assert lists[0].cap == int(g[f"cap_{style}"])
    assert len(lists[0].rows) == int(g[f"nentries_{style}"])
    assert sys.ranks[0].n_ghost == int(g[f"nghost_{style}"])
    e, f, w = md.lj_compute(sys, lists, 1.0, 1.0, 2.5)
    assert e == pytest.approx(float(g[f"E_{style}"]), rel=1e-12)
    if style == "full":
        assert e == pytest.approx(-215477.76387663497, rel=1e-12)
    assert np.abs(f[::37] - g[f"F_{style}_sub"]).max() <= 1e-10 * float(g[f"Fmax_{style}"])
    assert np.allclose(w, g[f"W_{style}"], rtol=1e-12)


def test_lattice_kat_energy():
    """SURVEY §8(c) KAT (1): perfect 32k fcc E_pot and KE at T=1.44."""
    pos, lengths = md.lattice("fcc", 0.8442, (20, 20, 20))
    sys = md.Ranked(lengths, 1, pos, np.zeros_like(pos))
    lists = md.build_all(sys, 2.5, 0.3, "full", False)
    e, _, _ = md.lj_compute(sys, lists, 1.0, 1.0, 2.5)
    assert e == pytest.approx(-216747.77770409072, rel=1e-13)
    v = md.seeded_velocities(len(pos), 1.44, 1.0, 87287)
    assert 0.5 * float(np.sum(v * v)) == pytest.approx(69120.0, rel=1e-13)


def test_melt_500_thermo_matches_reference():
    g = golden("lj_runs.npz")
    ref = g["melt500_rows"]
    pos, lengths = md.lattice("fcc", 0.8442, (5, 5, 5))
    vel = md.seeded_velocities(len(pos), 0.05, 1.0, 87287)
    run = md.LJRun(pos, vel, lengths, rc=2.2, skin=0.3, style="half", newton=True)
    rows = np.array(run.run(200, thermo=100))
    assert np.allclose(rows[:, 1:], ref[:3, 1:], rtol=1e-10, atol=1e-10)


# ----------------------------------------------------------------- SNAP
def test_snap_counts_and_cg():
    assert snap.block_offsets(8)[-1] == 285
    assert len(snap.triples(8)) == 55
    assert snap.triples(8)[:3] == [(0, 0, 0), (1, 1, 0), (2, 1, 1)]
    assert sum(len(t[3]) for t in snap.coupling_terms(8)) == 32578
    assert snap.clebsch_gordan(1, 1, 1, -1, 0, 0) == pytest.approx(np.sqrt(0.5), rel=1e-15)
    assert snap.clebsch_gordan(2, 2, 2, -2, 4, 0) == pytest.approx(1 / np.sqrt(6), rel=1e-15)
    assert snap.clebsch_gordan(2, 0, 2, 0, 3, 0) == 0.0


@pytest.mark.parametrize("tag,twoj", [("j2", 2), ("j4", 4), ("j8", 8)])
def test_snap_cluster_matches_reference(tag, twoj):
    g = golden("snap.npz")
    pos = g[f"{tag}_pos"]
    lengths = np.array([12.0] * 3)
    sys = md.Ranked(lengths, 1, pos, np.zeros_like(pos))
    lists = md.build_all(sys, 1.9, 0.2, "full", False)
    so = snap.SnapOracle(twoj, g[f"{tag}_beta"], 1.9)
    rk = sys.ranks[0]
    e, U, Y, F = so.evaluate(rk.x, rk.n_local, lists[0].rows, lists[0].cols)
    o = np.argsort(rk.gid[: rk.n_local])
    assert e == pytest.approx(float(g[f"{tag}_E"]), rel=1e-12)
    assert np.allclose(U[o], g[f"{tag}_U"], rtol=1e-12, atol=1e-14)
    assert np.allclose(Y[o], g[f"{tag}_Y"], rtol=1e-11, atol=1e-13)
    e2, f = snap.snap_compute(sys, lists, so)
    scale = max(1.0, np.abs(g[f"{tag}_F"]).max())
    assert np.abs(f - g[f"{tag}_F"]).max() / scale < 1e-12


def test_snap_periodic_matches_reference():
    g = golden("snap.npz")
    sys = md.Ranked(np.array([6.0] * 3), 1, g["per_pos"], np.zeros_like(g["per_pos"]))
    lists = md.build_all(sys, 1.4, 0.3, "full", False)
    so = snap.SnapOracle(4, g["per_beta"], 1.4)
    e, f = snap.snap_compute(sys, lists, so)
    assert e == pytest.approx(float(g["per_E"]), rel=1e-12)
    assert np.abs(f - g["per_F"]).max() < 1e-12 * max(1.0, np.abs(g["per_F"]).max())
    assert np.abs(f.sum(axis=0)).max() < 1e-10


@pytest.mark.slow
def test_snap_c4_matches_reference():
    g = golden("snap.npz")
    pos, lengths = md.lattice("bcc", 3.1803, (10, 10, 10))
    pos = md.jittered(pos, 0.05, 1)
    sys = md.Ranked(lengths, 1, pos, np.zeros_like(pos))
    lists = md.build_all(sys, 4.73, 0.3, "full", False)
    so = snap.SnapOracle(8, np.linspace(0.05, 0.1, 55), 4.73)
    e, f = snap.snap_compute(sys, lists, so)
    assert e == pytest.approx(float(g["c4_E"]), rel=1e-12)
    assert e == pytest.approx(65509.51457722162, rel=1e-12)
    assert np.abs(f - g["c4_F"]).max() <= 1e-10 * np.abs(g["c4_F"]).max()


def test_qeq_oracle_pinned_to_reference():
    """oracle/qeq.py vs the unmodified reference's QEq outputs (tests/golden/qeq.npz)."""
    from oracle import qeq as oq
    g = golden("qeq.npz")
    for tag in ("a", "b"):
        H = oq.dense_matrix(g[f"{tag}_pos"], g[f"{tag}_L"], 0.8, 20.0, 2.0)
        assert np.abs(H - g[f"{tag}_H"]).max() <= 1e-13
        q, e = oq.solve_qeq(H, g[f"{tag}_chi"], tol=1e-10)
        assert np.allclose(q, g[f"{tag}_q"], rtol=1e-8, atol=1e-12)
        assert e == pytest.approx(float(g[f"{tag}_E"]), rel=1e-8)
        assert np.allclose(oq.kkt_charges(H, g[f"{tag}_chi"]), g[f"{tag}_q"], rtol=1e-6, atol=1e-9)
