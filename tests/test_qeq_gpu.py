"""GPU charge equilibration vs the reference (mdkk tests/test_qeq.py, test_acceptance.py:105-160).

The matrix is checked against the pairwise definition (1e-13), the solves
against the dense KKT system and the reference's golden charges, and the
fused dual CG against two sequential solves bit for bit.  Matrix rows are the
store's local rows (as in the reference); the engine keeps owned rows in
spatial order, so the checks map them to global ids (store.global_ids).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import qeq as oq

pytestmark = pytest.mark.gpu

GAMMA, ETA, CHI, RC = 0.8, 20.0, -0.35, 2.0


def _setup(pos, lengths, eta=ETA):
    from paper_2508_13523_b200 import Box, RankedSystem, build_all
    from paper_2508_13523_b200.qeq import QeqParams, build_matrix
    params = QeqParams(gamma=GAMMA, eta=eta, chi=CHI, cutoff=RC)
    system = RankedSystem.distribute(Box(lengths), 1, pos, np.zeros_like(pos))
    (nl,) = build_all(system, RC, 0.3, style="full", newton=False)
    H = build_matrix(system.stores[0], nl, params)
    st = system.stores[0]
    return H, system, st.global_ids[: st.n_local].astype(np.int64)


def test_matrix_layout_and_values(gpu):
    g = golden("qeq.npz")
    H, system, gid = _setup(g["a_pos"], g["a_L"])
    assert np.abs(H.to_dense() - g["a_H"][np.ix_(gid, gid)]).max() <= 1e-13
    starts = H.row_offsets[:-1]
    assert np.all(H.values[starts] == ETA)                       # diagonal first in every row
    assert np.array_equal(H.columns[starts], np.arange(H.n_rows))
    caps = np.diff(H.row_offsets)
    assert H.row_offsets.dtype == np.int64
    assert np.all(H.row_nnz <= caps) and np.any(H.row_nnz < caps)   # over-allocation is real


def test_spmv_fused_and_solvers(gpu):
    from paper_2508_13523_b200.qeq import cg_solve, cg_solve_fused, spmv, spmv_fused, spmv_rowchunk
    g = golden("qeq.npz")
    H, _, gid = _setup(g["b_pos"], g["b_L"])
    Hd = g["b_H"][np.ix_(gid, gid)]
    rng = np.random.default_rng(20260825)
    x1, x2 = rng.normal(size=(2, H.n_rows))
    y = spmv(H, x1)
    assert np.allclose(y, Hd @ x1, rtol=1e-13, atol=1e-13)
    f1, f2 = spmv_fused(H, x1, x2)
    assert np.array_equal(f1, y) and np.array_equal(f2, spmv(H, x2))
    assert np.allclose(spmv_rowchunk(H, x1, 3), y, rtol=1e-13, atol=1e-13)
    x, iters = cg_solve(H, x1, tol=1e-12)
    assert np.allclose(x, np.linalg.solve(Hd, x1), rtol=1e-8, atol=1e-10) and 0 < iters < 200
    t1, t2, u1, u2 = [], [], [], []
    a1, i1 = cg_solve(H, x1, trajectory=t1)
    a2, i2 = cg_solve(H, x2, trajectory=t2)
    b1, b2, j1, j2 = cg_solve_fused(H, x1, x2, trajectories=(u1, u2))
    assert (i1, i2) == (j1, j2)
    assert np.array_equal(a1, b1) and np.array_equal(a2, b2)
    for (ia, xa, ra), (ib, xb, rb) in zip(t1 + t2, u1 + u2):
        assert ia == ib and np.array_equal(xa, xb) and np.array_equal(ra, rb)


def test_solve_qeq_matches_reference_and_kkt(gpu):
    from paper_2508_13523_b200.qeq import QeqSystem, qeq_energy, solve_qeq
    g = golden("qeq.npz")
    for tag in ("a", "b"):
        H, _, gid = _setup(g[f"{tag}_pos"], g[f"{tag}_L"])
        qs = QeqSystem(H, g[f"{tag}_chi"][gid], tol=1e-10)
        q = np.empty(H.n_rows)
        q[gid] = solve_qeq(qs)          # back to global-id order
        assert abs(q.sum()) <= 1e-10
        assert np.allclose(q, g[f"{tag}_q"], rtol=1e-8, atol=1e-12)
        assert np.allclose(q, oq.kkt_charges(g[f"{tag}_H"], g[f"{tag}_chi"]), rtol=1e-6, atol=1e-9)
        assert qeq_energy(qs) == pytest.approx(float(g[f"{tag}_E"]), rel=1e-8)
        assert tuple(qs.iterations) == tuple(g[f"{tag}_iters"])


def test_guards_and_errors(gpu):
    from paper_2508_13523_b200.qeq import QeqConfigError, QeqError, QeqSystem, cg_solve, check_spd, solve_qeq
    g = golden("qeq.npz")
    H, _, _ = _setup(g["a_pos"], g["a_L"], eta=0.01)
    with pytest.raises(QeqConfigError):
        check_spd(H)
    with pytest.raises(QeqConfigError):
        solve_qeq(QeqSystem(H, np.full(H.n_rows, CHI)))
    H, _, _ = _setup(g["a_pos"], g["a_L"])
    with pytest.raises(QeqError):
        cg_solve(H, np.ones(H.n_rows), tol=1e-30, max_iter=2)
    with pytest.raises(QeqError):
        QeqSystem(H, np.zeros(3))


def test_qeq_thermo_diagnostic(gpu):
    """`qeq on ...` logs (step, iters_s, iters_t, sum_q, energy) at thermo steps (mdkk/driver/simulation.py:417-429)."""
    from paper_2508_13523_b200.driver import RunConfig, run_script
    text = ("units lj\nboundary p p p\nlattice fcc 0.8442\ncreate_box 5 5 5\ncreate_atoms\nmass 1.0\n"
            "velocity 1.0 87287\npair_style lj/cut 2.5\npair_coeff 1.0 1.0\nqeq on 0.8 20.0 -0.35 2.0\n"
            "timestep 0.005\nthermo 10\nrun 20\n")
    sim = run_script(text, RunConfig(), log=None)
    log = sim.results[-1].qeq_log
    assert [r[0] for r in log] == [0, 10, 20]
    for step, its, itt, sq, e in log:
        assert its >= 0 and itt > 0 and abs(sq) < 1e-10 and np.isfinite(e)


def test_energy_stationary_net_charge_target_and_order(gpu):
    """mdkk tests/test_qeq.py:147-184: constrained minimum (perturbations preserving the
    net charge do not lower the energy), a nonzero net-charge target, energy before solve."""
    from paper_2508_13523_b200.qeq import QeqError, QeqSystem, qeq_energy, solve_qeq
    g = golden("qeq.npz")
    H, _, gid = _setup(g["b_pos"], g["b_L"])
    Hd = g["b_H"][np.ix_(gid, gid)]
    chi = np.full(H.n_rows, CHI)
    with pytest.raises(QeqError):
        qeq_energy(QeqSystem(H, chi))
    qs = QeqSystem(H, chi, tol=1e-10)
    q = solve_qeq(qs)
    e = qeq_energy(qs)
    rng = np.random.default_rng(1)
    for _ in range(5):
        d = rng.normal(size=H.n_rows)
        d -= d.mean()
        d *= 1e-4 / np.linalg.norm(d)
        assert chi @ (q + d) + 0.5 * (q + d) @ (Hd @ (q + d)) >= e - 1e-9
    q5 = solve_qeq(QeqSystem(H, chi, net_charge=0.5, tol=1e-10))
    assert q5.sum() == pytest.approx(0.5, abs=1e-10)
