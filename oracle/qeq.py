"""CPU oracle for charge equilibration (TEST INFRASTRUCTURE ONLY: imported by
tests/ and never by the product path).

numpy restatement of mdkk/qeq.py: the dense shielded matrix by its pairwise
definition (mdkk tests/test_qeq.py:20-32, the reference's own test oracle),
SpMV, conjugate gradient (mdkk/qeq.py:197-230), and the constrained solve
q = s + lambda t (mdkk/qeq.py:293-315) plus the dense KKT reference
(mdkk tests/test_acceptance.py:150-156).  Pinned to the reference's outputs
in tests/golden/qeq.npz (tests/golden/make_golden.py, qeq_fixtures).
"""

from __future__ import annotations

import numpy as np


def dense_matrix(pos, lengths, gamma, eta, cutoff) -> np.ndarray:
    """H_ii = eta, H_ij = (r^3 + gamma^-3)^(-1/3) for minimum-image r < cutoff."""
    n = len(pos)
    lengths = np.asarray(lengths, dtype=np.float64)
    H = np.diag(np.full(n, eta))
    for i in range(n):
        dr = pos - pos[i]
        dr -= lengths * np.round(dr / lengths)
        r = np.sqrt((dr * dr).sum(axis=1))
        for j in range(n):
            if j != i and r[j] < cutoff:
                H[i, j] = (r[j] ** 3 + gamma ** -3.0) ** (-1.0 / 3.0)
    return H


def cg_solve(H, b, tol=1e-6, max_iter=500):
    """Textbook CG to relative residual tol (mdkk/qeq.py:197-230); returns (x, iterations)."""
    b = np.asarray(b, dtype=np.float64)
    x, r = np.zeros_like(b), b.copy()
    p = r.copy()
    rr, bb = float(r @ r), float(b @ b)
    it = 0
    if bb == 0.0:
        return x, 0
    while rr > tol * tol * bb:
        if it >= max_iter:
            raise RuntimeError("CG did not converge")
        Ap = H @ p
        alpha = rr / float(p @ Ap)
        x = x + alpha * p
        r = r - alpha * Ap
        rr_new = float(r @ r)
        p = r + (rr_new / rr) * p
        rr = rr_new
        it += 1
    return x, it


def solve_qeq(H, chi, net_charge=0.0, tol=1e-6):
    """q = s + lambda t, H s = -chi, H t = -1 (mdkk/qeq.py:293-307); returns (q, energy)."""
    n = len(chi)
    s, _ = cg_solve(H, -np.asarray(chi, dtype=np.float64), tol)
    t, _ = cg_solve(H, -np.ones(n), tol)
    lam = (net_charge - s.sum()) / t.sum()
    q = s + lam * t
    return q, float(np.dot(chi, q) + 0.5 * q @ (H @ q))


def kkt_charges(H, chi, net_charge=0.0):
    """Exact constrained minimiser from the dense KKT system."""
    n = len(chi)
    K = np.zeros((n + 1, n + 1))
    K[:n, :n] = H
    K[:n, n] = 1.0
    K[n, :n] = 1.0
    rhs = np.concatenate([-np.asarray(chi, dtype=np.float64), [net_charge]])
    return np.linalg.solve(K, rhs)[:n]
