"""Host-side SNAP tables (CPU): the Z-list product list the yi kernel consumes equals the
reference's three-slot adjoint Y (mdkk/snap/compute.py:303-340) element-wise.

The kernel evaluates Yh[f] = sum coef * op(U[g]) * op(U[h]) over the half set
and mirrors the rest; `zlist_apply` is the same arithmetic in numpy, checked
here against the oracle's compute_y (itself pinned to reference goldens in
test_oracle.py) on U fields built from random neighbourhoods.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import snap as S
from paper_2508_13523_b200.snap.coupling import (device_product_list, make_coupling_tables, zlist_apply,
                                                 zlist_entries)


def _u_field(tjm, beta, seed):
    o = S.SnapOracle(tjm, beta, 4.73)
    rng = np.random.default_rng(seed)
    dr = rng.normal(size=(80, 3))
    dr *= (rng.uniform(1.2, 4.6, 80) / np.linalg.norm(dr, axis=1))[:, None]
    rows = np.repeat(np.arange(4), 20)
    U = o.compute_u(4, rows, dr)
    return o, U


@pytest.mark.parametrize("tjm", [0, 1, 2, 3, 4, 6, 8])
def test_zlist_equals_three_slot_adjoint(tjm):
    n_beta = len(S.triples(tjm))
    beta = np.random.default_rng(tjm).uniform(-1.0, 1.0, n_beta)
    o, U = _u_field(tjm, beta, 7 + tjm)
    Y = o.compute_y(U)
    Yz = zlist_apply(U, tjm, zlist_entries(make_coupling_tables(tjm / 2.0), beta))
    assert np.abs(Yz - Y).max() <= 1e-13 * np.abs(Y).max()
    # and the adjoint-route energy that yi accumulates from the half set
    assert o.energy_from_y(U, Yz) == pytest.approx(o.energy(U), rel=1e-12)


def test_product_list_packing_2j8():
    tab = make_coupling_tables(4.0)
    beta = np.linspace(0.05, 0.1, 55)
    coef, code, n_half, fmap = device_product_list(tab, beta)
    f = (code >> 16) & 255
    assert n_half == 145 and len(fmap) == 285
    assert np.all(np.diff(f) >= 0) and set(f.tolist()) == set(range(145))      # sorted, every output present
    last = (code >> 26) & 1
    assert last[-1] == 1 and np.array_equal(np.flatnonzero(last), np.flatnonzero(np.r_[np.diff(f) != 0, True]))
    assert ((code & 255) < 145).all() and (((code >> 8) & 255) < 145).all()
    assert len(set(f[((code >> 27) & 1) == 1].tolist())) == 5   # self-mirror centre of each even level
    assert len(coef) < 32578   # fewer products than the reference's term count


# --------------------------------------------------------------------------
# The recursion and reverse-mode force the ui / deidrj kernels implement
# (csrc/snap.cu rec2, k_snap_deidrj), restated in numpy and checked against
# the oracle's four-term recursion and forward-mode derivative
# (mdkk/snap/compute.py:125-235, :390-409).

def _in_c(tj, P, Q):
    return 2 * Q < tj or (2 * Q == tj and 2 * P <= tj)


def _levels_two_term(a, b, tj_max):
    u = [np.ones((1, 1), complex)]
    for tj in range(1, tj_max + 1):
        v, new = u[-1], np.zeros((tj + 1, tj + 1), complex)
        for P in range(tj + 1):
            for Q in range(tj + 1):
                if _in_c(tj, P, Q):
                    x = np.sqrt((tj - P) / (tj - Q)) * np.conj(a) * v[P, Q] if P < tj else 0.0
                    if P >= 1:
                        x = x + np.sqrt(P / (tj - Q)) * b * v[P - 1, Q]
                    new[P, Q] = x
                    new[tj - P, tj - Q] = (-1) ** (P + Q) * np.conj(x)
        u.append(new)
    return u


def _pair_force_reverse(d, Y, tj_max, rc):
    r, a, b, fc, dfc, z0, r0 = S.pair_params(d[None], rc)
    da, db = S.pair_grads(d[None], r, rc, a, b, z0, r0)
    a, b, fc, dfc, r, da, db = a[0], b[0], fc[0], dfc[0], r[0], da[0], db[0]
    off = S.block_offsets(tj_max)
    yl = [Y[off[t]:off[t + 1]].reshape(t + 1, t + 1) for t in range(tj_max + 1)]
    u = _levels_two_term(a, b, tj_max)
    Sv = sum((np.conj(yl[t]) * u[t]).sum().real for t in range(tj_max + 1))
    Ga = Gb = 0j
    ln = None
    for tj in range(tj_max, 0, -1):
        lc = np.zeros((tj + 1, tj + 1), complex)

        def g(p, q):
            T, out = tj + 1, 0j
            if ln is None:
                return out
            if _in_c(T, p, q):
                out += np.sqrt((T - p) / (T - q)) * a * ln[p, q]
            if _in_c(T, p + 1, q):
                out += np.sqrt((p + 1) / (T - q)) * np.conj(b) * ln[p + 1, q]
            return out
        for P in range(tj + 1):
            for Q in range(tj + 1):
                if not _in_c(tj, P, Q):
                    continue
                center = 2 * P == tj and 2 * Q == tj
                lam = (1.0 if center else 2.0) * yl[tj][P, Q] + g(P, Q)
                if not center:
                    lam += (-1) ** (P + Q) * np.conj(g(tj - P, tj - Q))
                lc[P, Q] = lam
                v = u[tj - 1]
                if P < tj:
                    Ga += np.conj(lam) * np.sqrt((tj - P) / (tj - Q)) * v[P, Q]
                if P >= 1:
                    Gb += np.conj(lam) * np.sqrt(P / (tj - Q)) * v[P - 1, Q]
        ln = lc
    return np.array([dfc * d[k] / r * Sv + fc * (Ga * np.conj(da[k]) + Gb * db[k]).real for k in range(3)])


def test_two_term_recursion_matches_reference_levels():
    rng = np.random.default_rng(11)
    d = rng.normal(size=(6, 3)) * 2.0
    _, a, b, _, _, _, _ = S.pair_params(d, 4.73)
    u_ref, _ = S.pair_levels(a, b, 8)
    off = S.block_offsets(8)
    for k in range(len(d)):
        u2 = _levels_two_term(a[k], b[k], 8)
        for tj in range(9):
            assert np.abs(u2[tj].ravel() - u_ref[k, off[tj]:off[tj + 1]]).max() < 1e-14


@pytest.mark.parametrize("tjm", [2, 5, 8])
def test_reverse_mode_pair_force_matches_forward_mode(tjm):
    beta = np.linspace(0.05, 0.1, len(S.triples(tjm)))
    o, U = _u_field(tjm, beta, 3)
    Y = o.compute_y(U)[0]
    rng = np.random.default_rng(tjm)
    for _ in range(3):
        d = rng.normal(size=3)
        d *= rng.uniform(1.5, 4.5) / np.linalg.norm(d)
        r, a, b, fc, dfc, z0, r0 = S.pair_params(d[None], 4.73)
        da, db = S.pair_grads(d[None], r, 4.73, a, b, z0, r0)
        u, du = S.pair_levels(a, b, tjm, da, db)
        wdu = fc[:, None, None] * du + (dfc[:, None] * d[None] / r[:, None])[:, :, None] * u[:, None, :]
        t_ref = np.einsum("f,df->d", Y, np.conj(wdu[0])).real
        t = _pair_force_reverse(d, Y, tjm, 4.73)
        assert np.abs(t - t_ref).max() <= 1e-13 * np.abs(t_ref).max()


def test_packed_reuse_ordered_list_still_equals_adjoint():
    """The device list (greedy operand-reuse order, operands swapped where needed) computes
    the same Y as the canonical Z-list, and is ordered for U[g] reuse."""
    tjm = 8
    beta = np.linspace(0.05, 0.1, 55)
    o, U = _u_field(tjm, beta, 21)
    coef, code, n_half, _ = device_product_list(make_coupling_tables(4.0), beta)
    dec = (code >> 16) & 255, code & 255, (code >> 8) & 255, (code >> 24) & 1, (code >> 25) & 1, coef
    Y = o.compute_y(U)
    assert np.abs(zlist_apply(U, tjm, dec) - Y).max() <= 1e-13 * np.abs(Y).max()
    f, g = dec[0], dec[1]
    assert np.sum((f[1:] == f[:-1]) & (g[1:] == g[:-1])) > 0.65 * len(f)
