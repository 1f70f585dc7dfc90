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
