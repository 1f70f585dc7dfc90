"""Numpy restatement of the reference SNAP pipeline — TEST INFRASTRUCTURE ONLY.

Restates (does not import) mdkk/snap/{indexing,coupling,compute}.py:

* flat (tj, p, q) index, coupled triples     — snap/indexing.py:24-68
* exact-rational Clebsch-Gordan, term tables — snap/coupling.py:28-133
* Cayley-Klein map, switch, gradients        — snap/compute.py:27-63
* four-term level recursion (+ derivative)   — snap/compute.py:125-184
* U, full three-slot adjoint Y, energy, F    — snap/compute.py:279-409

Used by tests/ and bench.py's CPU-baseline legs only.
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


class SnapOracleError(RuntimeError):
    pass


# ------------------------------------------------------------------ indexing
def block_offsets(twojmax: int) -> np.ndarray:
    """off[tj] = sum_{t<tj} (t+1)^2 (snap/indexing.py:30-32)."""
    return np.concatenate([[0], np.cumsum([(t + 1) ** 2 for t in range(twojmax + 1)])]).astype(np.int64)


def triples(twojmax: int):
    """(tj, tj1, tj2), tj slowest; tj2<=tj1<=tj, triangle + parity (snap/indexing.py:56-68)."""
    return [(tj, tj1, tj2) for tj in range(twojmax + 1) for tj1 in range(tj + 1)
            for tj2 in range(tj1 + 1) if tj <= tj1 + tj2 and (tj1 + tj2 - tj) % 2 == 0]


# ------------------------------------------------------------------ coupling
def _hf(twice: int) -> int:
    return math.factorial(twice // 2)


def clebsch_gordan(tj1, tm1, tj2, tm2, tj, tm) -> float:
    """<j1 m1; j2 m2 | j m>, doubled args, Racah sum in exact rationals (snap/coupling.py:28-66)."""
    if tm1 + tm2 != tm or not (abs(tj1 - tj2) <= tj <= tj1 + tj2) or (tj1 + tj2 - tj) % 2:
        return 0.0
    if abs(tm1) > tj1 or abs(tm2) > tj2 or abs(tm) > tj:
        return 0.0
    if (tj1 + tm1) % 2 or (tj2 + tm2) % 2 or (tj + tm) % 2:
        return 0.0
    pref = Fraction((tj + 1) * _hf(tj1 + tj2 - tj) * _hf(tj1 - tj2 + tj) * _hf(tj2 - tj1 + tj)
                    * _hf(tj1 + tm1) * _hf(tj1 - tm1) * _hf(tj2 + tm2) * _hf(tj2 - tm2)
                    * _hf(tj + tm) * _hf(tj - tm), _hf(tj1 + tj2 + tj + 2))
    s = Fraction(0)
    k_lo = max(0, (tj2 - tj - tm1) // 2, (tj1 - tj + tm2) // 2)
    k_hi = min((tj1 + tj2 - tj) // 2, (tj1 - tm1) // 2, (tj2 + tm2) // 2)
    for k in range(k_lo, k_hi + 1):
        d = (math.factorial(k) * _hf(tj1 + tj2 - tj - 2 * k) * _hf(tj1 - tm1 - 2 * k)
             * _hf(tj2 + tm2 - 2 * k) * _hf(tj - tj2 + tm1 + 2 * k) * _hf(tj - tj1 - tm2 + 2 * k))
        s += Fraction((-1) ** k, d)
    if s == 0:
        return 0.0
    return math.copysign(math.sqrt(float(s * s * pref)), float(s))


def coupling_terms(twojmax: int):
    """Per-triple flattened (iz, iu1, iu2, coeff) lists (snap/coupling.py:106-133)."""
    off = block_offsets(twojmax)
    out = []
    for (tj, tj1, tj2) in triples(twojmax):
        cg = np.zeros((tj1 + 1, tj2 + 1))
        for p1 in range(tj1 + 1):
            for p2 in range(tj2 + 1):
                tm = 2 * p1 - tj1 + 2 * p2 - tj2
                if abs(tm) <= tj:
                    cg[p1, p2] = clebsch_gordan(tj1, 2 * p1 - tj1, tj2, 2 * p2 - tj2, tj, tm)
        sh = (tj1 + tj2 - tj) // 2
        p1, p2, q1, q2 = (v.ravel() for v in np.meshgrid(np.arange(tj1 + 1), np.arange(tj2 + 1),
                                                         np.arange(tj1 + 1), np.arange(tj2 + 1),
                                                         indexing="ij"))
        p, q = p1 + p2 - sh, q1 + q2 - sh
        c = cg[p1, p2] * cg[q1, q2]
        k = (p >= 0) & (p <= tj) & (q >= 0) & (q <= tj) & (c != 0.0)
        out.append((off[tj] + p[k] * (tj + 1) + q[k],
                    off[tj1] + p1[k] * (tj1 + 1) + q1[k],
                    off[tj2] + p2[k] * (tj2 + 1) + q2[k], c[k]))
    return out


# --------------------------------------------------------------- pair params
def pair_params(dr, rc):
    """a, b, f_c, f_c', z0, r0 (snap/compute.py:27-45)."""
    r = np.sqrt(np.einsum("ij,ij->i", dr, dr))
    ct = 0.99 * np.pi / rc
    z0 = r / np.tan(ct * r)
    r0 = np.sqrt(r * r + z0 * z0)
    a = (z0 - 1j * dr[:, 2]) / r0
    b = (dr[:, 1] - 1j * dr[:, 0]) / r0
    fc = 0.5 * (1.0 + np.cos(np.pi * r / rc))
    dfc = -np.pi / (2.0 * rc) * np.sin(np.pi * r / rc)
    return r, a, b, fc, dfc, z0, r0


def pair_grads(dr, r, rc, a, b, z0, r0):
    """d a / d dr_d, d b / d dr_d (snap/compute.py:48-63)."""
    ct = 0.99 * np.pi / rc
    dz0 = ((z0 / r - ct * (r * r + z0 * z0) / r) / r)[:, None] * dr
    dr0 = (dr + z0[:, None] * dz0) / r0[:, None]
    ez = np.zeros((len(r), 3), complex)
    ez[:, 2] = -1j
    eb = np.zeros((len(r), 3), complex)
    eb[:, 0], eb[:, 1] = -1j, 1.0
    da = (dz0 + ez) / r0[:, None] - a[:, None] * dr0 / r0[:, None]
    db = eb / r0[:, None] - b[:, None] * dr0 / r0[:, None]
    return da, db


def _weights(tj):
    p = np.arange(1, tj + 1, dtype=np.float64)
    q = np.arange(tj, dtype=np.float64)
    return (np.sqrt(np.outer(p, q + 1)) / tj, np.sqrt(np.outer(p, tj - q)) / tj,
            np.sqrt(np.outer(tj - p + 1, q + 1)) / tj, np.sqrt(np.outer(tj - p + 1, tj - q)) / tj)


def pair_levels(a, b, twojmax, da=None, db=None):
    """Flat u (n, F) and optionally du (n, 3, F) (snap/compute.py:138-184,187-235)."""
    off = block_offsets(twojmax)
    n = len(a)
    u = np.empty((n, off[-1]), complex)
    u[:, 0] = 1.0
    want_d = da is not None
    if want_d:
        du = np.zeros((n, 3, off[-1]), complex)
    lev = np.ones((n, 1, 1), complex)
    dlev = np.zeros((n, 3, 1, 1), complex)
    ca, cb = np.conj(a), np.conj(b)
    for tj in range(1, twojmax + 1):
        if tj == 1:
            new = np.stack([np.stack([ca, -cb], -1), np.stack([b, a], -1)], -2)
            if want_d:
                dnew = np.stack([np.stack([np.conj(da), -np.conj(db)], -1),
                                 np.stack([db, da], -1)], -2)
        else:
            w11, w10, w01, w00 = _weights(tj)
            new = np.zeros((n, tj + 1, tj + 1), complex)
            new[:, 1:, 1:] += w11 * (lev * a[:, None, None])
            new[:, 1:, :-1] += w10 * (lev * b[:, None, None])
            new[:, :-1, 1:] += w01 * (lev * (-cb)[:, None, None])
            new[:, :-1, :-1] += w00 * (lev * ca[:, None, None])
            if want_d:
                L = lev[:, None]
                dnew = np.zeros((n, 3, tj + 1, tj + 1), complex)
                dnew[:, :, 1:, 1:] += w11 * (dlev * a[:, None, None, None] + L * da[:, :, None, None])
                dnew[:, :, 1:, :-1] += w10 * (dlev * b[:, None, None, None] + L * db[:, :, None, None])
                dnew[:, :, :-1, 1:] += w01 * (dlev * (-cb)[:, None, None, None]
                                              + L * (-np.conj(db))[:, :, None, None])
                dnew[:, :, :-1, :-1] += w00 * (dlev * ca[:, None, None, None]
                                               + L * np.conj(da)[:, :, None, None])
        lev = new
        u[:, off[tj]:off[tj + 1]] = new.reshape(n, -1)
        if want_d:
            dlev = dnew
            du[:, :, off[tj]:off[tj + 1]] = dnew.reshape(n, 3, -1)
    return (u, du) if want_d else (u, None)


# ------------------------------------------------------------------ pipeline
class SnapOracle:
    """U / Y / energy / forces for one rank's full list (snap/compute.py:105-409)."""

    def __init__(self, twojmax: int, beta, rc: float):
        self.twojmax = int(twojmax)
        self.off = block_offsets(self.twojmax)
        self.nf = int(self.off[-1])
        self.tri = triples(self.twojmax)
        self.beta = np.asarray(beta, dtype=np.float64)
        if self.beta.shape != (len(self.tri),):
            raise SnapOracleError("beta must have one value per coupled triple")
        self.rc = float(rc)
        self.terms = coupling_terms(self.twojmax)

    def pairs_from_list(self, x, rows, cols):
        """r < rc filter, order (row, dz, dy, dx) (snap/compute.py:66-119)."""
        dr = x[cols] - x[rows]
        r2 = np.einsum("ij,ij->i", dr, dr)
        m = r2 < self.rc * self.rc
        rows, cols, dr, r2 = rows[m], cols[m], dr[m], r2[m]
        if np.any(r2 <= 0.0):
            raise SnapOracleError("neighbor at zero distance")
        o = np.lexsort((dr[:, 0], dr[:, 1], dr[:, 2], rows))
        return rows[o], cols[o], dr[o]

    def compute_u(self, n_atoms, rows, dr, chunk=16384):
        U = np.zeros((n_atoms, self.nf), complex)
        for s in range(0, len(rows), chunk):
            sl = slice(s, s + chunk)
            r, a, b, fc, _, _, _ = pair_params(dr[sl], self.rc)
            u, _ = pair_levels(a, b, self.twojmax)
            np.add.at(U, rows[sl], fc[:, None] * u)
        return U

    def compute_y(self, U):
        """Full three-slot adjoint (snap/compute.py:303-340)."""
        Y = np.zeros_like(U)
        for bt, (iz, i1, i2, c) in zip(self.beta, self.terms):
            if bt == 0.0:
                continue
            u1, u2, uz = U[:, i1], U[:, i2], U[:, iz]
            np.add.at(Y.T, iz, (bt * (c * u1) * u2).T)
            np.add.at(Y.T, i1, (bt * (c * np.conj(u2)) * uz).T)
            np.add.at(Y.T, i2, (bt * (c * np.conj(u1)) * uz).T)
        return Y

    def bispectrum(self, U):
        """Re B per atom and triple (snap/compute.py:354-373)."""
        out = np.empty((len(U), len(self.terms)))
        for t, (iz, i1, i2, c) in enumerate(self.terms):
            out[:, t] = ((c * U[:, i1]) * U[:, i2] * np.conj(U[:, iz])).sum(axis=1).real
        return out

    def energy(self, U):
        return float(np.sum(self.bispectrum(U) @ self.beta)) if len(U) else 0.0

    @staticmethod
    def energy_from_y(U, Y):
        return float(np.sum(Y * np.conj(U)).real) / 3.0

    def compute_forces(self, Y, rows, cols, dr, n_total, chunk=4096):
        """F_i += Re sum Y_i conj(d(fc u)/d dr); F_k -= same (snap/compute.py:390-409)."""
        F = np.zeros((n_total, 3))
        for s in range(0, len(rows), chunk):
            sl = slice(s, s + chunk)
            d = dr[sl]
            r, a, b, fc, dfc, z0, r0 = pair_params(d, self.rc)
            da, db = pair_grads(d, r, self.rc, a, b, z0, r0)
            u, du = pair_levels(a, b, self.twojmax, da, db)
            wdu = fc[:, None, None] * du + (dfc[:, None] * d / r[:, None])[:, :, None] * u[:, None, :]
            t = np.einsum("pf,pdf->pd", Y[rows[sl]], np.conj(wdu)).real
            np.add.at(F, rows[sl], t)
            np.subtract.at(F, cols[sl], t)
        return F

    def evaluate(self, x, n_local, rows, cols):
        """Full single-rank pipeline: (E, U, Y, F over all rows incl. ghosts)."""
        rows, cols, dr = self.pairs_from_list(x, rows, cols)
        U = self.compute_u(n_local, rows, dr)
        E = self.energy(U)
        Y = self.compute_y(U)
        F = self.compute_forces(Y, rows, cols, dr, len(x))
        return E, U, Y, F


def snap_compute(sys, lists, oracle: SnapOracle):
    """SnapStyle.compute over all ranks + reverse comm (mdkk/driver/simulation.py:115-142)."""
    e = 0.0
    for rk, nl in zip(sys.ranks, lists):
        if nl.style != "full":
            raise SnapOracleError("descriptor pipeline requires a full-style neighbor list")
        E, _, _, F = oracle.evaluate(rk.x, rk.n_local, nl.rows, nl.cols)
        e += E
        rk.f[:] = F
    sys.reverse()
    return e, sys.gather_forces()
