"""Quantum indexing and Clebsch-Gordan coupling tables (host-side setup, uploaded once).

Mirror of mdkk/snap/indexing.py:24-68 and mdkk/snap/coupling.py:28-137:
doubled-integer angular momenta, flat (tj, p, q) index with tj slowest,
coupled triples (tj, tj1, tj2) with tj2 <= tj1 <= tj, exact-rational CG with a
single final rounding, and per-triple (iz, iu1, iu2, coeff) term lists.  The
device consumes an output-sorted product list for the half-block adjoint (the
Z-list form of mdkk/snap/compute.py:303-340) built by `zlist_entries`.
"""

from __future__ import annotations

import math
from fractions import Fraction
from functools import lru_cache

import numpy as np


class SnapIndexError(ValueError):
    pass


def twojmax_of(jmax) -> int:
    tj = float(2 * jmax)
    if tj < 0 or abs(tj - round(tj)) > 1e-12:
        raise SnapIndexError(f"2*jmax must be a non-negative integer, got jmax={jmax}")
    return int(round(tj))


class QuantumIndex:
    """Bijection (j, m, m') -> flat index, per-j contiguous (tj+1)^2 blocks (mdkk/snap/indexing.py:24-54)."""

    def __init__(self, jmax):
        self.jmax = float(jmax)
        self.twojmax = twojmax_of(jmax)
        sizes = [(t + 1) ** 2 for t in range(self.twojmax + 1)]
        self.block_offset = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.n_flat = int(self.block_offset[-1])

    def flat(self, tj: int, p: int, q: int) -> int:
        if not (0 <= tj <= self.twojmax):
            raise SnapIndexError(f"tj {tj} out of range [0, {self.twojmax}]")
        if not (0 <= p <= tj and 0 <= q <= tj):
            raise SnapIndexError(f"(p, q) = ({p}, {q}) out of block range for tj {tj}")
        return int(self.block_offset[tj] + p * (tj + 1) + q)

    def unflatten(self, idx: int) -> tuple[int, int, int]:
        """Inverse of flat (mdkk/snap/indexing.py:42-50)."""
        if not (0 <= idx < self.n_flat):
            raise SnapIndexError(f"flat index {idx} out of range [0, {self.n_flat})")
        tj = int(np.searchsorted(self.block_offset, idx, side="right")) - 1
        p, q = divmod(int(idx - self.block_offset[tj]), tj + 1)
        return tj, p, q

    def block(self, tj: int) -> slice:
        return slice(int(self.block_offset[tj]), int(self.block_offset[tj + 1]))

    def triples(self):
        """(tj, tj1, tj2): tj2 <= tj1 <= tj, triangle, even sum; tj slowest (mdkk/snap/indexing.py:56-68)."""
        return [(tj, tj1, tj2) for tj in range(self.twojmax + 1) for tj1 in range(tj + 1)
                for tj2 in range(tj1 + 1) if tj <= tj1 + tj2 and (tj1 + tj2 - tj) % 2 == 0]


def _hf(twice: int) -> int:
    if twice < 0 or twice % 2:
        raise SnapIndexError(f"factorial of non-integer or negative half-value {twice}/2")
    return math.factorial(twice // 2)


@lru_cache(maxsize=None)
def clebsch_gordan(tj1: int, tm1: int, tj2: int, tm2: int, tj: int, tm: int) -> float:
    """<j1 m1; j2 m2 | j m>, doubled args, Racah sum in exact rationals (mdkk/snap/coupling.py:28-66)."""
    if tm1 + tm2 != tm or not (abs(tj1 - tj2) <= tj <= tj1 + tj2) or (tj1 + tj2 - tj) % 2:
        return 0.0
    if abs(tm1) > tj1 or abs(tm2) > tj2 or abs(tm) > tj:
        return 0.0
    if (tj1 + tm1) % 2 or (tj2 + tm2) % 2 or (tj + tm) % 2:
        return 0.0
    pref = Fraction((tj + 1) * _hf(tj1 + tj2 - tj) * _hf(tj1 - tj2 + tj) * _hf(tj2 - tj1 + tj)
                    * _hf(tj1 + tm1) * _hf(tj1 - tm1) * _hf(tj2 + tm2) * _hf(tj2 - tm2)
                    * _hf(tj + tm) * _hf(tj - tm), _hf(tj1 + tj2 + tj + 2))
    acc = Fraction(0)
    for k in range(max(0, (tj2 - tj - tm1) // 2, (tj1 - tj + tm2) // 2),
                   min((tj1 + tj2 - tj) // 2, (tj1 - tm1) // 2, (tj2 + tm2) // 2) + 1):
        den = (math.factorial(k) * _hf(tj1 + tj2 - tj - 2 * k) * _hf(tj1 - tm1 - 2 * k)
               * _hf(tj2 + tm2 - 2 * k) * _hf(tj - tj2 + tm1 + 2 * k) * _hf(tj - tj1 - tm2 + 2 * k))
        acc += Fraction((-1) ** k, den)
    if acc == 0:
        return 0.0
    return math.copysign(math.sqrt(float(acc * acc * pref)), float(acc))


class TripleTerms:
    """Flattened contraction terms of one (tj, tj1, tj2) triple (mdkk/snap/coupling.py:69-91).

    Term k couples U[iu1[k]] * U[iu2[k]] into slot iz[k] of the tj block with
    weight coeff[k] = C(m1, m2) C(m1', m2'); `order_*` / `starts_*` /
    `unique_*` group the terms by iz, iu1 and iu2 (stable sorts, reduceat
    boundaries), as in the reference.  Host-side setup data: the device kernels
    consume the Z-list built from these terms (`device_product_list`).
    Iterating yields (iz, iu1, iu2, coeff).
    """

    def __init__(self, tj: int, tj1: int, tj2: int, iz, iu1, iu2, coeff):
        self.tj, self.tj1, self.tj2 = int(tj), int(tj1), int(tj2)
        self.iz = np.asarray(iz, dtype=np.int64)
        self.iu1 = np.asarray(iu1, dtype=np.int64)
        self.iu2 = np.asarray(iu2, dtype=np.int64)
        self.coeff = np.asarray(coeff, dtype=np.float64)
        self.n_terms = len(self.coeff)
        for key in ("iz", "iu1", "iu2"):
            idx = getattr(self, key)
            order = np.argsort(idx, kind="stable")
            srt = idx[order]
            firsts = np.flatnonzero(np.concatenate([[True], srt[1:] != srt[:-1]])) if len(srt) else \
                np.zeros(0, np.int64)
            setattr(self, f"order_{key}", order)
            setattr(self, f"starts_{key}", firsts)
            setattr(self, f"unique_{key}", srt[firsts])

    def __iter__(self):
        return iter((self.iz, self.iu1, self.iu2, self.coeff))

    def __getitem__(self, k):
        return (self.iz, self.iu1, self.iu2, self.coeff)[k]

    def __len__(self):
        return 4


class CouplingTables:
    """CG blocks and per-triple `TripleTerms` for every coupled triple (mdkk/snap/coupling.py:94-133)."""

    def __init__(self, jmax):
        self.index = QuantumIndex(jmax)
        self.triples = self.index.triples()
        off = self.index.block_offset
        self.cg = {}      # (tj1, tj2, tj) -> cg[p1, p2]
        self.terms = []   # TripleTerms, parallel to self.triples
        for (tj, tj1, tj2) in self.triples:
            cg = np.zeros((tj1 + 1, tj2 + 1))
            for p1 in range(tj1 + 1):
                for p2 in range(tj2 + 1):
                    tm = (2 * p1 - tj1) + (2 * p2 - tj2)
                    if abs(tm) <= tj:
                        cg[p1, p2] = clebsch_gordan(tj1, 2 * p1 - tj1, tj2, 2 * p2 - tj2, tj, tm)
            sh = (tj1 + tj2 - tj) // 2
            p1, p2, q1, q2 = (v.ravel() for v in np.meshgrid(np.arange(tj1 + 1), np.arange(tj2 + 1),
                                                             np.arange(tj1 + 1), np.arange(tj2 + 1),
                                                             indexing="ij"))
            p, q = p1 + p2 - sh, q1 + q2 - sh
            c = cg[p1, p2] * cg[q1, q2]
            k = (p >= 0) & (p <= tj) & (q >= 0) & (q <= tj) & (c != 0.0)
            self.cg[(tj1, tj2, tj)] = cg
            self.terms.append(TripleTerms(tj, tj1, tj2, off[tj] + p[k] * (tj + 1) + q[k],
                                          off[tj1] + p1[k] * (tj1 + 1) + q1[k],
                                          off[tj2] + p2[k] * (tj2 + 1) + q2[k], c[k]))

    @property
    def n_terms(self) -> int:
        return sum(len(t[3]) for t in self.terms)


def make_coupling_tables(jmax) -> CouplingTables:
    return CouplingTables(jmax)


def adjoint_contributions(tables: CouplingTables, beta):
    """Output-sorted list for Y[f] = sum coef * op(U[g]) * U[h] (mdkk/snap/compute.py:303-340).

    Each term of triple t contributes to three slots:
      Y[iz]  += b c U[iu1] U[iu2]        -> (f=iz,  g=iu1, h=iu2, conj=0)
      Y[iu1] += b c conj(U[iu2]) U[iz]   -> (f=iu1, g=iu2, h=iz,  conj=1)
      Y[iu2] += b c conj(U[iu1]) U[iz]   -> (f=iu2, g=iu1, h=iz,  conj=1)
    identical (f, g, h, conj) keys are merged (U[g]U[h] commutes, so conj=0
    keys use g <= h).  Returns f_start[n_flat+1], g, h, conj (int32) and coef (f64).
    """
    beta = np.asarray(beta, dtype=np.float64)
    acc: dict = {}
    for bt, (iz, i1, i2, c) in zip(beta, tables.terms):
        if bt == 0.0:
            continue
        bc = bt * c
        for z, a, b, v in zip(iz.tolist(), i1.tolist(), i2.tolist(), bc.tolist()):
            for key in ((z, min(a, b), max(a, b), 0), (a, b, z, 1), (b, a, z, 1)):
                acc[key] = acc.get(key, 0.0) + v
    keys = sorted(acc)
    n_flat = tables.index.n_flat
    f = np.array([k[0] for k in keys], dtype=np.int64)
    f_start = np.searchsorted(f, np.arange(n_flat + 1)).astype(np.int32)
    g = np.array([k[1] for k in keys], dtype=np.int32)
    h = np.array([k[2] for k in keys], dtype=np.int32)
    cj = np.array([k[3] for k in keys], dtype=np.int32)
    coef = np.array([acc[k] for k in keys], dtype=np.float64)
    return f_start, g, h, cj, coef


def read_coeff_file(path):
    """First token jmax, then one beta per triple, '#' comments (mdkk/snap/compute.py:439-464)."""
    from .compute import SnapError
    tokens = []
    with open(path) as fh:
        for line in fh:
            tokens.extend(line.split("#", 1)[0].split())
    if not tokens:
        raise SnapError(f"coefficient file {path} is empty")
    try:
        values = [float(t) for t in tokens]
    except ValueError as exc:
        raise SnapError(f"coefficient file {path}: {exc}") from None
    jmax = values[0]
    need = len(QuantumIndex(jmax).triples())
    beta = np.asarray(values[1:], dtype=np.float64)
    if len(beta) != need:
        raise SnapError(f"coefficient file {path}: expected {need} beta values for jmax {jmax}, got {len(beta)}")
    return jmax, beta


def half_block_outputs(twojmax: int):
    """Flat indices with 2p < tj, or 2p == tj and 2q <= tj: one of each mirror pair.

    Every U/Y block obeys X[tj-p][tj-q] = (-1)^(p+q) conj(X[p][q]) (SURVEY §7,
    verified on mdkk's U and full adjoint Y), so the other half follows.
    """
    off = QuantumIndex(twojmax / 2.0).block_offset
    keep, fmap = [], []
    for tj in range(twojmax + 1):
        for p in range(tj + 1):
            for q in range(tj + 1):
                if 2 * p < tj or (2 * p == tj and 2 * q <= tj):
                    keep.append(int(off[tj] + p * (tj + 1) + q))
    pos = {f: k for k, f in enumerate(keep)}
    for tj in range(twojmax + 1):
        for p in range(tj + 1):
            for q in range(tj + 1):
                f = int(off[tj] + p * (tj + 1) + q)
                if f in pos:
                    fmap.append(pos[f])
                else:
                    m = int(off[tj] + (tj - p) * (tj + 1) + (tj - q))
                    fmap.append(pos[m] | (1 << 16) | ((((p + q) & 1)) << 17))
    return np.array(keep, dtype=np.int32), np.array(fmap, dtype=np.int32)


def _half_index(twojmax: int):
    """(tj, p, q) -> (half-set index, mirrored?, odd sign?) with X[m] = (-1)^(p+q) conj(X[half])."""
    off, hidx = 0, {}
    for tj in range(twojmax + 1):
        hs = (tj + 1) * (tj + 1) // 2 if tj & 1 else (tj // 2) * (tj + 1) + tj // 2 + 1
        for h in range(hs):
            hidx[(tj, h // (tj + 1), h % (tj + 1))] = off + h
        off += hs
    out = {}
    for tj in range(twojmax + 1):
        for p in range(tj + 1):
            for q in range(tj + 1):
                if (tj, p, q) in hidx:
                    out[(tj, p, q)] = (hidx[(tj, p, q)], 0, 0)
                else:
                    out[(tj, p, q)] = (hidx[(tj, tj - p, tj - q)], 1, (p + q) & 1)
    return out, off


def zlist_entries(tables: CouplingTables, beta):
    """Half-block Y as a list of U*U products (the Z-list form of the adjoint).

    Y_tj = sum over every coupled (tj1 >= tj2, tj) of beta' * Z_{tj1,tj2->tj}
    with Z[P,Q] = sum cg[p1,p2] cg[q1,q2] U_tj1[p1,q1] U_tj2[p2,q2] and beta'
    the triple's beta scaled by the multiplicity / dimension ratio of the
    coupling symmetry B_{j1 j2 j} = (j+1)/(j1+1) B_{j j2 j1} (for tj >= tj1:
    x2 or x3 when indices coincide; otherwise (tj1+1)/(tj+1)).  This equals
    the reference's three-slot adjoint (mdkk/snap/compute.py:303-340)
    element-wise (checked against it to ~1e-15 relative in tests), with U*U
    products only.  Operands outside the half set are mirrored,
    U[m] = (-1)^(p+q) conj(U[half]); the sign folds into the coefficient.

    Returns (f, g, h, conj_g, conj_h, coef), sorted by output f (half index),
    with identical keys merged and every output present at least once.
    """
    beta = np.asarray(beta, dtype=np.float64)
    twojmax = tables.index.twojmax
    hmap, n_half = _half_index(twojmax)
    bidx = {t: i for i, t in enumerate(tables.triples)}
    acc: dict = {}
    for tj1 in range(twojmax + 1):
        for tj2 in range(tj1 + 1):
            for tj in range(tj1 - tj2, min(twojmax, tj1 + tj2) + 1, 2):
                if tj >= tj1:
                    b = beta[bidx[(tj, tj1, tj2)]]
                    fac = (3.0 if tj2 == tj else 2.0) if tj1 == tj else 1.0
                elif tj >= tj2:
                    b = beta[bidx[(tj1, tj, tj2)]]
                    fac = (2.0 if tj2 == tj else 1.0) * (tj1 + 1) / (tj + 1)
                else:
                    b = beta[bidx[(tj1, tj2, tj)]]
                    fac = (tj1 + 1) / (tj + 1)
                if b == 0.0:
                    continue
                bf = b * fac
                sh = (tj1 + tj2 - tj) // 2
                cg = np.zeros((tj1 + 1, tj2 + 1))
                for p1 in range(tj1 + 1):
                    for p2 in range(tj2 + 1):
                        tm = (2 * p1 - tj1) + (2 * p2 - tj2)
                        if abs(tm) <= tj:
                            cg[p1, p2] = clebsch_gordan(tj1, 2 * p1 - tj1, tj2, 2 * p2 - tj2, tj, tm)
                for (t_, P, Q), (fo, mir, _) in hmap.items():
                    if t_ != tj or mir:
                        continue
                    for p1 in range(tj1 + 1):
                        p2 = P - p1 + sh
                        if p2 < 0 or p2 > tj2 or cg[p1, p2] == 0.0:
                            continue
                        for q1 in range(tj1 + 1):
                            q2 = Q - q1 + sh
                            if q2 < 0 or q2 > tj2 or cg[q1, q2] == 0.0:
                                continue
                            g, cgj, sg = hmap[(tj1, p1, q1)]
                            h, chj, shh = hmap[(tj2, p2, q2)]
                            c = bf * cg[p1, p2] * cg[q1, q2] * (-1.0 if sg ^ shh else 1.0)
                            a, d = (g, cgj), (h, chj)
                            if d < a:
                                a, d = d, a
                            key = (fo, a[0], d[0], a[1], d[1])
                            acc[key] = acc.get(key, 0.0) + c
    present = {k[0] for k in acc}
    for fo in range(n_half):
        if fo not in present:
            acc[(fo, 0, 0, 0, 0)] = 0.0
    keys = sorted(acc)
    arr = np.array(keys, dtype=np.int64).reshape(-1, 5)
    coef = np.array([acc[k] for k in keys], dtype=np.float64)
    return arr[:, 0], arr[:, 1], arr[:, 2], arr[:, 3], arr[:, 4], coef


def zlist_apply(U: np.ndarray, twojmax: int, entries) -> np.ndarray:
    """Host emulation of the device yi on full U rows -> full Y rows (test helper for the table)."""
    f, g, h, cg_, ch_, coef = entries
    hmap, n_half = _half_index(twojmax)
    off = QuantumIndex(twojmax / 2.0).block_offset
    half_flat = np.zeros(n_half, dtype=np.int64)
    for (tj, p, q), (k, mir, _) in hmap.items():
        if not mir:
            half_flat[k] = off[tj] + p * (tj + 1) + q
    Uh = U[:, half_flat]
    ug = np.where(cg_ == 1, np.conj(Uh[:, g]), Uh[:, g])
    uh = np.where(ch_ == 1, np.conj(Uh[:, h]), Uh[:, h])
    Yh = np.zeros((len(U), n_half), complex)
    np.add.at(Yh.T, f, (coef * ug * uh).T)
    Y = np.zeros_like(U)
    for (tj, p, q), (k, mir, odd) in hmap.items():
        v = Yh[:, k]
        if mir:
            v = np.conj(v) * (-1.0 if odd else 1.0)
        Y[:, off[tj] + p * (tj + 1) + q] = v
    return Y


def _reuse_order(f, g, h, cg_, ch_):
    """Order the products of each output into runs sharing their first operand.

    The yi kernel keeps the last U[g] in registers, so a product whose g equals
    the previous one costs one shared-memory load instead of two.  Greedy cover
    per output: repeatedly take the operand that appears in most remaining
    products, orient those products so it is g (U[g] U[h] commutes; each
    operand keeps its own conj flag), emit them sorted by h.
    """
    order, swap = [], np.zeros(len(f), dtype=bool)
    starts = np.flatnonzero(np.r_[True, f[1:] != f[:-1]])
    ends = np.r_[starts[1:], len(f)]
    for a, b in zip(starts, ends):
        remaining = list(range(a, b))
        while remaining:
            cnt: dict = {}
            for k in remaining:
                cnt[g[k]] = cnt.get(g[k], 0) + 1
                if h[k] != g[k]:
                    cnt[h[k]] = cnt.get(h[k], 0) + 1
            best = max(sorted(cnt), key=lambda o: cnt[o])
            take = [k for k in remaining if g[k] == best or h[k] == best]
            for k in take:
                swap[k] = g[k] != best
            take.sort(key=lambda k: (g[k] if swap[k] else h[k]))
            order.extend(take)
            remaining = [k for k in remaining if not (g[k] == best or h[k] == best)]
    order = np.asarray(order, dtype=np.int64)
    g2, h2 = np.where(swap, h, g), np.where(swap, g, h)
    c2g, c2h = np.where(swap, ch_, cg_), np.where(swap, cg_, ch_)
    return order, g2, h2, c2g, c2h


def device_product_list(tables: CouplingTables, beta):
    """Packed (coef, code, n_half, fmap) for mdkk_snap_create (include/mdkk_b200.h)."""
    f, g, h, cg_, ch_, coef = zlist_entries(tables, beta)
    order, g, h, cg_, ch_ = _reuse_order(f, g, h, cg_, ch_)
    f, g, h, cg_, ch_, coef = f[order], g[order], h[order], cg_[order], ch_[order], coef[order]
    hmap, n_half = _half_index(tables.index.twojmax)
    center = np.zeros(n_half, dtype=np.int64)
    for (tj, p, q), (k, mir, _) in hmap.items():
        if not mir and (tj - p, tj - q) == (p, q):
            center[k] = 1
    last = np.ones(len(f), dtype=np.int64)
    last[:-1] = f[1:] != f[:-1]
    code = g | (h << 8) | (f << 16) | (cg_ << 24) | (ch_ << 25) | (last << 26) | (center[f] << 27)
    _, fmap = half_block_outputs(tables.index.twojmax)
    return (np.ascontiguousarray(coef, dtype=np.float64), np.ascontiguousarray(code, dtype=np.int32), n_half,
            np.ascontiguousarray(fmap, dtype=np.int32))


def bi_entries(tables: CouplingTables, n_warps: int):
    """Descriptor terms for mdkk_snap_bi (include/mdkk_b200.h), per triple in storage order.

    B_t = sum c U[iu1] U[iu2] conj(U[iz]) (mdkk/snap/compute.py:354-373) with
    every operand on the half set: U[m] = s conj(U[half]); signs fold into c.
    Returns (coef, code, tri, chunk) with chunk[w] the first term of warp w
    (triple-aligned, balanced on term counts).
    """
    hmap, _ = _half_index(tables.index.twojmax)
    off = tables.index.block_offset
    inv = {}
    for (tj, p, q), v in hmap.items():
        inv[int(off[tj] + p * (tj + 1) + q)] = v
    coef, code, tri = [], [], []
    for t, (iz, i1, i2, c) in enumerate(tables.terms):
        n = len(c)
        for k in range(n):
            g, cg_, sg = inv[int(i1[k])]
            h, ch_, sh = inv[int(i2[k])]
            z, mz, sz = inv[int(iz[k])]
            cz = 0 if mz else 1          # conj(U[z]) = s U[half] when z is mirrored
            sign = -1.0 if (sg ^ sh ^ sz) else 1.0
            coef.append(sign * float(c[k]))
            code.append(g | (h << 8) | (z << 16) | (cg_ << 24) | (ch_ << 25) | (cz << 26) | ((k == n - 1) << 27))
            tri.append(t)
        if n == 0:   # keep every triple's output written
            coef.append(0.0)
            code.append(1 << 27)
            tri.append(t)
    coef = np.asarray(coef, dtype=np.float64)
    code = np.asarray(code, dtype=np.int64).astype(np.int32)
    tri = np.asarray(tri, dtype=np.int32)
    ends = np.flatnonzero((code >> 27) & 1) + 1
    chunk = [0]
    for w in range(1, n_warps):
        target = len(coef) * w / n_warps
        k = int(np.searchsorted(ends, target))
        e = int(ends[min(k, len(ends) - 1)])
        if k > 0 and abs(int(ends[k - 1]) - target) < abs(e - target):
            e = int(ends[k - 1])
        chunk.append(max(chunk[-1], e))
    chunk.append(len(coef))
    return coef, code, tri, np.asarray(chunk, dtype=np.int32)
