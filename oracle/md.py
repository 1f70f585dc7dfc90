"""Numpy restatement of the reference LJ hot path — TEST INFRASTRUCTURE ONLY.

Restates (does not import) the reference `mdkk` algorithms:

* lattices / velocities      — mdkk/driver/simulation.py:156-194
* box, bricks, ghosts, comm  — mdkk/domain.py:22-354
* cell-list neighbor builds  — mdkk/neighbor.py:83-231
* truncated LJ pair engine   — mdkk/pair_lj.py:55-179
* velocity-Verlet NVE loop   — mdkk/driver/simulation.py:407-481

Used by tests/ (parity checker), __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never imported by the product package.
"""

from __future__ import annotations

import itertools

import numpy as np


class OracleError(RuntimeError):
    pass


# ----------------------------------------------------------------- lattices
def lattice(style: str, rho: float, cells) -> tuple[np.ndarray, np.ndarray]:
    """Replicated unit-cell sites (cells x basis, meshgrid 'ij' order) and box lengths.

    fcc / sc follow mdkk/driver/simulation.py:156-178 (a = (4/rho)^(1/3) for
    fcc, (1/rho)^(1/3) for sc).  ``style="bcc"`` is the SURVEY §8(d) C4/C5
    generator (mdkk has none): ``rho`` is then the lattice constant ``a``
    (tungsten a = 3.1803), basis (0,0,0), (1/2,1/2,1/2).
    """
    if style == "fcc":
        a = (4.0 / rho) ** (1.0 / 3.0)
        basis = np.array([[0, 0, 0], [.5, .5, 0], [.5, 0, .5], [0, .5, .5]], dtype=np.float64)
    elif style == "sc":
        a = (1.0 / rho) ** (1.0 / 3.0)
        basis = np.zeros((1, 3))
    elif style == "bcc":
        a = float(rho)
        basis = np.array([[0, 0, 0], [.5, .5, .5]], dtype=np.float64)
    else:
        raise OracleError(f"unknown lattice {style!r}")
    nx, ny, nz = (int(c) for c in cells)
    grid = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"),
                    axis=-1).reshape(-1, 3).astype(np.float64)
    pos = (grid[:, None, :] + basis[None]).reshape(-1, 3) * a
    return pos, np.array([a * nx, a * ny, a * nz])


def seeded_velocities(n: int, temperature: float, mass: float, seed: int) -> np.ndarray:
    """Gaussian, zero momentum, exact-T rescale (mdkk/driver/simulation.py:181-194)."""
    if temperature == 0.0 or n == 0:
        return np.zeros((n, 3))
    v = np.random.default_rng(seed).normal(0.0, np.sqrt(temperature / mass), (n, 3))
    v -= v.mean(axis=0)
    t_now = mass * float(np.sum(v * v)) / (3.0 * n)
    if t_now > 0:
        v *= np.sqrt(temperature / t_now)
    return v


def jittered(pos: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """Lattice + N(0, sigma) displacement from default_rng(seed) (SURVEY §8(c) KATs)."""
    return pos + np.random.default_rng(seed).normal(0.0, sigma, pos.shape)


def random_config(n: int, rho: float, seed: int, min_sep: float = 0.85):
    """Jittered cubic-lattice configuration (mdkk tests/conftest.py:16-31)."""
    rng = np.random.default_rng(seed)
    cells = int(np.ceil(n ** (1.0 / 3.0)))
    a = (1.0 / rho) ** (1.0 / 3.0)
    lo = np.stack(np.meshgrid(*[np.arange(cells)] * 3, indexing="ij"), axis=-1).reshape(-1, 3)
    order = rng.permutation(len(lo))[:n]
    jit = rng.uniform(-0.5, 0.5, (n, 3)) * (a - min_sep)
    return (lo[order] + 0.5) * a + jit, np.array([a * cells] * 3)


# -------------------------------------------------------------------- domain
def wrap(pos: np.ndarray, lengths: np.ndarray) -> np.ndarray:
    """Wrap into [0, L) (mdkk/domain.py:56-63)."""
    pos = np.array(pos, dtype=np.float64, copy=True)
    return pos - lengths * np.floor(pos / lengths)


def min_surface_grid(lengths: np.ndarray, n: int) -> tuple[int, int, int]:
    """Brick grid with minimal surface, ties -> split lower axes (mdkk/domain.py:98-123)."""
    best = None
    for gx in range(1, n + 1):
        if n % gx:
            continue
        for gy in range(1, n // gx + 1):
            if (n // gx) % gy:
                continue
            gz = n // gx // gy
            e = lengths / np.array([gx, gy, gz])
            key = (2.0 * (e[0] * e[1] + e[0] * e[2] + e[1] * e[2]), (-gx, -gy, -gz))
            if best is None or key < best[0]:
                best = (key, (gx, gy, gz))
    return best[1]


def brick_bounds(lengths, grid):
    """Per-rank [lo, hi) bricks, rank = (cx*gy + cy)*gz + cz (mdkk/domain.py:69-87)."""
    gx, gy, gz = grid
    n = gx * gy * gz
    lo, hi = np.zeros((n, 3)), np.zeros((n, 3))
    for r in range(n):
        c = (r // (gy * gz), (r // gz) % gy, r % gz)
        for d in range(3):
            lo[r, d] = lengths[d] * c[d] / grid[d]
            hi[r, d] = lengths[d] * (c[d] + 1) / grid[d]
    return lo, hi


def rank_of(pos, lengths, grid) -> np.ndarray:
    """Owning rank of wrapped positions (mdkk/domain.py:89-95)."""
    g = np.array(grid)
    c = np.clip(np.floor(pos / lengths * g.astype(np.float64)).astype(np.int64), 0, g - 1)
    return (c[:, 0] * g[1] + c[:, 1]) * g[2] + c[:, 2]


class Rank:
    """One logical rank's rows: n_local owned + ghosts (mdkk/domain.py:126-193)."""

    def __init__(self, rank, x, v, gid):
        self.rank = int(rank)
        self.n_local = len(x)
        self.x = np.array(x, dtype=np.float64).reshape(-1, 3)
        self.v = np.array(v, dtype=np.float64).reshape(-1, 3)
        self.f = np.zeros_like(self.x)
        self.gid = np.asarray(gid, dtype=np.int64).copy()
        self.owner_rank = np.full(self.n_local, self.rank, dtype=np.int32)
        self.owner_index = np.arange(self.n_local, dtype=np.int32)
        self.shift = np.zeros((self.n_local, 3))

    @property
    def n_total(self):
        return len(self.x)

    @property
    def n_ghost(self):
        return self.n_total - self.n_local


class Ranked:
    """All logical ranks + ghost plan (RankedSystem, mdkk/domain.py:210-354)."""

    def __init__(self, lengths, n_ranks, positions, velocities, gids=None):
        self.lengths = np.asarray(lengths, dtype=np.float64)
        self.grid = min_surface_grid(self.lengths, n_ranks)
        self.lo, self.hi = brick_bounds(self.lengths, self.grid)
        pos = wrap(np.asarray(positions, dtype=np.float64), self.lengths)
        vel = np.asarray(velocities, dtype=np.float64)
        gids = np.arange(len(pos), dtype=np.int64) if gids is None else np.asarray(gids)
        self._assign(pos, vel, gids)
        self.plan = []

    def _assign(self, pos, vel, gids):
        owner = rank_of(pos, self.lengths, self.grid)
        self.ranks = []
        for r in range(len(self.lo)):
            sel = np.flatnonzero(owner == r)
            self.ranks.append(Rank(r, pos[sel], vel[sel], gids[sel]))

    @property
    def n_ranks(self):
        return len(self.ranks)

    def exchange_ghosts(self, halo):
        """27-shift halo selection, src-major then shift order (mdkk/domain.py:246-293)."""
        if halo > 0.5 * self.lengths.min():
            raise OracleError("halo exceeds half the shortest box length")
        shifts = [np.array(s, dtype=np.float64) * self.lengths
                  for s in itertools.product((-1, 0, 1), repeat=3)]
        owned = [r.x[: r.n_local].copy() for r in self.ranks]
        self.plan = []
        for dst in self.ranks:
            lo, hi = self.lo[dst.rank] - halo, self.hi[dst.rank] + halo
            xs, ids, orank, oidx, sh = [], [], [], [], []
            cursor = dst.n_local
            for src in self.ranks:
                for s in shifts:
                    if src.rank == dst.rank and not s.any():
                        continue
                    moved = owned[src.rank] + s
                    idx = np.flatnonzero(np.all((moved >= lo) & (moved < hi), axis=1))
                    if not len(idx):
                        continue
                    self.plan.append((src.rank, dst.rank, idx, s, cursor))
                    cursor += len(idx)
                    xs.append(moved[idx])
                    ids.append(src.gid[idx])
                    orank.append(np.full(len(idx), src.rank, dtype=np.int32))
                    oidx.append(idx.astype(np.int32))
                    sh.append(np.broadcast_to(s, (len(idx), 3)))
            nl = dst.n_local
            cat = (lambda a, shape, dt: np.concatenate(a).astype(dt) if a
                   else np.zeros(shape, dtype=dt))
            dst.x = np.concatenate([dst.x[:nl], cat(xs, (0, 3), np.float64)])
            dst.f = np.zeros_like(dst.x)
            dst.gid = np.concatenate([dst.gid[:nl], cat(ids, (0,), np.int64)])
            dst.owner_rank = np.concatenate([dst.owner_rank[:nl], cat(orank, (0,), np.int32)])
            dst.owner_index = np.concatenate([dst.owner_index[:nl], cat(oidx, (0,), np.int32)])
            dst.shift = np.concatenate([dst.shift[:nl], cat(sh, (0, 3), np.float64)])

    def forward(self):
        """ghost x = owner x + shift (mdkk/domain.py:295-305)."""
        bufs = [self.ranks[s].x[idx] + sh for (s, _, idx, sh, _) in self.plan]
        for (_, d, idx, _, start), b in zip(self.plan, bufs):
            self.ranks[d].x[start:start + len(idx)] = b

    def reverse(self):
        """Fold ghost forces onto owners, zero ghost rows (mdkk/domain.py:307-322)."""
        bufs = [self.ranks[d].f[start:start + len(idx)].copy()
                for (_, d, idx, _, start) in self.plan]
        for (s, _, idx, _, _), b in zip(self.plan, bufs):
            np.add.at(self.ranks[s].f, idx, b)
        for r in self.ranks:
            r.f[r.n_local:] = 0.0

    def gather(self):
        """Owned (x, v, gid) of all ranks in gid order (mdkk/domain.py:336-342)."""
        x = np.concatenate([r.x[: r.n_local] for r in self.ranks])
        v = np.concatenate([r.v for r in self.ranks])
        g = np.concatenate([r.gid[: r.n_local] for r in self.ranks])
        o = np.argsort(g, kind="stable")
        return x[o], v[o], g[o]

    def gather_forces(self):
        """Owned forces in gid order (mdkk/domain.py:344-348)."""
        f = np.concatenate([r.f[: r.n_local] for r in self.ranks])
        g = np.concatenate([r.gid[: r.n_local] for r in self.ranks])
        return f[np.argsort(g, kind="stable")]

    def migrate(self, halo):
        """Gather, wrap, reassign, zero forces, rebuild ghosts (mdkk/domain.py:324-334)."""
        x, v, g = self.gather()
        self._assign(wrap(x, self.lengths), v, g)
        self.exchange_ghosts(halo)


# ------------------------------------------------------------------ neighbor
def candidate_pairs(x: np.ndarray, n_local: int, bc: float):
    """Directed (owned row, partner) pairs with r^2 < bc^2 via bbox cell bins.

    Restates mdkk/neighbor.py:83-131: bins of width span/floor(span/bc), a
    27-cell stencil, self excluded by index, strict r^2 < bc^2 evaluated with
    the same `einsum("ij,ij->i")` reduction the reference uses (:126).
    """
    if len(x) == 0 or n_local == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    lo = x.min(axis=0)
    span = np.maximum(x.max(axis=0) - lo, 1e-12)
    nb = np.maximum(1, np.floor(span / bc).astype(np.int64))
    cell = np.minimum((np.maximum(x - lo, 0.0) / (span / nb)).astype(np.int64), nb - 1)
    cid = (cell[:, 0] * nb[1] + cell[:, 1]) * nb[2] + cell[:, 2]
    order = np.argsort(cid, kind="stable")
    cnt = np.bincount(cid, minlength=int(nb.prod()))
    start = np.concatenate([[0], np.cumsum(cnt)])
    out_r, out_c = [], []
    rows0 = np.arange(n_local, dtype=np.int64)
    for off in itertools.product((-1, 0, 1), repeat=3):
        nc = cell[:n_local] + np.asarray(off)
        ok = np.all((nc >= 0) & (nc < nb), axis=1)
        ncid = ((nc[:, 0] * nb[1] + nc[:, 1]) * nb[2] + nc[:, 2])[ok]
        r = rows0[ok]
        k = cnt[ncid]
        r, ncid, k = r[k > 0], ncid[k > 0], k[k > 0]
        if not len(r):
            continue
        rows = np.repeat(r, k)
        first = np.repeat(start[ncid], k)
        within = np.arange(len(rows)) - np.repeat(np.cumsum(k) - k, k)
        cols = order[first + within]
        keep = rows != cols
        rows, cols = rows[keep], cols[keep]
        dr = x[cols] - x[rows]
        keep = np.einsum("ij,ij->i", dr, dr) < bc * bc
        out_r.append(rows[keep])
        out_c.append(cols[keep])
    if not out_r:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(out_r), np.concatenate(out_c)


def apply_style(rk: Rank, rows, cols, style: str, newton: bool):
    """Entry selection, energy weight, partner-write flag (mdkk/neighbor.py:134-179)."""
    if style == "full":
        return rows, cols, np.full(len(rows), 0.5), np.zeros(len(rows), bool)
    if style != "half":
        raise OracleError(f"unknown list style {style!r}")
    local = cols < rk.n_local
    keep = np.zeros(len(rows), bool)
    keep[local] = rk.gid[rows[local]] < rk.gid[cols[local]]
    g = ~local
    if newton:
        orank = rk.owner_rank[cols[g]]
        sub = orank > rk.rank
        same = orank == rk.rank
        xi, xj = rk.x[rows[g]], rk.x[cols[g]]
        tie = ((xi[:, 2] < xj[:, 2])
               | ((xi[:, 2] == xj[:, 2]) & (xi[:, 1] < xj[:, 1]))
               | ((xi[:, 2] == xj[:, 2]) & (xi[:, 1] == xj[:, 1]) & (xi[:, 0] < xj[:, 0])))
        sub = np.where(same, tie, sub)
        keep[g] = sub
        rows, cols = rows[keep], cols[keep]
        return rows, cols, np.ones(len(rows)), np.ones(len(rows), bool)
    keep[g] = True
    rows, cols = rows[keep], cols[keep]
    local = cols < rk.n_local
    return rows, cols, np.where(local, 1.0, 0.5), local.copy()


class NList:
    """Directed entries + padded table (NeighborList, mdkk/neighbor.py:38-80)."""

    def __init__(self, rk, style, newton, cutoff, skin):
        self.rk, self.style, self.newton = rk, style, bool(newton)
        self.cutoff, self.skin = float(cutoff), float(skin)
        self.ref_x = rk.x[: rk.n_local].copy()

    def max_displacement(self):
        if self.rk.n_local == 0:
            return 0.0
        d = self.rk.x[: self.rk.n_local] - self.ref_x
        return float(np.sqrt(np.einsum("ij,ij->i", d, d).max()))

    def needs_rebuild(self):
        return self.max_displacement() > 0.5 * self.skin


def build(rk: Rank, lengths, cutoff, skin, style="full", newton=True, capacity=16) -> NList:
    """One rank's list: candidates, style, canonical order, table (mdkk/neighbor.py:182-219)."""
    bc = cutoff + skin
    if bc > 0.5 * np.min(lengths):
        raise OracleError("cutoff+skin exceeds half the shortest periodic box length")
    rows, cols = candidate_pairs(rk.x, rk.n_local, bc)
    rows, cols, w, wj = apply_style(rk, rows, cols, style, newton)
    if len(rows):
        pc = rk.x[cols]
        p = np.lexsort((pc[:, 0], pc[:, 1], pc[:, 2], rk.gid[cols], rows))
        rows, cols, w, wj = rows[p], cols[p], w[p], wj[p]
    nl = NList(rk, style, newton, cutoff, skin)
    nl.rows, nl.cols, nl.weight, nl.write_j = rows, cols, w, wj
    nl.counts = np.bincount(rows, minlength=rk.n_local).astype(np.int32)
    need = int(nl.counts.max()) if rk.n_local else 0
    cap = max(capacity, 1)
    while cap < need:
        cap = int(np.ceil(cap * 1.5))
    nl.cap = cap
    tbl = np.full((max(rk.n_local, 1), cap), -1, dtype=np.int32)
    if len(rows):
        first = np.concatenate([[0], np.cumsum(nl.counts)])[:-1]
        tbl[rows, np.arange(len(rows)) - first[rows]] = cols
    nl.table = tbl
    return nl


def build_all(sys: Ranked, cutoff, skin, style="full", newton=True, capacity=16):
    """Ghost exchange then per-rank builds (mdkk/neighbor.py:222-227)."""
    sys.exchange_ghosts(cutoff + skin)
    return [build(r, sys.lengths, cutoff, skin, style, newton, capacity) for r in sys.ranks]


def pair_set_brute(pos, lengths, cutoff) -> set:
    """O(N^2) min-image unordered pair set (mdkk tests/conftest.py:67-77)."""
    out = set()
    for i in range(len(pos) - 1):
        dr = pos[i + 1:] - pos[i]
        dr -= lengths * np.round(dr / lengths)
        for j in np.flatnonzero((dr * dr).sum(axis=1) < cutoff * cutoff):
            out.add((i, i + 1 + int(j)))
    return out


# ------------------------------------------------------------------------ LJ
def lj_pair(r2, eps, sigma):
    """e = 4eps(s12-s6), fp = 24eps(2 s12 - s6)/r^2 (mdkk/pair_lj.py:81-91)."""
    if r2.size and r2.min() <= 0.0:
        raise OracleError("coincident atoms (r = 0)")
    s2 = (sigma * sigma) / r2
    s6 = s2 * s2 * s2
    s12 = s6 * s6
    return 4.0 * eps * (s12 - s6), 24.0 * eps * (2.0 * s12 - s6) / r2


def lj_compute(sys: Ranked, lists, eps, sigma, rc):
    """Weighted E, scattered F, 6-virial, reverse comm (mdkk/pair_lj.py:114-179).

    Returns (energy, forces in gid order, virial[xx,yy,zz,xy,xz,yz]).
    """
    energy, virial = 0.0, np.zeros(6)
    for rk, nl in zip(sys.ranks, lists):
        if nl.needs_rebuild():
            raise OracleError("neighbor list stale")
        rk.f[:] = 0.0
        dr = rk.x[nl.cols] - rk.x[nl.rows]
        r2 = np.einsum("ij,ij->i", dr, dr)
        m = r2 < rc * rc
        rows, cols, dr, r2 = nl.rows[m], nl.cols[m], dr[m], r2[m]
        w, wj = nl.weight[m], nl.write_j[m]
        e, fp = lj_pair(r2, eps, sigma)
        energy += float(np.dot(w, e))
        fv = fp[:, None] * dr
        np.add.at(rk.f, rows, -fv)
        np.add.at(rk.f, cols[wj], fv[wj])
        wfp = w * fp
        for k, (a, b) in enumerate(((0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2))):
            virial[k] += float(np.dot(wfp, dr[:, a] * dr[:, b]))
    if any(r.n_ghost for r in sys.ranks):
        sys.reverse()
    return energy, sys.gather_forces(), virial


def lj_reference_n2(pos, lengths, eps, sigma, rc):
    """O(N^2) minimum-image LJ E/F/W (mdkk tests/conftest.py:38-64)."""
    n = len(pos)
    e, f, w = 0.0, np.zeros((n, 3)), np.zeros(6)
    for i in range(n - 1):
        dr = pos[i + 1:] - pos[i]
        dr -= lengths * np.round(dr / lengths)
        r2 = (dr * dr).sum(axis=1)
        m = r2 < rc * rc
        dr, r2 = dr[m], r2[m]
        s6 = (sigma * sigma / r2) ** 3
        e += float(np.sum(4.0 * eps * (s6 * s6 - s6)))
        fp = 24.0 * eps * (2.0 * s6 * s6 - s6) / r2
        fv = fp[:, None] * dr
        f[i] -= fv.sum(axis=0)
        f[i + 1:][m] += fv
        for k, (a, b) in enumerate(((0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2))):
            w[k] += float(np.dot(fp, dr[:, a] * dr[:, b]))
    return e, f, w


# ---------------------------------------------------------------- integrator
class LJRun:
    """Velocity-Verlet NVE with skin rebuilds (mdkk/driver/simulation.py:348-481)."""

    def __init__(self, pos, vel, lengths, eps=1.0, sigma=1.0, rc=2.5, skin=0.3,
                 style="half", newton=True, n_ranks=1, dt=0.005, mass=1.0):
        self.eps, self.sigma, self.rc, self.skin = eps, sigma, rc, skin
        self.style, self.newton, self.dt, self.mass = style, newton, dt, mass
        self.sys = Ranked(lengths, n_ranks, pos, vel)
        self.lists = build_all(self.sys, rc, skin, style, newton)
        self.n_builds = 1

    def forces(self):
        e, _, _ = lj_compute(self.sys, self.lists, self.eps, self.sigma, self.rc)
        return e

    def kinetic(self):
        ke = sum(0.5 * self.mass * float(np.sum(r.v * r.v)) for r in self.sys.ranks)
        n = sum(r.n_local for r in self.sys.ranks)
        return ke, (2.0 * ke / (3.0 * n) if n else 0.0)

    def step(self):
        """mdkk/driver/simulation.py:431-450."""
        h = 0.5 * self.dt / self.mass
        for r in self.sys.ranks:
            r.v += h * r.f[: r.n_local]
            r.x[: r.n_local] += self.dt * r.v
        if any(nl.needs_rebuild() for nl in self.lists):
            self.sys.migrate(self.rc + self.skin)
            self.lists = [build(r, self.sys.lengths, self.rc, self.skin, self.style, self.newton)
                          for r in self.sys.ranks]
            self.n_builds += 1
        else:
            self.sys.forward()
        e = self.forces()
        for r in self.sys.ranks:
            r.v += h * r.f[: r.n_local]
        return e

    def run(self, n_steps, thermo=100):
        """Thermo rows (step, pe, ke, etot, T) at 0, every `thermo`, and last (:452-481)."""
        rows = []
        e = self.forces()
        ke, t = self.kinetic()
        rows.append((0, e, ke, e + ke, t))
        for s in range(1, n_steps + 1):
            e = self.step()
            if not np.isfinite(e):
                raise OracleError(f"non-finite potential energy at step {s}")
            if s % thermo == 0 or s == n_steps:
                ke, t = self.kinetic()
                rows.append((s, e, ke, e + ke, t))
        return rows
