"""Box, brick decomposition, device-resident atom stores and halo communication.

Mirror of mdkk/domain.py (Box :22-42, minimum_image :45-53, wrap_positions
:56-63, RankSet :66-95, decompose :98-123, AtomStore :126-193, RankedSystem
:210-354) with every per-atom operation on the GPU:

* rows live in HBM as AoS double4 (x, y, z, pad);
* owned rows are kept in spatial (cell) order — re-sorted at every migrate —
  so neighbour gathers stay in L1/L2; outputs are still returned in global-id
  order (`gather`, `gather_forces`), as the reference guarantees;
* ghost selection, forward pack (+ periodic shift), reverse fold and
  migration are CUDA kernels (csrc/domain.cu, csrc/neighbor.cu); in-process
  logical ranks on one device exchange through device copies, one-rank-per-GPU
  runs go through `paper_2508_13523_b200.dist` (NCCL).
"""

from __future__ import annotations

import itertools

import numpy as np
import torch

from . import _lib
from .memspace import DualArray, download, download_async, upload


class DomainError(RuntimeError):
    """Invalid decomposition, box, or communication request (mdkk/domain.py:18)."""


# shift code c = (sx+1)*9 + (sy+1)*3 + (sz+1) == itertools.product((-1,0,1), repeat=3) order
SHIFT_UNITS = np.array(list(itertools.product((-1, 0, 1), repeat=3)), dtype=np.float64)
IDENTITY_CODE = 13


class Box:
    """Orthorhombic periodic box (mdkk/domain.py:22-42)."""

    def __init__(self, lengths, periodic=(True, True, True)):
        self.lengths = np.asarray(lengths, dtype=np.float64)
        if self.lengths.shape != (3,) or np.any(self.lengths <= 0):
            raise DomainError(f"box lengths must be 3 positive reals, got {lengths}")
        self.periodic = tuple(bool(p) for p in periodic)
        if len(self.periodic) != 3:
            raise DomainError("periodic must have 3 flags")
        if not all(self.periodic):
            raise DomainError("only fully periodic boxes are supported (mdkk/driver/simulation.py:257-259)")

    @property
    def volume(self) -> float:
        return float(np.prod(self.lengths))

    def min_periodic_length(self) -> float:
        return float(self.lengths.min())

    def __repr__(self):
        return f"Box(lengths={self.lengths.tolist()}, periodic={self.periodic})"


def minimum_image(dr, box: Box) -> np.ndarray:
    """Host helper: components mapped into [-L/2, L/2) (mdkk/domain.py:45-53)."""
    dr = np.array(dr, dtype=np.float64, copy=True)
    v = dr.reshape(-1, 3)
    v -= box.lengths * np.floor(v / box.lengths + 0.5)
    return v.reshape(dr.shape)


def wrap_positions(pos, box: Box) -> np.ndarray:
    """Host helper: wrap into [0, L) (mdkk/domain.py:56-63)."""
    pos = np.array(pos, dtype=np.float64, copy=True)
    return pos - box.lengths * np.floor(pos / box.lengths)


class RankSet:
    """Brick tiling of the box (mdkk/domain.py:66-95)."""

    def __init__(self, box: Box, grid):
        self.box = box
        self.grid = tuple(int(g) for g in grid)
        if any(g < 1 for g in self.grid):
            raise DomainError(f"invalid rank grid {grid}")
        self.n_ranks = self.grid[0] * self.grid[1] * self.grid[2]
        self.lo = np.zeros((self.n_ranks, 3))
        self.hi = np.zeros((self.n_ranks, 3))
        for r in range(self.n_ranks):
            c = self.coords(r)
            for d in range(3):
                self.lo[r, d] = box.lengths[d] * c[d] / self.grid[d]
                self.hi[r, d] = box.lengths[d] * (c[d] + 1) / self.grid[d]

    def coords(self, rank: int):
        gx, gy, gz = self.grid
        return (rank // (gy * gz), (rank // gz) % gy, rank % gz)

    def rank_of(self, pos: np.ndarray) -> np.ndarray:
        g = np.array(self.grid)
        c = np.clip(np.floor(pos / self.box.lengths * g.astype(np.float64)).astype(np.int64), 0, g - 1)
        return (c[:, 0] * g[1] + c[:, 1]) * g[2] + c[:, 2]


def decompose(box: Box, n_ranks: int) -> RankSet:
    """Minimal-surface brick grid, ties split lower axes (mdkk/domain.py:98-123)."""
    if n_ranks < 1:
        raise DomainError(f"n_ranks must be >= 1, got {n_ranks}")
    best = None
    for gx in range(1, n_ranks + 1):
        if n_ranks % gx:
            continue
        rem = n_ranks // gx
        for gy in range(1, rem + 1):
            if rem % gy:
                continue
            gz = rem // gy
            e = box.lengths / np.array([gx, gy, gz])
            key = (2.0 * (e[0] * e[1] + e[0] * e[2] + e[1] * e[2]), (-gx, -gy, -gz))
            if best is None or key < best[0]:
                best = (key, (gx, gy, gz))
    return RankSet(box, best[1])


def _rows4(n: int, device, zero: bool = True) -> torch.Tensor:
    t = torch.empty((max(n, 1), 4), dtype=torch.float64, device=device)
    return t.zero_() if zero else t


def _to4(a: np.ndarray, device, cap: int | None = None) -> torch.Tensor:
    t = _rows4(max(cap or 0, len(a)), device)
    if len(a):
        t[: len(a), :3] = upload(np.asarray(a, dtype=np.float64), device)
    return t


def _dense_ids(gids: np.ndarray, n: int) -> bool:
    """gids is a permutation of 0..n-1 (O(n), no sort)."""
    if n == 0:
        return True
    if gids.min() != 0 or gids.max() != n - 1:
        return False
    seen = np.zeros(n, dtype=bool)
    seen[gids] = True
    return bool(seen.all())


def device_partition(box: Box, rs: RankSet, positions, velocities, global_ids, device, ranks=None):
    """Upload once, wrap and assign owners on the device (mdkk/domain.py:220-235).

    Returns ({rank: (x rows4 with ghost headroom, v rows4, gid int64, n)}, dense).
    Rows of each brick keep the input order (the reference's
    ``np.flatnonzero(owner == r)``): the owner partition is a stable radix
    sort.  Wrap is bit-identical to mdkk/domain.py:62.
    """
    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
    vel = np.ascontiguousarray(np.asarray(velocities, dtype=np.float64).reshape(-1, 3))
    n = len(pos)
    if global_ids is None:
        dense = True
        gid = torch.arange(max(n, 1), dtype=torch.int64, device=device)
    else:
        g_host = np.asarray(global_ids, dtype=np.int64).reshape(-1)
        dense = _dense_ids(g_host, n)
        gid = torch.from_numpy(g_host).to(device) if n else torch.zeros(1, dtype=torch.int64, device=device)
    R = rs.n_ranks
    ranks = range(R) if ranks is None else ranks
    lib, stream = _lib.lib(), _lib.stream(device)
    cap_all = int(n * 1.3) + 64 if R == 1 else n
    x = _rows4(cap_all, device)
    v = _rows4(n, device)
    if n:
        x[:n, :3] = upload(pos, device)
        v[:n, :3] = upload(vel, device)
        _lib.check(lib.mdkk_wrap(x.data_ptr(), n, _lib.dbl3(box.lengths), stream), "mdkk_wrap")
    if R == 1:
        g = torch.zeros(cap_all, dtype=torch.int64, device=device)
        g[:n] = gid[:n]
        return {0: (x, v, g, n)}, dense
    ctx = _lib.ctx(device)
    keys = torch.empty(max(n, 1), dtype=torch.int32, device=device)
    start = torch.zeros(R + 1, dtype=torch.int32, device=device)
    order = torch.empty(max(n, 1), dtype=torch.int32, device=device)
    if n:
        _lib.check(lib.mdkk_rank_keys(x.data_ptr(), n, _lib.dbl3(box.lengths), _lib.int_arr(rs.grid),
                                      keys.data_ptr(), stream), "mdkk_rank_keys")
        _lib.check(lib.mdkk_bucket_sort(ctx, keys.data_ptr(), n, R, start.data_ptr(), order.data_ptr(), stream),
                   "mdkk_bucket_sort")
    st = start.cpu().numpy().astype(np.int64)
    out = {}
    for r in ranks:
        a, b = int(st[r]), int(st[r + 1])
        c = b - a
        cap = int(c * 1.3) + 64
        xr, vr = _rows4(cap, device), _rows4(c, device)
        gr = torch.zeros(cap, dtype=torch.int64, device=device)
        if c:
            o = order[a:b]
            _lib.check(lib.mdkk_gather_rows4(x.data_ptr(), o.data_ptr(), c, xr.data_ptr(), stream), "g4")
            _lib.check(lib.mdkk_gather_rows4(v.data_ptr(), o.data_ptr(), c, vr.data_ptr(), stream), "g4")
            _lib.check(lib.mdkk_gather_i64(gid.data_ptr(), o.data_ptr(), c, gr.data_ptr(), stream), "g64")
        out[r] = (xr, vr, gr, c)
    return out, dense


_ROW = None


class AtomStore:
    """One rank's rows in HBM: n_local owned rows followed by n_ghost ghosts (mdkk/domain.py:126-193).

    Device buffers have spare capacity so rebuilds reuse them: ``x``/``f``
    (cap, 4) f64, ``gid`` int64, ``orank``/``oidx`` int32 per row, ``v``
    (cap_local, 4).  Rows [0, n_total) are valid.  ``pos``/``vel``/``force``
    are DualArray views over the valid rows (space "a" = host numpy,
    "b" = HBM), following the reference's protocol (mdkk/memspace.py:77-156).
    """

    def __init__(self, rank: int, device, x: torch.Tensor, v: torch.Tensor, gid: torch.Tensor, n_local: int):
        self.rank = int(rank)
        self.device = torch.device(device)
        self.n_local = int(n_local)
        self.n_ghost = 0
        self.x, self.v, self.gid = x, v, gid
        cap = x.shape[0]
        if gid.shape[0] < cap:
            g = torch.empty(cap, dtype=torch.int64, device=self.device)
            g[: gid.shape[0]] = gid
            self.gid = g
        self.f = torch.zeros_like(x)
        self.orank = torch.full((cap,), self.rank, dtype=torch.int32, device=self.device)
        self.oidx = torch.arange(cap, dtype=torch.int32, device=self.device)
        self.pos = None
        self.lo = self.hi = None  # brick bounds, set by RankedSystem
        self._lengths = None
        self._lanes_in = []       # lanes whose ghost rows live here (for ghost_shift)
        self._alt = None          # double buffers for the spatial sort
        self._bins = None         # (width, n_local, bucket starts) of the last spatial sort
        self._views()
        self.device_wrote(pos=True, vel=True)   # the rows were uploaded: HBM holds the current data

    @property
    def capacity(self) -> int:
        return self.x.shape[0]

    def _views(self):
        nt, nl = max(self.n_total, 1), max(self.n_local, 1)
        if getattr(self, "pos", None) is None:
            self.pos = DualArray((nt, 3), device=self.device, pad_last=4, storage_b=self.x[:nt], layout_b=_ROW)
            self.vel = DualArray((nl, 3), device=self.device, pad_last=4, storage_b=self.v[:nl], layout_b=_ROW)
            self.force = DualArray((nt, 3), device=self.device, pad_last=4, storage_b=self.f[:nt], layout_b=_ROW)
        else:   # rebuilds: re-point the existing mirrors (fresh and clean, as new ones would be)
            self.pos.rebind((nt, 3), self.x[:nt])
            self.vel.rebind((nl, 3), self.v[:nl])
            self.force.rebind((nt, 3), self.f[:nt])
        self._host_cache = {}

    def ensure_capacity(self, rows: int) -> None:
        """Grow the per-row buffers (keeping owned rows) when `rows` exceeds capacity."""
        if rows <= self.capacity:
            return
        cap = int(rows * 1.15) + 64
        nl = self.n_local
        x = _rows4(cap, self.device)   # zeroed once: the double4 pad lane is read by 256-bit loads
        x[:nl] = self.x[:nl]
        g = torch.empty(cap, dtype=torch.int64, device=self.device)
        g[:nl] = self.gid[:nl]
        self.x, self.gid = x, g
        self.f = torch.zeros((cap, 4), dtype=torch.float64, device=self.device)
        self.orank = torch.full((cap,), self.rank, dtype=torch.int32, device=self.device)
        self.oidx = torch.arange(cap, dtype=torch.int32, device=self.device)
        self._alt = None

    def to_device(self):
        """Make device storage current before a kernel reads it."""
        if self.pos.modified_a:
            # host-written positions: the last spatial sort's cell order no longer holds,
            # so the boundary-row halo scan and ghost-only binning must not reuse it
            self._bins = None
        self.pos.sync("b")
        self.vel.sync("b")
        self.force.sync("b")

    def device_wrote(self, pos=False, vel=False, force=False):
        if pos:
            self.pos.mark_modified("b")
        if vel:
            self.vel.mark_modified("b")
        if force:
            self.force.mark_modified("b")

    @property
    def n_total(self) -> int:
        return self.n_local + self.n_ghost

    def positions(self) -> np.ndarray:
        return self.pos.read("a")[: self.n_total]

    def velocities(self) -> np.ndarray:
        return self.vel.read("a")[: self.n_local]

    def forces(self) -> np.ndarray:
        return self.force.read("a")[: self.n_total]

    def _host(self, name, t, n):
        h = self._host_cache.get(name)
        if h is None:
            h = self._host_cache[name] = t[:n].cpu().numpy()
        return h

    @property
    def global_ids(self) -> np.ndarray:
        return self._host("gid", self.gid, self.n_total)

    @property
    def owner_rank(self) -> np.ndarray:
        return self._host("orank", self.orank, self.n_total)

    @property
    def owner_index(self) -> np.ndarray:
        return self._host("oidx", self.oidx, self.n_total)

    @property
    def ghost_shift(self) -> np.ndarray:
        h = self._host_cache.get("shift")
        if h is None:
            h = np.zeros((self.n_total, 3))
            for ln in self._lanes_in:
                codes = ln.code.cpu().numpy().astype(np.int64)
                h[ln.start:ln.start + ln.count] = SHIFT_UNITS[codes] * self._lengths
            self._host_cache["shift"] = h
        return h


def _init_layout():
    global _ROW
    from .memspace import LayoutPolicy
    _ROW = LayoutPolicy.row_major(2)


_init_layout()


_COMBO_MEMO: dict = {}   # (device, src, halo, box, grid) -> (meta, combo table, codes)


class _Lane:
    """One (src rank -> dst rank) forward/reverse lane: ghost rows [start, start+count) of dst."""

    __slots__ = ("src", "dst", "idx", "code", "start", "count")

    def __init__(self, src, dst, idx, code, start, count):
        self.src, self.dst, self.idx, self.code, self.start, self.count = src, dst, idx, code, start, count


class RankedSystem:
    """All in-process ranks of one device plus their halo plan (mdkk/domain.py:210-354)."""

    def __init__(self, box: Box, rankset: RankSet, stores: list[AtomStore], device, dense_gids: bool):
        self.box = box
        self.rankset = rankset
        self.stores = stores
        self.device = torch.device(device)
        self.halo = 0.0
        self.lanes: list[_Lane] = []
        self.dense_gids = dense_gids
        self.n_atoms = sum(s.n_local for s in stores)
        self._shift_dev = torch.from_numpy(SHIFT_UNITS * box.lengths).to(self.device)
        self._lengths_c = _lib.dbl3(box.lengths)   # ctypes double[3] for the per-rebuild calls
        self._combo_cache = {}
        self._scratch = {}
        self.sort_width = None  # spatial-sort bin width (set by the first neighbour build)
        for s in stores:
            self._attach(s)

    def _attach(self, s: AtomStore):
        s.lo, s.hi, s._lengths = self.rankset.lo[s.rank], self.rankset.hi[s.rank], self.box.lengths

    def _buf(self, name, n, dtype):
        t = self._scratch.get(name)
        if t is None or t.numel() < n:
            t = self._scratch[name] = torch.empty(max(int(n * 1.15) + 64, 1), dtype=dtype, device=self.device)
        return t

    @property
    def n_ranks(self) -> int:
        return self.rankset.n_ranks

    @classmethod
    def distribute(cls, box: Box, n_ranks: int, positions, velocities, global_ids=None,
                   device=None) -> "RankedSystem":
        """Wrap, assign owners, upload (mdkk/domain.py:220-235); one upload, owners assigned on device."""
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        rs = decompose(box, n_ranks)
        parts, dense = device_partition(box, rs, positions, velocities, global_ids, device)
        stores = [AtomStore(r, device, *parts[r]) for r in range(rs.n_ranks)]
        return cls(box, rs, stores, device, dense)

    # ------------------------------------------------------------ ghosts
    def _combos(self, src: int, halo: float):
        """(dst, code) combos for src, dst-major then shift order (mdkk/domain.py:263-271) + device table."""
        key = (src, halo)
        hit = self._combo_cache.get(key)
        if hit is not None:
            return hit
        # the table depends only on the box, the brick grid and the halo: shared by every
        # system on this device with the same decomposition (a new Simulation reuses it)
        gkey = (str(self.device), src, float(halo), tuple(float(v) for v in self.box.lengths),
                tuple(self.rankset.grid))
        hit = _COMBO_MEMO.get(gkey)
        if hit is not None:
            self._combo_cache[key] = hit
            return hit
        L = self.box.lengths
        rs = self.rankset
        meta, rows = [], []
        for dst in range(self.n_ranks):
            lo, hi = rs.lo[dst] - halo, rs.hi[dst] + halo
            for code in range(27):
                if dst == src and code == IDENTITY_CODE:
                    continue
                shift = SHIFT_UNITS[code] * L
                # prune combos whose shifted (halo-padded) source brick cannot reach dst
                slo, shi = rs.lo[src] - halo + shift, rs.hi[src] + halo + shift
                if np.any(shi <= lo) or np.any(slo >= hi):
                    continue
                meta.append((dst, code))
                rows.append(np.concatenate([lo, hi, shift]))
        tab = torch.from_numpy(np.array(rows) if rows else np.zeros((0, 9))).to(self.device)
        codes = torch.tensor([c for _, c in meta], dtype=torch.int8, device=self.device)
        hit = self._combo_cache[key] = _COMBO_MEMO[gkey] = (meta, tab, codes)
        return hit

    def exchange_ghosts(self, halo: float) -> None:
        """Select ghosts on device and rebuild ghost rows + lanes (mdkk/domain.py:246-293).

        One host sync (the per-combo totals); everything else is launched
        asynchronously into reused buffers.
        """
        if halo <= 0:
            raise DomainError(f"halo must be positive, got {halo}")
        if halo > 0.5 * self.box.min_periodic_length():
            raise DomainError(f"halo {halo} exceeds half the shortest periodic box length "
                              f"{self.box.min_periodic_length()}; periodic image is ambiguous")
        self.halo = float(halo)
        lib, stream = _lib.lib(), _lib.stream(self.device)
        ctx = _lib.ctx(self.device)
        for s in self.stores:
            s.to_device()
        if self.n_ranks == 1 and self.stores[0].n_local and self._combos(0, halo)[0]:
            return self._exchange_single(halo, lib, stream, ctx)
        self._run_tails()
        plans = []
        for src in self.stores:
            meta, tab, codes = self._combos(src.rank, halo)
            C_ = len(meta)
            if C_ == 0 or src.n_local == 0:
                plans.append(None)
                continue
            nb = (src.n_local + 255) // 256
            blk = self._buf(f"blk{src.rank}", nb * C_, torch.int32)
            tot = self._buf(f"tot{src.rank}", C_, torch.int32)[:C_]
            _lib.check(lib.mdkk_halo_count(ctx, src.x.data_ptr(), src.n_local, tab.data_ptr(), C_,
                                           blk.data_ptr(), tot.data_ptr(), None, None, stream), "mdkk_halo_count")
            plans.append((meta, tab, codes, blk, tot))
        live = [p for p in plans if p is not None]
        host_tot = torch.cat([p[4] for p in live]).cpu().numpy() if live else np.zeros(0, np.int64)
        sel = {}   # (src, dst) -> (idx view, code tensor, count)
        off_all = 0
        for src, plan in zip(self.stores, plans):
            if plan is None:
                continue
            meta, tab, codes, blk, tot = plan
            C_ = len(meta)
            totals = host_tot[off_all:off_all + C_].astype(np.int64)
            off_all += C_
            idx = self._buf(f"idx{src.rank}", int(totals.sum()) + 1, torch.int32)
            cds = self._buf(f"cds{src.rank}", int(totals.sum()) + 1, torch.int8)
            _lib.check(lib.mdkk_halo_fill(ctx, src.x.data_ptr(), src.n_local, tab.data_ptr(), C_, blk.data_ptr(),
                                          tot.data_ptr(), idx.data_ptr(), codes.data_ptr(), cds.data_ptr(),
                                          None, None, stream), "mdkk_halo_fill")
            # combos are dst-major: each (src, dst) lane is one contiguous run of idx
            start = np.concatenate([[0], np.cumsum(totals)])
            d_of = np.array([d for d, _ in meta])
            for d in np.unique(d_of):
                ks = np.flatnonzero(d_of == d)
                a, b = int(start[ks[0]]), int(start[ks[-1] + 1])
                if b > a:
                    sel[(src.rank, int(d))] = (idx[a:b], cds[a:b], b - a)
        self.lanes = []
        for dst in self.stores:
            nl = dst.n_local
            ng = sum(sel[(s, dst.rank)][2] for s in range(self.n_ranks) if (s, dst.rank) in sel)
            dst.ensure_capacity(nl + ng)
            dst._lanes_in = []
            cur = nl
            for s in range(self.n_ranks):
                if (s, dst.rank) not in sel:
                    continue
                ix, code, t = sel[(s, dst.rank)]
                sst = self.stores[s]
                _lib.check(lib.mdkk_gather_i64(sst.gid.data_ptr(), ix.data_ptr(), t, dst.gid[cur:].data_ptr(),
                                               stream), "mdkk_gather_i64")
                if self.n_ranks > 1:   # one rank: orank is uniformly 0 from allocation on
                    dst.orank[cur:cur + t].fill_(s)
                dst.oidx[cur:cur + t].copy_(ix)
                ln = _Lane(s, dst.rank, ix, code, cur, t)
                self.lanes.append(ln)
                dst._lanes_in.append(ln)
                cur += t
            dst.n_ghost = ng
            if nl and self.n_ranks > 1:
                dst.orank[:nl].fill_(dst.rank)
            dst._views()
        self._pack_all()
        for s in self.stores:
            s.device_wrote(pos=True)

    def _exchange_single(self, halo, lib, stream, ctx) -> None:
        """One rank (periodic self-images only): the same selection, lane and rows as the
        general path with a fraction of its host work -- one pinned totals read-back and
        one fused ghost-row kernel (position + gid + owner index)."""
        s = self.stores[0]
        meta, tab, codes = self._combos(0, halo)
        C_, nl = len(meta), s.n_local
        nb = (nl + 255) // 256
        blk = self._buf("blk0", nb * C_, torch.int32)
        tot = self._buf("tot0", C_, torch.int32)[:C_]
        rows = nrow = None
        bins = getattr(s, "_bins", None)
        if bins is not None and bins[1] == nl and bins[0] >= halo:
            # owned rows are cell-sorted on the shell grid with cells >= halo wide: only
            # rows within two cell layers of the faces can be selected (ascending list)
            _, _, _, narr, _ = shell_grid_args(s.lo, s.hi, bins[0])
            rows = self._buf("brows0", nl, torch.int32)
            nrow = self._buf("bcount0", 1, torch.int32)
            _lib.check(lib.mdkk_boundary_rows(ctx, bins[2].data_ptr(), narr, 2, rows.data_ptr(), nrow.data_ptr(),
                                              stream), "mdkk_boundary_rows")
        rp = rows.data_ptr() if rows is not None else None
        cp = nrow.data_ptr() if nrow is not None else None
        _lib.check(lib.mdkk_halo_count(ctx, s.x.data_ptr(), nl, tab.data_ptr(), C_, blk.data_ptr(), tot.data_ptr(),
                                       rp, cp, stream), "mdkk_halo_count")
        pin = self._scratch.get("tot_pin")
        if pin is None or pin.numel() < C_:
            pin = self._scratch["tot_pin"] = torch.zeros(max(C_, 64), dtype=torch.int32, pin_memory=True)
        pin[:C_].copy_(tot, non_blocking=True)
        ev = self._scratch.get("tot_ev")
        if ev is None:
            ev = self._scratch["tot_ev"] = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self._run_tails()   # deferred sort gathers: device work while the host waits for the totals
        ev.synchronize()
        ng = sum(pin[:C_].tolist())
        idx = self._buf("idx0", ng + 1, torch.int32)
        cds = self._buf("cds0", ng + 1, torch.int8)
        _lib.check(lib.mdkk_halo_fill(ctx, s.x.data_ptr(), nl, tab.data_ptr(), C_, blk.data_ptr(), tot.data_ptr(),
                                      idx.data_ptr(), codes.data_ptr(), cds.data_ptr(), rp, cp, stream),
                   "mdkk_halo_fill")
        s.ensure_capacity(nl + ng)
        _lib.check(lib.mdkk_ghost_rows(s.x.data_ptr(), s.gid.data_ptr(), idx.data_ptr(), cds.data_ptr(),
                                       self._shift_dev.data_ptr(), ng, s.x[nl:].data_ptr(), s.gid[nl:].data_ptr(),
                                       s.oidx[nl:].data_ptr(), stream), "mdkk_ghost_rows")
        ln = _Lane(0, 0, idx[:ng], cds[:ng], nl, ng)
        self.lanes = [ln] if ng else []
        s._lanes_in = list(self.lanes)
        s.n_ghost = ng
        s._views()
        s.device_wrote(pos=True)

    def _migrate_single(self, halo: float, width: float, zero_forces: bool, ref_out=None) -> int:
        """One rank, periodic self-images only: migrate = wrap + spatial sort + ghost
        selection + ghost rows, with everything up to the ghost totals issued by one
        library call (mdkk_rebuild1_select).  The same kernels in the same order as the
        general path (bit-identical rows, ghosts and bins); 0 when the fast path does
        not apply (nothing done), 1 when done, 2 when `ref_out` was also written."""
        s = self.stores[0]
        n = s.n_local
        # the call's fixed arguments, prepared once per (halo, width, n): a rebuild goes from
        # the host's decision to the first kernel with little Python in between
        pre = self._scratch.get(("sel", halo, width, n))
        if pre is None:
            if halo <= 0 or halo > 0.5 * self.box.min_periodic_length():
                return 0   # the general path raises the reference's DomainError
            meta, tab, codes = self._combos(0, halo)
            C_ = len(meta)
            if C_ == 0:
                return 0
            _, _, garr, narr, ncell = shell_grid_args(s.lo, s.hi, width)
            pin = self._scratch.get("tot_pin")
            if pin is None or pin.numel() < C_:
                pin = self._scratch["tot_pin"] = torch.zeros(max(C_, 64), dtype=torch.int32, pin_memory=True)
            pre = self._scratch[("sel", halo, width, n)] = (
                C_, tab, codes, garr, narr, ncell, self._buf("sk0", n, torch.int32),
                self._buf("ss0", ncell + 1, torch.int32), self._buf("so0", n, torch.int32),
                self._buf("brows0", n, torch.int32), self._buf("bcount0", 1, torch.int32),
                self._buf("blk0", ((n + 255) // 256) * C_, torch.int32), self._buf("tot0", C_, torch.int32), pin)
        C_, tab, codes, garr, narr, ncell, keys, start, order, rows, nrow, blk, tot, pin = pre
        if ref_out is not None and (ref_out.shape[0] < n or ref_out.device != self.device):
            ref_out = None
        lib, stream, ctx = _lib.lib(), _lib.stream(self.device), _lib.ctx(self.device)
        s.to_device()
        s.n_ghost = 0
        s._lanes_in = []
        if s._alt is None or s._alt[0].shape[0] != s.capacity or s._alt[1].shape[0] < n:
            s._alt = (_rows4(s.capacity, self.device), _rows4(s.v.shape[0], self.device),
                      torch.empty(s.capacity, dtype=torch.int64, device=self.device))
        x2, v2, g2 = s._alt
        ngh = _lib.C.c_int(0)
        _lib.check(lib.mdkk_rebuild1_select(
            ctx, s.x.data_ptr(), n, self._lengths_c, garr, narr, keys.data_ptr(), start.data_ptr(),
            order.data_ptr(), x2.data_ptr(), s.v.data_ptr(), v2.data_ptr(), s.gid.data_ptr(), g2.data_ptr(),
            rows.data_ptr(), nrow.data_ptr(), tab.data_ptr(), C_, blk.data_ptr(), tot.data_ptr(), pin.data_ptr(),
            _lib.C.byref(ngh), ref_out.data_ptr() if ref_out is not None else None, stream), "mdkk_rebuild1_select")
        ng = ngh.value
        s._alt = (s.x, s.v, s.gid)
        s.x, s.v, s.gid = x2, v2, g2
        s._bins = (float(width), n, start)   # owned rows sorted on shell_grid_args(lo, hi, width)
        self.halo = float(halo)
        idx = self._buf("idx0", ng + 1, torch.int32)
        cds = self._buf("cds0", ng + 1, torch.int8)
        _lib.check(lib.mdkk_halo_fill(ctx, s.x.data_ptr(), n, tab.data_ptr(), C_, blk.data_ptr(), tot.data_ptr(),
                                      idx.data_ptr(), codes.data_ptr(), cds.data_ptr(), rows.data_ptr(),
                                      nrow.data_ptr(), stream), "mdkk_halo_fill")
        s.ensure_capacity(n + ng)
        xp, gp, op = s.x.data_ptr(), s.gid.data_ptr(), s.oidx.data_ptr()
        _lib.check(lib.mdkk_ghost_rows(xp, gp, idx.data_ptr(), cds.data_ptr(), self._shift_dev.data_ptr(), ng,
                                       xp + 32 * n, gp + 8 * n, op + 4 * n, stream), "mdkk_ghost_rows")
        ln = _Lane(0, 0, idx[:ng], cds[:ng], n, ng)
        self.lanes = [ln] if ng else []
        s._lanes_in = list(self.lanes)
        s.n_ghost = ng
        s._views()
        s.device_wrote(pos=True, vel=True, force=True)
        if zero_forces:
            s.f[: s.n_total].zero_()
        return 2 if ref_out is not None else 1

    def _run_tails(self):
        for s in self.stores:
            t = getattr(s, "_tail", None)
            if t is not None:
                s._tail = None
                t()

    def _pack_all(self):
        lib, stream = _lib.lib(), _lib.stream(self.device)
        for ln in self.lanes:
            s, d = self.stores[ln.src], self.stores[ln.dst]
            _lib.check(lib.mdkk_pack_shift(s.x.data_ptr(), ln.idx.data_ptr(), ln.code.data_ptr(),
                                           self._shift_dev.data_ptr(), ln.count,
                                           d.x[ln.start:].data_ptr(), stream), "mdkk_pack_shift")

    def forward_comm(self) -> None:
        """ghost x = owner x + shift, on device (mdkk/domain.py:295-305)."""
        for s in self.stores:
            s.to_device()
        self._pack_all()
        for s in self.stores:
            if s.n_ghost:
                s.device_wrote(pos=True)

    def reverse_comm(self, ordered: bool = False) -> None:
        """Fold ghost forces onto owners, zero ghost rows (mdkk/domain.py:307-322).

        FP64 RED folds; `ordered` (the Serial strategy) folds each owner row's
        contributions one by one in lane order instead -- deterministic, like the
        reference's np.add.at."""
        lib, stream = _lib.lib(), _lib.stream(self.device)
        for s in self.stores:
            s.to_device()
        for ln in self.lanes:
            s, d = self.stores[ln.src], self.stores[ln.dst]
            if ordered:
                from .memspace import ordered_scatter
                if ln.count:
                    ordered_scatter(s.f, 4, 3, ln.idx[: ln.count].long(),
                                    d.f[ln.start:ln.start + ln.count, :3].contiguous())
                continue
            _lib.check(lib.mdkk_fold_add(s.f.data_ptr(), ln.idx.data_ptr(), d.f[ln.start:].data_ptr(),
                                         ln.count, stream), "mdkk_fold_add")
        for s in self.stores:
            if s.n_ghost:
                s.f[s.n_local:s.n_total].zero_()
            s.device_wrote(force=True)

    # ----------------------------------------------------------- migration
    def migrate(self, halo: float, sort_width: float | None = None, zero_forces: bool = True,
                ref_out: torch.Tensor | None = None) -> bool:
        """Wrap, reassign bricks, re-sort spatially, zero forces, rebuild ghosts (mdkk/domain.py:324-334).
        `zero_forces=False` (engine-internal: the forces are recomputed right away, and every
        force path clears or overwrites the rows it reads) skips the reset.  `ref_out`
        (engine-internal, one rank): rows4 buffer that also receives the sorted owned
        positions (the next lists' skin-test reference); returns whether it was written."""
        lib, stream = _lib.lib(), _lib.stream(self.device)
        ctx = _lib.ctx(self.device)
        L = _lib.dbl3(self.box.lengths)
        R = self.n_ranks
        w = sort_width or self.sort_width
        if R == 1 and w and w >= halo and self.stores[0].n_local >= 2:
            done = self._migrate_single(halo, w, zero_forces, ref_out)
            if done:
                return done == 2
        grid = _lib.int_arr(self.rankset.grid)
        for s in self.stores:
            s.to_device()
            _lib.check(lib.mdkk_wrap(s.x.data_ptr(), s.n_local, L, stream), "mdkk_wrap")
        if R > 1:
            parts = {}  # dst -> list of (src, order segment)
            for s in self.stores:
                keys = self._buf(f"rk{s.rank}", s.n_local + 1, torch.int32)
                start = torch.empty(R + 1, dtype=torch.int32, device=self.device)
                order = torch.empty(max(s.n_local, 1), dtype=torch.int32, device=self.device)
                _lib.check(lib.mdkk_rank_keys(s.x.data_ptr(), s.n_local, L, grid, keys.data_ptr(), stream),
                           "mdkk_rank_keys")
                _lib.check(lib.mdkk_bucket_sort(ctx, keys.data_ptr(), s.n_local, R, start.data_ptr(),
                                                order.data_ptr(), stream), "mdkk_bucket_sort")
                st = start.cpu().numpy()
                for d in range(R):
                    if st[d + 1] > st[d]:
                        parts.setdefault(d, []).append((s, order[st[d]:st[d + 1]], int(st[d + 1] - st[d])))
            new = []
            for d in range(R):
                segs = parts.get(d, [])
                n = sum(p[2] for p in segs)
                cap = int(n * 1.3) + 64
                x, v = _rows4(cap, self.device), _rows4(n, self.device)
                gid = torch.zeros(cap, dtype=torch.int64, device=self.device)
                cur = 0
                for s, o, c in segs:
                    _lib.check(lib.mdkk_gather_rows4(s.x.data_ptr(), o.data_ptr(), c, x[cur:].data_ptr(), stream), "g4")
                    _lib.check(lib.mdkk_gather_rows4(s.v.data_ptr(), o.data_ptr(), c, v[cur:].data_ptr(), stream), "g4")
                    _lib.check(lib.mdkk_gather_i64(s.gid.data_ptr(), o.data_ptr(), c, gid[cur:].data_ptr(), stream), "g64")
                    cur += c
                st = AtomStore(d, self.device, x, v, gid, n)
                self._attach(st)
                new.append(st)
            self.stores = new
        else:
            s = self.stores[0]
            s.n_ghost = 0
            s._lanes_in = []
        if w:
            for s in self.stores:
                # one rank: the v / gid gathers go behind the exchange's totals read-back
                self._spatial_sort(s, w, halo, defer_tail=R == 1)
        for s in self.stores:
            s.n_ghost = 0
            s._views()
            s.device_wrote(pos=True, vel=True, force=True)
        self.exchange_ghosts(halo)
        if zero_forces:
            for s in self.stores:   # the reference resets forces at migration (new AtomStores)
                s.f[: s.n_total].zero_()
        return False

    def sort_local(self, width: float) -> None:
        """Re-order every rank's owned rows into serpentine cell order (drops ghosts; call before exchange)."""
        for s in self.stores:
            s.to_device()
            s.n_ghost = 0
            s._lanes_in = []
            self._spatial_sort(s, width, width)
            s._views()
            s.device_wrote(pos=True, vel=True, force=True)
        self.lanes = []

    def _spatial_sort(self, s: AtomStore, width: float, halo: float, defer_tail: bool = False):
        """Reorder owned rows by cell (double-buffered) so neighbour gathers are local; gids travel.
        `defer_tail`: the velocity / gid gathers are left in `s._tail` for the caller to queue
        later (the one-rank exchange queues them behind its totals read-back, so the device
        has work while the host waits for the totals)."""
        if s.n_local < 2:
            return
        lib, stream = _lib.lib(), _lib.stream(self.device)
        ctx = _lib.ctx(self.device)
        # the brick's cells plus a shell layer: the owned rows' sort order and bucket starts
        # are then reused by the neighbour build's binning (mdkk_bin_merge)
        _, _, garr, narr, ncell = shell_grid_args(s.lo, s.hi, width)
        n = s.n_local
        keys = self._buf(f"sk{s.rank}", n, torch.int32)
        start = self._buf(f"ss{s.rank}", ncell + 1, torch.int32)
        order = self._buf(f"so{s.rank}", n, torch.int32)
        _lib.check(lib.mdkk_bin_atoms(ctx, s.x.data_ptr(), n, garr, narr,
                                      keys.data_ptr(), start.data_ptr(), order.data_ptr(), stream), "bin")
        if s._alt is None or s._alt[0].shape[0] != s.capacity or s._alt[1].shape[0] < n:
            s._alt = (_rows4(s.capacity, self.device), _rows4(s.v.shape[0], self.device),
                      torch.empty(s.capacity, dtype=torch.int64, device=self.device))
        x2, v2, g2 = s._alt
        _lib.check(lib.mdkk_gather_rows4(s.x.data_ptr(), order.data_ptr(), n, x2.data_ptr(), stream), "g4")
        vp, gp, op = s.v.data_ptr(), s.gid.data_ptr(), order.data_ptr()

        def tail():
            _lib.check(lib.mdkk_gather_rows4(vp, op, n, v2.data_ptr(), stream), "g4")
            _lib.check(lib.mdkk_gather_i64(gp, op, n, g2.data_ptr(), stream), "g64")
        if defer_tail:
            s._tail = tail
        else:
            tail()
        s._alt = (s.x, s.v, s.gid)
        s.x, s.v, s.gid = x2, v2, g2
        s._bins = (float(width), n, start)   # owned rows sorted on shell_grid_args(lo, hi, width)

    # -------------------------------------------------------------- gather
    def _gid_order(self, rows_fn, width, asynchronous=False):
        """Owned rows of all ranks in global-id order (device scatter when gids are 0..N-1).
        `asynchronous`: return a callable that finishes the read-back (dense gids: the
        device->host copy overlaps the work queued after this call)."""
        n = self.n_atoms
        if not self.dense_gids and asynchronous:
            rows = self._gid_order(rows_fn, width)
            return lambda: rows
        if self.dense_gids:
            lib, stream = _lib.lib(), _lib.stream(self.device)
            out = _rows4(n, self.device, zero=False)   # dense gids: every row is written
            for s in self.stores:
                if s.n_local:
                    gi = s.gid[: s.n_local].to(torch.int32)
                    _lib.check(lib.mdkk_scatter_rows4(rows_fn(s).data_ptr(), gi.data_ptr(), s.n_local,
                                                      out.data_ptr(), stream), "scatter")
            return (download_async if asynchronous else download)(out[:n, :width])
        rows = np.concatenate([rows_fn(s)[: s.n_local, :width].cpu().numpy() for s in self.stores])
        gid = np.concatenate([s.global_ids[: s.n_local] for s in self.stores])
        return rows[np.argsort(gid, kind="stable")]

    def gather(self):
        """(pos, vel, gid) of owned atoms in global-id order (mdkk/domain.py:336-342)."""
        for s in self.stores:
            s.to_device()
        pos = self._gid_order(lambda s: s.x, 3)
        vel = self._gid_order(lambda s: s.v, 3)
        if self.dense_gids:
            gid = np.arange(self.n_atoms, dtype=np.int64)
        else:
            gid = np.sort(np.concatenate([s.global_ids[: s.n_local] for s in self.stores]), kind="stable")
        return pos, vel, gid

    def gather_positions(self) -> np.ndarray:
        """Owned positions in global-id order (the thermo snapshot; no velocity read-back)."""
        for s in self.stores:
            s.to_device()
        return self._gid_order(lambda s: s.x, 3)

    def gather_positions_async(self):
        """`gather_positions` whose device->host copy overlaps the work queued next; call
        the returned function for the array."""
        for s in self.stores:
            s.to_device()
        return self._gid_order(lambda s: s.x, 3, asynchronous=True)

    def gather_forces(self) -> np.ndarray:
        """Owned forces in global-id order (mdkk/domain.py:344-348)."""
        for s in self.stores:
            s.force.sync("b")
        return self._gid_order(lambda s: s.f, 3)

    def zero_forces(self) -> None:
        for s in self.stores:
            s.force.sync("b")
            s.f.zero_()
            s.device_wrote(force=True)


_GRID_MEMO: dict = {}


def grid_args(lo, hi, halo: float, width: float):
    """cell_grid plus its ctypes arrays, memoised (bricks are fixed for a run): (grid,
    ncell[3], grid_c, ncell_c, total cells)."""
    key = (*(float(v) for v in lo), *(float(v) for v in hi), float(halo), float(width))
    hit = _GRID_MEMO.get(key)
    if hit is None:
        if len(_GRID_MEMO) > 256:
            _GRID_MEMO.clear()
        g, nc = cell_grid(lo, hi, halo, width)
        hit = _GRID_MEMO[key] = (g, nc, _lib.dbl3(g), _lib.int_arr(nc), nc[0] * nc[1] * nc[2])
    return hit


def shell_grid_args(lo, hi, width: float):
    """grid_args for the brick's own cells (width >= `width`, tiling [lo, hi) exactly) plus
    one shell layer on each side, so the same grid bins the owned rows (interior cells)
    and the ghosts within one cell width of the faces (the shell).  Memoised."""
    key = ("shell", *(float(v) for v in lo), *(float(v) for v in hi), float(width))
    hit = _GRID_MEMO.get(key)
    if hit is None:
        g, nc = cell_grid(lo, hi, 0.0, width)
        inv = np.asarray(g[3:], dtype=np.float64)
        w = 1.0 / inv
        g = [*(np.asarray(g[:3]) - w).tolist(), *inv.tolist()]
        nc = [int(v) + 2 for v in nc]
        hit = _GRID_MEMO[key] = (g, nc, _lib.dbl3(g), _lib.int_arr(nc), nc[0] * nc[1] * nc[2])
    return hit


def cell_grid(lo, hi, halo: float, width: float):
    """Bins over [lo - halo, hi + halo] with every width >= `width` (the build cutoff).

    Returns ({origin[3], inv_width[3]}, [nx, ny, nz]).  Equivalent to the
    reference's bbox bins (mdkk/neighbor.py:88-92) for the candidate set: any
    width >= cutoff with a 27-cell stencil visits every pair within cutoff.
    """
    lo = np.asarray(lo, dtype=np.float64) - halo
    span = (np.asarray(hi, dtype=np.float64) + halo) - lo
    span = span * (1.0 + 1e-12) + 1e-12
    n = np.maximum(1, np.floor(span / width).astype(np.int64))
    inv = n / span
    return [*lo.tolist(), *inv.tolist()], [int(v) for v in n]
