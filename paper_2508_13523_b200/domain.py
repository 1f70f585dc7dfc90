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

import ctypes as C
import itertools
import math

import numpy as np
import torch

from . import _lib
from .memspace import DualArray


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


def _rows4(n: int, device) -> torch.Tensor:
    return torch.zeros((max(n, 1), 4), dtype=torch.float64, device=device)


def _to4(a: np.ndarray, device) -> torch.Tensor:
    t = _rows4(len(a), device)
    if len(a):
        t[: len(a), :3] = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)
    return t


class AtomStore:
    """One rank's rows in HBM: n_local owned rows followed by n_ghost ghosts (mdkk/domain.py:126-193).

    Device tensors: ``x``/``f`` (n_total, 4) f64, ``v`` (n_local, 4) f64,
    ``gid`` int64, ``orank``/``oidx`` int32 per row, ``gcode`` int8 shift code
    per ghost.  ``pos``/``vel``/``force`` are DualArray views over them
    (space "a" = host numpy, "b" = these tensors).
    """

    def __init__(self, rank: int, device, x: torch.Tensor, v: torch.Tensor, gid: torch.Tensor, n_local: int):
        self.rank = int(rank)
        self.device = torch.device(device)
        self.n_local = int(n_local)
        self.n_ghost = 0
        self.gid = gid
        self.orank = torch.full((max(n_local, 1),), self.rank, dtype=torch.int32, device=self.device)
        self.oidx = torch.arange(max(n_local, 1), dtype=torch.int32, device=self.device)
        self.gcode = torch.zeros(0, dtype=torch.int8, device=self.device)
        self._adopt(x, v, torch.zeros_like(x))
        self.lo = self.hi = None  # brick bounds, set by RankedSystem
        self._host_cache = {}

    # -- DualArray plumbing (mdkk/memspace.py protocol) ----------------------
    def _adopt(self, x, v, f):
        self.x, self.v, self.f = x, v, f
        nt = max(self.n_total, 1)
        self.pos = DualArray((nt, 3), device=self.device, pad_last=4, storage_b=x,
                             layout_b=_ROW)
        self.vel = DualArray((max(self.n_local, 1), 3), device=self.device, pad_last=4, storage_b=v,
                             layout_b=_ROW)
        self.force = DualArray((nt, 3), device=self.device, pad_last=4, storage_b=f, layout_b=_ROW)
        self._host_cache = {}

    def to_device(self):
        """Make device storage current before a kernel reads it."""
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
            s = np.zeros((self.n_total, 3))
            if self.n_ghost:
                s[self.n_local:] = SHIFT_UNITS[self.gcode.cpu().numpy().astype(np.int64)] * self._lengths
            h = self._host_cache["shift"] = s
        return h


_ROW = None  # set below (row-major device layout for (n, 3) padded rows)


def _init_layout():
    global _ROW
    from .memspace import LayoutPolicy
    _ROW = LayoutPolicy.row_major(2)


_init_layout()


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
        self.sort_width = None  # spatial-sort bin width (set by the first neighbour build)
        for s in stores:
            s.lo, s.hi = rankset.lo[s.rank], rankset.hi[s.rank]
            s._lengths = box.lengths

    @property
    def n_ranks(self) -> int:
        return self.rankset.n_ranks

    @classmethod
    def distribute(cls, box: Box, n_ranks: int, positions, velocities, global_ids=None,
                   device=None) -> "RankedSystem":
        """Wrap, assign owners, upload (mdkk/domain.py:220-235).  Setup is host-side, as in the reference."""
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        pos = wrap_positions(np.asarray(positions, dtype=np.float64).reshape(-1, 3), box)
        vel = np.asarray(velocities, dtype=np.float64).reshape(-1, 3)
        n = len(pos)
        gids = np.arange(n, dtype=np.int64) if global_ids is None else np.asarray(global_ids, dtype=np.int64)
        dense = bool(n == 0 or (gids.min() == 0 and gids.max() == n - 1 and len(np.unique(gids)) == n))
        rs = decompose(box, n_ranks)
        owner = rs.rank_of(pos)
        stores = []
        for r in range(rs.n_ranks):
            sel = np.flatnonzero(owner == r)
            g = torch.zeros(max(len(sel), 1), dtype=torch.int64, device=device)
            if len(sel):
                g[: len(sel)] = torch.from_numpy(gids[sel]).to(device)
            stores.append(AtomStore(r, device, _to4(pos[sel], device), _to4(vel[sel], device), g, len(sel)))
        return cls(box, rs, stores, device, dense)

    # ------------------------------------------------------------ ghosts
    def _combos(self, src: int, halo: float):
        """(dst, code, lo, hi, shift) combos for src, dst-major then shift order (mdkk/domain.py:263-271)."""
        L = self.box.lengths
        rs = self.rankset
        out = []
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
                out.append((dst, code, lo, hi, shift))
        return out

    def exchange_ghosts(self, halo: float) -> None:
        """Select ghosts on device and rebuild ghost rows + lanes (mdkk/domain.py:246-293)."""
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
        # per src: selected indices per combo
        sel = {}  # (src, dst) -> list of (code, idx_tensor_view, count)
        for src in self.stores:
            combos = self._combos(src.rank, halo)
            C_ = len(combos)
            if C_ == 0 or src.n_local == 0:
                continue
            tab = np.array([np.concatenate([lo, hi, sh]) for (_, _, lo, hi, sh) in combos])
            tab_dev = torch.from_numpy(tab).to(self.device)
            nb = (src.n_local + 255) // 256
            blk = torch.empty(nb * C_, dtype=torch.int32, device=self.device)
            tot = torch.empty(C_, dtype=torch.int32, device=self.device)
            _lib.check(lib.mdkk_halo_count(ctx, src.x.data_ptr(), src.n_local, tab_dev.data_ptr(), C_,
                                           blk.data_ptr(), tot.data_ptr(), stream), "mdkk_halo_count")
            totals = tot.cpu().numpy()
            idx = torch.empty(max(int(totals.sum()), 1), dtype=torch.int32, device=self.device)
            _lib.check(lib.mdkk_halo_fill(ctx, src.x.data_ptr(), src.n_local, tab_dev.data_ptr(), C_,
                                          blk.data_ptr(), tot.data_ptr(), idx.data_ptr(), stream),
                       "mdkk_halo_fill")
            off = 0
            for (dst, code, _, _, _), t in zip(combos, totals):
                if t:
                    sel.setdefault((src.rank, dst), []).append((code, idx[off:off + t], int(t)))
                off += int(t)
        self.lanes = []
        for dst in self.stores:
            nl = dst.n_local
            parts = []
            for src in range(self.n_ranks):
                for code, ix, t in sel.get((src, dst.rank), []):
                    parts.append((src, code, ix, t))
            ng = sum(p[3] for p in parts)
            x = _rows4(nl + ng, self.device)
            x[:nl] = dst.x[:nl]
            gid = torch.empty(max(nl + ng, 1), dtype=torch.int64, device=self.device)
            gid[:nl] = dst.gid[:nl]
            orank = torch.empty(max(nl + ng, 1), dtype=torch.int32, device=self.device)
            orank[:nl] = self.stores[dst.rank].rank
            oidx = torch.empty(max(nl + ng, 1), dtype=torch.int32, device=self.device)
            oidx[:nl] = torch.arange(nl, dtype=torch.int32, device=self.device)
            codes = np.zeros(ng, dtype=np.int8)
            cur = nl
            lane_src, lane_start, lane_parts = None, 0, []
            for src, code, ix, t in parts:
                codes[cur - nl:cur - nl + t] = code
                orank[cur:cur + t] = src
                oidx[cur:cur + t] = ix
                sst = self.stores[src]
                _lib.check(lib.mdkk_gather_i64(sst.gid.data_ptr(), ix.data_ptr(), t,
                                               gid[cur:].data_ptr(), stream), "mdkk_gather_i64")
                if src != lane_src:
                    if lane_parts:
                        self._add_lane(lane_src, dst.rank, lane_parts, lane_start)
                    lane_src, lane_start, lane_parts = src, cur, []
                lane_parts.append((code, ix, t))
                cur += t
            if lane_parts:
                self._add_lane(lane_src, dst.rank, lane_parts, lane_start)
            gcode = torch.from_numpy(codes).to(self.device)
            v = dst.v
            dst.n_ghost = ng
            dst.gid, dst.orank, dst.oidx, dst.gcode = gid, orank, oidx, gcode
            dst._adopt(x, v, torch.zeros_like(x))
        self._pack_all()
        for s in self.stores:
            s.device_wrote(pos=True)

    def _add_lane(self, src, dst, parts, start):
        idx = torch.cat([p[1] for p in parts]) if len(parts) > 1 else parts[0][1]
        count = sum(p[2] for p in parts)
        code = torch.from_numpy(np.concatenate([np.full(p[2], p[0], np.int8) for p in parts])).to(self.device)
        self.lanes.append(_Lane(src, dst, idx, code, start, count))

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

    def reverse_comm(self) -> None:
        """Fold ghost forces onto owners, zero ghost rows (mdkk/domain.py:307-322)."""
        lib, stream = _lib.lib(), _lib.stream(self.device)
        for s in self.stores:
            s.to_device()
        for ln in self.lanes:
            s, d = self.stores[ln.src], self.stores[ln.dst]
            _lib.check(lib.mdkk_fold_add(s.f.data_ptr(), ln.idx.data_ptr(), d.f[ln.start:].data_ptr(),
                                         ln.count, stream), "mdkk_fold_add")
        for s in self.stores:
            if s.n_ghost:
                s.f[s.n_local:s.n_total].zero_()
            s.device_wrote(force=True)

    # ----------------------------------------------------------- migration
    def migrate(self, halo: float, sort_width: float | None = None) -> None:
        """Wrap, reassign bricks, re-sort spatially, zero forces, rebuild ghosts (mdkk/domain.py:324-334)."""
        lib, stream = _lib.lib(), _lib.stream(self.device)
        ctx = _lib.ctx(self.device)
        L = _lib.dbl3(self.box.lengths)
        grid = _lib.int_arr(self.rankset.grid)
        R = self.n_ranks
        for s in self.stores:
            s.to_device()
            _lib.check(lib.mdkk_wrap(s.x.data_ptr(), s.n_local, L, stream), "mdkk_wrap")
        if R > 1:
            parts = {}  # dst -> list of (src, order segment)
            for s in self.stores:
                keys = torch.empty(max(s.n_local, 1), dtype=torch.int32, device=self.device)
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
                x, v = _rows4(n, self.device), _rows4(n, self.device)
                gid = torch.zeros(max(n, 1), dtype=torch.int64, device=self.device)
                cur = 0
                for s, o, c in segs:
                    _lib.check(lib.mdkk_gather_rows4(s.x.data_ptr(), o.data_ptr(), c, x[cur:].data_ptr(), stream), "g4")
                    _lib.check(lib.mdkk_gather_rows4(s.v.data_ptr(), o.data_ptr(), c, v[cur:].data_ptr(), stream), "g4")
                    _lib.check(lib.mdkk_gather_i64(s.gid.data_ptr(), o.data_ptr(), c, gid[cur:].data_ptr(), stream), "g64")
                    cur += c
                st = AtomStore(d, self.device, x, v, gid, n)
                st.lo, st.hi, st._lengths = self.rankset.lo[d], self.rankset.hi[d], self.box.lengths
                new.append(st)
            self.stores = new
        else:
            s = self.stores[0]
            st = AtomStore(0, self.device, s.x[: max(s.n_local, 1)].clone(), s.v, s.gid[: max(s.n_local, 1)].clone(),
                           s.n_local)
            st.lo, st.hi, st._lengths = s.lo, s.hi, s._lengths
            self.stores = [st]
        w = sort_width or self.sort_width
        if w:
            for s in self.stores:
                self._spatial_sort(s, w, halo)
        for s in self.stores:
            s.device_wrote(pos=True, vel=True, force=True)
        self.exchange_ghosts(halo)

    def sort_local(self, width: float) -> None:
        """Re-order every rank's owned rows into serpentine cell order (drops ghosts; call before exchange)."""
        for s in self.stores:
            s.to_device()
            s.n_ghost = 0
            self._spatial_sort(s, width, width)
            s.device_wrote(pos=True, vel=True, force=True)
        self.lanes = []

    def _spatial_sort(self, s: AtomStore, width: float, halo: float):
        """Reorder owned rows by cell so neighbour gathers are local (rows are re-indexed, gids travel)."""
        if s.n_local < 2:
            return
        lib, stream = _lib.lib(), _lib.stream(self.device)
        ctx = _lib.ctx(self.device)
        g, nc = cell_grid(s.lo, s.hi, halo, width)
        ncell = nc[0] * nc[1] * nc[2]
        keys = torch.empty(s.n_local, dtype=torch.int32, device=self.device)
        start = torch.empty(ncell + 1, dtype=torch.int32, device=self.device)
        order = torch.empty(s.n_local, dtype=torch.int32, device=self.device)
        _lib.check(lib.mdkk_bin_atoms(ctx, s.x.data_ptr(), s.n_local, _lib.dbl3(g), _lib.int_arr(nc),
                                      keys.data_ptr(), start.data_ptr(), order.data_ptr(), stream), "bin")
        x, v = _rows4(s.n_local, self.device), _rows4(s.n_local, self.device)
        gid = torch.empty(s.n_local, dtype=torch.int64, device=self.device)
        _lib.check(lib.mdkk_gather_rows4(s.x.data_ptr(), order.data_ptr(), s.n_local, x.data_ptr(), stream), "g4")
        _lib.check(lib.mdkk_gather_rows4(s.v.data_ptr(), order.data_ptr(), s.n_local, v.data_ptr(), stream), "g4")
        _lib.check(lib.mdkk_gather_i64(s.gid.data_ptr(), order.data_ptr(), s.n_local, gid.data_ptr(), stream), "g64")
        s.gid = gid
        s.orank = torch.full((s.n_local,), s.rank, dtype=torch.int32, device=self.device)
        s.oidx = torch.arange(s.n_local, dtype=torch.int32, device=self.device)
        s._adopt(x, v, torch.zeros_like(x))

    # -------------------------------------------------------------- gather
    def _gid_order(self, rows_fn, width):
        """Owned rows of all ranks in global-id order (device scatter when gids are 0..N-1)."""
        n = self.n_atoms
        if self.dense_gids:
            lib, stream = _lib.lib(), _lib.stream(self.device)
            out = _rows4(n, self.device)
            for s in self.stores:
                if s.n_local:
                    gi = s.gid[: s.n_local].to(torch.int32)
                    _lib.check(lib.mdkk_scatter_rows4(rows_fn(s).data_ptr(), gi.data_ptr(), s.n_local,
                                                      out.data_ptr(), stream), "scatter")
            return out[:n, :width].cpu().numpy()
        rows = np.concatenate([rows_fn(s)[: s.n_local, :width].cpu().numpy() for s in self.stores])
        gid = np.concatenate([s.global_ids[: s.n_local] for s in self.stores])
        return rows[np.argsort(gid, kind="stable")]

    def gather(self):
        """(pos, vel, gid) of owned atoms in global-id order (mdkk/domain.py:336-342)."""
        for s in self.stores:
            s.to_device()
        pos = self._gid_order(lambda s: s.x, 3)
        vel = self._gid_order(lambda s: s.v, 3)
        gid = np.sort(np.concatenate([s.global_ids[: s.n_local] for s in self.stores]), kind="stable")
        return pos, vel, gid

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
