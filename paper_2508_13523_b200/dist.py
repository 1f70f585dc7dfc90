"""One rank per GPU: spatial domain decomposition with NCCL halo exchange.

The distributed counterpart of RankedSystem (mdkk/domain.py:210-354): the
box is tiled by `decompose(box, world_size)` (min-surface bricks,
mdkk/domain.py:98-123) and each process owns ONE brick on its own GPU.
Every step that the reference performs in-process between logical ranks
becomes a neighbour exchange over torch.distributed (NCCL over NVLink on
the B200 box, gloo in the CPU tests):

* exchange_ghosts  (mdkk/domain.py:246-293): halo selection on device, counts
  all-gathered once, then (x + shift, gid, owner index) rows sent to each
  destination and received straight into the ghost rows, ordered by source
  rank then shift — the reference's order;
* forward_comm     (:295-305): pack x[idx] + shift per lane -> send/recv into
  ghost rows (one batched P2P group per step);
* reverse_comm     (:307-322): ghost force rows sent back to their owners and
  folded with FP64 atomics, ghost rows zeroed;
* migrate          (:324-334): wrap, device owner keys, leavers sent to their
  new bricks, arrivals appended in source-rank order, spatial re-sort;
* rebuild decision (mdkk/neighbor.py:230) and energy / KE sums: all_reduce.

Kernel calls go through an `ops` object (the CUDA library by default); the
CPU tests substitute a torch implementation to exercise this host logic with
gloo at world_size 2.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .domain import (SHIFT_UNITS, AtomStore, Box, RankSet, _rows4, _to4, decompose, shell_grid_args,
                     _dense_ids)


def _staged(group) -> bool:
    """gloo moves host memory only: CUDA tensors are staged through the host (single-GPU
    multi-process tests); NCCL (the product path) sends device buffers directly."""
    return dist.get_backend(group) == "gloo"


def _all_reduce(t: torch.Tensor, op, group) -> None:
    if t.is_cuda and _staged(group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)


def _all_gather(out: list, t: torch.Tensor, group) -> None:
    if t.is_cuda and _staged(group):
        hs = [torch.empty_like(o, device="cpu") for o in out]
        dist.all_gather(hs, t.cpu(), group=group)
        for o, h in zip(out, hs):
            o.copy_(h)
    else:
        dist.all_gather(out, t, group=group)


class CudaOps:
    """Kernel entry points of libmdkk_b200 used by the distributed system."""

    def __init__(self, device):
        self.device = device

    def _s(self):
        return _lib.stream(self.device)

    def halo_select(self, x, n, tab, C_, bins=None, lo=None, hi=None):
        """Per-combo ghost selection; with `bins` (the brick's cell sort on the shell grid,
        cells >= the halo wide) only the boundary-layer rows are scanned."""
        lib, ctx = _lib.lib(), _lib.ctx(self.device)
        nb = (n + 255) // 256
        blk = torch.empty(max(nb * C_, 1), dtype=torch.int32, device=self.device)
        tot = torch.empty(max(C_, 1), dtype=torch.int32, device=self.device)
        rp = cp = None
        if bins is not None:
            _, _, _, narr, _ = shell_grid_args(lo, hi, bins[0])
            rows = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
            cnt = torch.empty(1, dtype=torch.int32, device=self.device)
            _lib.check(lib.mdkk_boundary_rows(ctx, bins[2].data_ptr(), narr, 2, rows.data_ptr(), cnt.data_ptr(),
                                              self._s()), "mdkk_boundary_rows")
            rp, cp = rows.data_ptr(), cnt.data_ptr()
        _lib.check(lib.mdkk_halo_count(ctx, x.data_ptr(), n, tab.data_ptr(), C_, blk.data_ptr(), tot.data_ptr(),
                                       rp, cp, self._s()), "mdkk_halo_count")
        totals = tot[:C_].cpu().numpy().astype(np.int64)
        idx = torch.empty(int(totals.sum()) + 1, dtype=torch.int32, device=self.device)
        _lib.check(lib.mdkk_halo_fill(ctx, x.data_ptr(), n, tab.data_ptr(), C_, blk.data_ptr(), tot.data_ptr(),
                                      idx.data_ptr(), None, None, rp, cp, self._s()), "mdkk_halo_fill")
        return idx, totals

    def halo_count(self, x, n, tab, C_, bins=None, lo=None, hi=None):
        """First half of halo_select: per-combo totals stay on the device (the caller reads
        them together with the all-gathered counts matrix: one host sync per exchange)."""
        lib, ctx = _lib.lib(), _lib.ctx(self.device)
        nb = (n + 255) // 256
        blk = torch.empty(max(nb * C_, 1), dtype=torch.int32, device=self.device)
        tot = torch.empty(max(C_, 1), dtype=torch.int32, device=self.device)
        rp = cp = None
        if bins is not None:
            _, _, _, narr, _ = shell_grid_args(lo, hi, bins[0])
            rows = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
            cnt = torch.empty(1, dtype=torch.int32, device=self.device)
            _lib.check(lib.mdkk_boundary_rows(ctx, bins[2].data_ptr(), narr, 2, rows.data_ptr(), cnt.data_ptr(),
                                              self._s()), "mdkk_boundary_rows")
            rp, cp = (rows, cnt)
        _lib.check(lib.mdkk_halo_count(ctx, x.data_ptr(), n, tab.data_ptr(), C_, blk.data_ptr(), tot.data_ptr(),
                                       _lib.ptr(rp), _lib.ptr(cp), self._s()), "mdkk_halo_count")
        return tot[:C_], (blk, rp, cp)

    def halo_fill(self, x, n, tab, C_, tot, state, total):
        lib, ctx = _lib.lib(), _lib.ctx(self.device)
        blk, rp, cp = state
        idx = torch.empty(int(total) + 1, dtype=torch.int32, device=self.device)
        _lib.check(lib.mdkk_halo_fill(ctx, x.data_ptr(), n, tab.data_ptr(), C_, blk.data_ptr(), tot.data_ptr(),
                                      idx.data_ptr(), None, None, _lib.ptr(rp), _lib.ptr(cp), self._s()),
                   "mdkk_halo_fill")
        return idx

    def owner_partition_dev(self, x, n, lengths, grid, R):
        """owner_partition with the bucket starts left on the device."""
        lib, ctx = _lib.lib(), _lib.ctx(self.device)
        keys = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        start = torch.empty(R + 1, dtype=torch.int32, device=self.device)
        order = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        _lib.check(lib.mdkk_rank_keys(x.data_ptr(), n, _lib.dbl3(lengths), _lib.int_arr(grid), keys.data_ptr(),
                                      self._s()), "mdkk_rank_keys")
        _lib.check(lib.mdkk_bucket_sort(ctx, keys.data_ptr(), n, R, start.data_ptr(), order.data_ptr(), self._s()),
                   "mdkk_bucket_sort")
        return start, order

    def pack(self, x, idx, code, shifts, n, out):
        if n:
            _lib.check(_lib.lib().mdkk_pack_shift(x.data_ptr(), idx.data_ptr(), code.data_ptr(), shifts.data_ptr(), n,
                                                  out.data_ptr(), self._s()), "mdkk_pack_shift")

    def fold(self, f, idx, buf, n):
        if n:
            _lib.check(_lib.lib().mdkk_fold_add(f.data_ptr(), idx.data_ptr(), buf.data_ptr(), n, self._s()),
                       "mdkk_fold_add")

    def fold_ordered(self, f, idx, buf, n):
        """As fold, but each owner row takes its contributions one by one in lane order
        (no atomics: the Serial strategy's deterministic reverse comm)."""
        if n:
            from .memspace import ordered_scatter
            ordered_scatter(f, 4, 3, idx[:n].long(), buf[:n, :3].contiguous())

    def gather_rows(self, src, idx, n, out):
        if n:
            _lib.check(_lib.lib().mdkk_gather_rows4(src.data_ptr(), idx.data_ptr(), n, out.data_ptr(), self._s()),
                       "mdkk_gather_rows4")

    def gather_i64(self, src, idx, n, out):
        if n:
            _lib.check(_lib.lib().mdkk_gather_i64(src.data_ptr(), idx.data_ptr(), n, out.data_ptr(), self._s()),
                       "mdkk_gather_i64")

    def wrap(self, x, n, lengths):
        if n:
            _lib.check(_lib.lib().mdkk_wrap(x.data_ptr(), n, _lib.dbl3(lengths), self._s()), "mdkk_wrap")

    def owner_partition(self, x, n, lengths, grid, R):
        """Stable partition of rows by owning brick: (bucket starts on host, order)."""
        lib, ctx = _lib.lib(), _lib.ctx(self.device)
        keys = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        start = torch.empty(R + 1, dtype=torch.int32, device=self.device)
        order = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        _lib.check(lib.mdkk_rank_keys(x.data_ptr(), n, _lib.dbl3(lengths), _lib.int_arr(grid), keys.data_ptr(),
                                      self._s()), "mdkk_rank_keys")
        _lib.check(lib.mdkk_bucket_sort(ctx, keys.data_ptr(), n, R, start.data_ptr(), order.data_ptr(), self._s()),
                   "mdkk_bucket_sort")
        return start.cpu().numpy().astype(np.int64), order

    def cell_order(self, x, n, lo, hi, width):
        """Permutation putting rows in serpentine cell order on the brick's shell grid (its
        cells plus one shell layer: the neighbour build's grid); the bucket starts are kept
        in `last_bins` for the build's ghost-only binning and the boundary-row halo scan."""
        lib, ctx = _lib.lib(), _lib.ctx(self.device)
        _, _, garr, narr, ncell = shell_grid_args(lo, hi, width)
        keys = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        start = torch.empty(ncell + 1, dtype=torch.int32, device=self.device)
        order = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        _lib.check(lib.mdkk_bin_atoms(ctx, x.data_ptr(), n, garr, narr, keys.data_ptr(),
                                      start.data_ptr(), order.data_ptr(), self._s()), "mdkk_bin_atoms")
        self.last_bins = (float(width), n, start)
        return order


class _SendLane:
    __slots__ = ("dst", "idx", "code", "count", "fbuf", "rbuf")

    def __init__(self, dst, idx, code, count):
        self.dst, self.idx, self.code, self.count = dst, idx, code, count
        self.fbuf = self.rbuf = None


class _RecvLane:
    __slots__ = ("src", "start", "count", "codes")

    def __init__(self, src, start, count, codes=None):
        self.src, self.start, self.count, self.codes = src, start, count, codes


class DistSystem:
    """This process's brick of a world-wide decomposition (RankedSystem API, one store)."""

    def __init__(self, box: Box, rankset: RankSet, store: AtomStore, device, group=None, ops=None,
                 n_atoms: int = 0, dense_gids: bool = True):
        self.box = box
        self.rankset = rankset
        self.store = store
        self.stores = [store]
        self.device = torch.device(device)
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.ops = ops or CudaOps(self.device)
        self.n_atoms = n_atoms
        self.dense_gids = dense_gids
        self.halo = 0.0
        self.sort_width = None
        self.send_lanes: list[_SendLane] = []
        self.recv_lanes: list[_RecvLane] = []
        self._shift_dev = torch.from_numpy(SHIFT_UNITS * box.lengths).to(self.device)
        self._combo_cache = {}
        store.lo, store.hi, store._lengths = rankset.lo[store.rank], rankset.hi[store.rank], box.lengths

    @property
    def n_ranks(self) -> int:
        return self.world

    @classmethod
    def distribute(cls, box: Box, positions, velocities, global_ids=None, device=None, group=None, ops=None):
        """Every process passes the same initial arrays and keeps its own brick (mdkk/domain.py:220-235)."""
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
        vel = np.ascontiguousarray(np.asarray(velocities, dtype=np.float64).reshape(-1, 3))
        n = len(pos)
        rs = decompose(box, world)
        ops = ops or CudaOps(device)
        # one upload of the whole input, wrap + stable owner partition on the device
        x, v = _to4(pos, device), _to4(vel, device)
        if global_ids is None:
            dense, gid = True, torch.arange(max(n, 1), dtype=torch.int64, device=device)
        else:
            g_host = np.asarray(global_ids, dtype=np.int64).reshape(-1)
            dense = _dense_ids(g_host, n)
            gid = torch.from_numpy(g_host).to(device) if n else torch.zeros(1, dtype=torch.int64, device=device)
        ops.wrap(x, n, box.lengths)
        start, order = ops.owner_partition(x, n, box.lengths, rs.grid, world)
        a, b = int(start[rank]), int(start[rank + 1])
        c = b - a
        cap = int(c * 1.3) + 64
        xr, vr = _rows4(cap, device), _rows4(c, device)
        gr = torch.zeros(cap, dtype=torch.int64, device=device)
        if c:
            o = order[a:b]
            ops.gather_rows(x, o, c, xr)
            ops.gather_rows(v, o, c, vr)
            ops.gather_i64(gid, o, c, gr)
        store = AtomStore(rank, device, xr, vr, gr, c)
        return cls(box, rs, store, device, group, ops, n, dense)

    # ------------------------------------------------------------ helpers
    def allreduce_max(self, t: torch.Tensor) -> torch.Tensor:
        _all_reduce(t, dist.ReduceOp.MAX, self.group)
        return t

    def allreduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        _all_reduce(t, dist.ReduceOp.SUM, self.group)
        return t

    def _p2p(self, sends, recvs):
        """One batched group of isend/irecv (tensor, peer) pairs; waits for completion."""
        self._p2p_end(self._p2p_begin(sends, recvs))

    def _p2p_begin(self, sends, recvs):
        """Post the batched group; returns what `_p2p_end` completes.  Over NCCL the
        transfers run on NCCL's stream behind the work queued so far, so kernels queued
        before `_p2p_end` overlap them."""
        staged = _staged(self.group) and any(t.is_cuda for t, _ in list(sends) + list(recvs))
        if staged:
            sends = [(t.cpu(), p) for t, p in sends]
            host_recvs = [(torch.empty_like(t, device="cpu"), p) for t, p in recvs]
        else:
            host_recvs = recvs
        ops = [dist.P2POp(dist.isend, t, p, self.group) for t, p in sends if t.numel()]
        ops += [dist.P2POp(dist.irecv, t, p, self.group) for t, p in host_recvs if t.numel()]
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return reqs, (recvs, host_recvs) if staged else None

    def _p2p_end(self, pending) -> None:
        reqs, staged = pending
        for req in reqs:
            req.wait()   # NCCL: the current stream waits for the transfers (no host block)
        if staged:
            recvs, host_recvs = staged
            for (t, _), (h, _) in zip(recvs, host_recvs):
                if t.numel():
                    t.copy_(h)

    def remote_dims(self) -> int:
        """Bit d set when the bricks along d are more than one (ghosts across those faces
        come from other ranks by the exchange; along the others they are periodic
        self-images packed locally)."""
        return sum(1 << d for d in range(3) if int(self.rankset.grid[d]) > 1)

    def cluster_flags(self, nl, halo: float) -> torch.Tensor:
        """Per-cluster boundary flags of `nl` for the halo overlap (mdkk_cluster_flags)."""
        s = self.store
        ncl = (s.n_local + 31) // 32
        fl = getattr(nl, "_part_flags", None)
        if fl is None:
            fl = torch.ones(max(ncl, 1), dtype=torch.uint8, device=self.device)
            _lib.check(_lib.lib().mdkk_cluster_flags(s.x.data_ptr(), s.n_local, _lib.dbl3(s.lo), _lib.dbl3(s.hi),
                                                     float(halo), self.remote_dims(), fl.data_ptr(),
                                                     _lib.stream(self.device)), "mdkk_cluster_flags")
            nl._part_flags = fl
        return fl

    def _counts_matrix(self, mine: np.ndarray) -> np.ndarray:
        """All-gather of every rank's per-destination counts -> [src][dst]."""
        t = torch.as_tensor(mine, dtype=torch.int64, device=self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        _all_gather(out, t, self.group)
        return torch.stack(out).cpu().numpy()

    def _combos(self, halo):
        hit = self._combo_cache.get(halo)
        if hit is None:
            L, rs, src = self.box.lengths, self.rankset, self.rank
            meta, rows = [], []
            for dst in range(self.world):
                lo, hi = rs.lo[dst] - halo, rs.hi[dst] + halo
                for code in range(27):
                    if dst == src and code == 13:
                        continue
                    shift = SHIFT_UNITS[code] * L
                    slo, shi = rs.lo[src] - halo + shift, rs.hi[src] + halo + shift
                    if np.any(shi <= lo) or np.any(slo >= hi):
                        continue
                    meta.append((dst, code))
                    rows.append(np.concatenate([lo, hi, shift]))
            tab = torch.from_numpy(np.array(rows) if rows else np.zeros((0, 9))).to(self.device)
            hit = self._combo_cache[halo] = (meta, tab)
        return hit

    def _combo_dst(self, halo):
        """Destination rank of every halo combo, on the device (cached with the combos)."""
        key = ("dst", halo)
        hit = self._combo_cache.get(key)
        if hit is None:
            meta, _ = self._combos(halo)
            hit = self._combo_cache[key] = torch.tensor([d for d, _ in meta], dtype=torch.int64,
                                                        device=self.device)
        return hit

    # ------------------------------------------------------------ ghosts
    def exchange_ghosts(self, halo: float) -> None:
        from .domain import DomainError
        if halo <= 0 or halo > 0.5 * self.box.min_periodic_length():
            raise DomainError(f"invalid halo {halo} for box {self.box.lengths.tolist()}")
        self.halo = float(halo)
        s = self.store
        s.to_device()
        meta, tab = self._combos(halo)
        C_ = len(meta)
        per_dst = np.zeros(self.world, dtype=np.int64)
        self.send_lanes = []
        bins = getattr(s, "_bins", None)
        sorted_rows = isinstance(self.ops, CudaOps) and bins is not None and bins[1] == s.n_local and bins[0] >= halo
        M = None
        if hasattr(self.ops, "halo_count"):
            # device totals -> per-destination counts -> all-gather, then ONE host read-back of
            # both (the totals size the index buffer, the matrix sizes the receives)
            if C_ and s.n_local:
                tot, hstate = (self.ops.halo_count(s.x, s.n_local, tab, C_, bins=bins, lo=s.lo, hi=s.hi)
                               if sorted_rows else self.ops.halo_count(s.x, s.n_local, tab, C_))
            else:
                tot = torch.zeros(C_, dtype=torch.int32, device=self.device)
            per = torch.zeros(self.world, dtype=torch.int64, device=self.device)
            if C_:
                per.index_add_(0, self._combo_dst(halo), tot.long())
            out = [torch.empty_like(per) for _ in range(self.world)]
            _all_gather(out, per, self.group)
            host = torch.cat([tot.long(), torch.stack(out).flatten()]).cpu().numpy()
            totals, M = host[:C_], host[C_:].reshape(self.world, self.world)
            idx = (self.ops.halo_fill(s.x, s.n_local, tab, C_, tot, hstate, int(totals.sum()))
                   if C_ and s.n_local else None)
        elif C_ and s.n_local:
            idx, totals = self.ops.halo_select(s.x, s.n_local, tab, C_)
        if C_ and s.n_local:
            start = np.concatenate([[0], np.cumsum(totals)])
            d_of = np.array([d for d, _ in meta])
            codes_all = np.array([c for _, c in meta], dtype=np.int8)
            for d in range(self.world):
                ks = np.flatnonzero(d_of == d)
                if not len(ks):
                    continue
                a, b = int(start[ks[0]]), int(start[ks[-1] + 1])
                if b > a:
                    code = torch.from_numpy(np.repeat(codes_all[ks], totals[ks])).to(self.device)
                    self.send_lanes.append(_SendLane(d, idx[a:b], code, b - a))
                    per_dst[d] = b - a
        if M is None:
            M = self._counts_matrix(per_dst)      # M[src][dst]
        recv = M[:, self.rank]
        nl, ng = s.n_local, int(recv.sum())
        s.ensure_capacity(nl + ng)
        s.n_ghost = ng
        self.recv_lanes = []
        cur = nl
        for src in range(self.world):
            if recv[src]:
                self.recv_lanes.append(_RecvLane(src, cur, int(recv[src])))
                s.orank[cur:cur + recv[src]] = src
                cur += int(recv[src])
        # payload: x rows (+shift), gid, owner index
        sends, recvs = [], []
        for ln in self.send_lanes:
            if ln.dst == self.rank:
                continue
            bx = torch.empty((ln.count, 4), dtype=torch.float64, device=self.device)
            self.ops.pack(s.x, ln.idx, ln.code, self._shift_dev, ln.count, bx)
            bg = torch.empty(ln.count, dtype=torch.int64, device=self.device)
            self.ops.gather_i64(s.gid, ln.idx, ln.count, bg)
            sends += [(bx, ln.dst), (bg, ln.dst), (ln.idx.contiguous(), ln.dst), (ln.code.to(torch.int32), ln.dst)]
        codes_in = {}
        for ln in self.recv_lanes:
            if ln.src == self.rank:
                continue
            sl = slice(ln.start, ln.start + ln.count)
            codes_in[ln.src] = torch.empty(ln.count, dtype=torch.int32, device=self.device)
            recvs += [(s.x[sl], ln.src), (s.gid[sl], ln.src), (s.oidx[sl], ln.src), (codes_in[ln.src], ln.src)]
        # local lane (periodic self-images) straight into the ghost rows
        for ln in self.send_lanes:
            if ln.dst == self.rank:
                rl = next(r for r in self.recv_lanes if r.src == self.rank)
                self.ops.pack(s.x, ln.idx, ln.code, self._shift_dev, ln.count, s.x[rl.start:])
                self.ops.gather_i64(s.gid, ln.idx, ln.count, s.gid[rl.start:])
                s.oidx[rl.start:rl.start + ln.count] = ln.idx
                rl.codes = ln.code
        self._p2p(sends, recvs)
        for ln in self.recv_lanes:
            if ln.src in codes_in:
                ln.codes = codes_in[ln.src].to(torch.int8)
        s._lanes_in = [_CodeView(ln) for ln in self.recv_lanes]
        if nl:
            s.orank[:nl] = self.rank
        # per-step communication buffers, allocated once per exchange: a remote send lane's
        # packed positions (forward) and the ghost forces it gets back (reverse)
        for ln in self.send_lanes:
            if ln.dst != self.rank:
                ln.fbuf = torch.empty((ln.count, 4), dtype=torch.float64, device=self.device)
                ln.rbuf = torch.empty((ln.count, 4), dtype=torch.float64, device=self.device)
        s._views()
        s.device_wrote(pos=True)

    def forward_comm(self) -> None:
        """ghost x = owner x + shift: pack -> NCCL send/recv into ghost rows (mdkk/domain.py:295-305)."""
        self.forward_comm_end(self.forward_comm_begin())

    def forward_comm_end(self, pending) -> None:
        self._p2p_end(pending)
        if self.store.n_ghost:
            self.store.device_wrote(pos=True)

    def forward_comm_begin(self):
        """Pack and post the halo exchange; `forward_comm_end` completes it (kernels
        queued in between overlap the transfers)."""
        s = self.store
        s.to_device()
        sends, recvs = [], []
        for ln in self.send_lanes:
            if ln.dst == self.rank:
                rl = next(r for r in self.recv_lanes if r.src == self.rank)
                self.ops.pack(s.x, ln.idx, ln.code, self._shift_dev, ln.count, s.x[rl.start:])
            else:
                self.ops.pack(s.x, ln.idx, ln.code, self._shift_dev, ln.count, ln.fbuf)
                sends.append((ln.fbuf, ln.dst))
        for ln in self.recv_lanes:
            if ln.src != self.rank:
                recvs.append((s.x[ln.start:ln.start + ln.count], ln.src))
        return self._p2p_begin(sends, recvs)

    def reverse_comm(self, ordered: bool = False) -> None:
        """Ghost forces back to owners, folded with atomics; ghost rows zeroed (mdkk/domain.py:307-322).
        `ordered` (the Serial strategy): a deterministic ordered fold instead of atomics."""
        s = self.store
        s.to_device()
        fold = self.ops.fold_ordered if ordered and hasattr(self.ops, "fold_ordered") else self.ops.fold
        sends, recvs, folds = [], [], []
        for ln in self.recv_lanes:
            if ln.src != self.rank:
                sends.append((s.f[ln.start:ln.start + ln.count].contiguous(), ln.src))
        for ln in self.send_lanes:
            if ln.dst == self.rank:
                rl = next(r for r in self.recv_lanes if r.src == self.rank)
                fold(s.f, ln.idx, s.f[rl.start:], ln.count)
            else:
                recvs.append((ln.rbuf, ln.dst))
                folds.append((ln, ln.rbuf))
        self._p2p(sends, recvs)
        for ln, buf in folds:
            fold(s.f, ln.idx, buf, ln.count)
        if s.n_ghost:
            s.f[s.n_local:s.n_total].zero_()
        s.device_wrote(force=True)

    # ----------------------------------------------------------- migration
    def migrate(self, halo: float, sort_width: float | None = None, zero_forces: bool = True,
                ref_out=None) -> bool:
        """Wrap, send leavers to their bricks, append arrivals, re-sort, rebuild ghosts (mdkk/domain.py:324-334).
        `ref_out` is the one-rank engine hint of RankedSystem.migrate (not used here: returns False)."""
        s = self.store
        s.to_device()
        nl = s.n_local
        self.ops.wrap(s.x, nl, self.box.lengths)
        if hasattr(self.ops, "owner_partition_dev"):
            # bucket starts and the all-gathered counts matrix in one host read-back
            st_dev, order = self.ops.owner_partition_dev(s.x, nl, self.box.lengths, self.rankset.grid, self.world)
            cnt = (st_dev[1:] - st_dev[:-1]).long()
            out = [torch.empty_like(cnt) for _ in range(self.world)]
            _all_gather(out, cnt, self.group)
            host = torch.cat([st_dev.long(), torch.stack(out).flatten()]).cpu().numpy()
            start, M = host[: self.world + 1], host[self.world + 1:].reshape(self.world, self.world)
        else:
            start, order = self.ops.owner_partition(s.x, nl, self.box.lengths, self.rankset.grid, self.world)
            M = self._counts_matrix(np.diff(start))
        arrivals = M[:, self.rank]
        n_new = int(arrivals.sum())
        cap = max(s.capacity, int(n_new * 1.3) + 64)
        x = _rows4(cap, self.device, zero=False)
        v = _rows4(max(n_new, 1), self.device, zero=False)
        gid = torch.empty(cap, dtype=torch.int64, device=self.device)
        # arrivals laid out in source-rank order (own stayers at this rank's slot)
        offs = np.concatenate([[0], np.cumsum(arrivals)])
        sends, recvs = [], []
        for d in range(self.world):
            a, b = int(start[d]), int(start[d + 1])
            if b == a:
                continue
            seg = order[a:b]
            if d == self.rank:
                o = int(offs[self.rank])
                self.ops.gather_rows(s.x, seg, b - a, x[o:])
                self.ops.gather_rows(s.v, seg, b - a, v[o:])
                self.ops.gather_i64(s.gid, seg, b - a, gid[o:])
                continue
            bx = torch.empty((b - a, 4), dtype=torch.float64, device=self.device)
            bv = torch.empty((b - a, 4), dtype=torch.float64, device=self.device)
            bg = torch.empty(b - a, dtype=torch.int64, device=self.device)
            self.ops.gather_rows(s.x, seg, b - a, bx)
            self.ops.gather_rows(s.v, seg, b - a, bv)
            self.ops.gather_i64(s.gid, seg, b - a, bg)
            sends += [(bx, d), (bv, d), (bg, d)]
        for src in range(self.world):
            c = int(arrivals[src])
            if c and src != self.rank:
                o = int(offs[src])
                recvs += [(x[o:o + c], src), (v[o:o + c], src), (gid[o:o + c], src)]
        self._p2p(sends, recvs)
        st = AtomStore(self.rank, self.device, x, v, gid, n_new)
        st.lo, st.hi, st._lengths = s.lo, s.hi, s._lengths
        self.store = st
        self.stores = [st]
        w = sort_width or self.sort_width
        if w:
            self._sort(w)
        st._views()
        st.device_wrote(pos=True, vel=True, force=True)
        self.exchange_ghosts(halo)
        if zero_forces:
            st.f[: st.n_total].zero_()

    def _sort(self, width: float) -> None:
        s = self.store
        n = s.n_local
        if n < 2:
            return
        order = self.ops.cell_order(s.x, n, s.lo, s.hi, width)
        x = _rows4(s.capacity, self.device, zero=False)
        v = _rows4(max(n, 1), self.device, zero=False)
        g = torch.empty(s.capacity, dtype=torch.int64, device=self.device)
        self.ops.gather_rows(s.x, order, n, x)
        self.ops.gather_rows(s.v, order, n, v)
        self.ops.gather_i64(s.gid, order, n, g)
        s.x, s.v, s.gid = x, v, g
        s._bins = getattr(self.ops, "last_bins", None)   # owned rows now sorted on the shell grid

    def sort_local(self, width: float) -> None:
        s = self.store
        s.to_device()
        s.n_ghost = 0
        self._sort(width)
        s._views()
        s.device_wrote(pos=True, vel=True, force=True)

    # -------------------------------------------------------------- gather
    def _gather_rows(self, t: torch.Tensor, width: int):
        s = self.store
        n = torch.tensor([s.n_local], dtype=torch.int64, device=self.device)
        ns = [torch.empty_like(n) for _ in range(self.world)]
        _all_gather(ns, n, self.group)
        ns = [int(v.item()) for v in ns]
        m = max(ns) if ns else 0
        rows = torch.zeros((max(m, 1), width), dtype=t.dtype, device=self.device)
        rows[: s.n_local] = t[: s.n_local, :width]
        gid = torch.full((max(m, 1),), -1, dtype=torch.int64, device=self.device)
        gid[: s.n_local] = s.gid[: s.n_local]
        R = [torch.empty_like(rows) for _ in range(self.world)]
        G = [torch.empty_like(gid) for _ in range(self.world)]
        _all_gather(R, rows, self.group)
        _all_gather(G, gid, self.group)
        if self.dense_gids and sum(ns) == self.n_atoms:
            # gids are 0..N-1: place rows by gid on the device, one read-back
            out = torch.empty((max(self.n_atoms, 1), width), dtype=t.dtype, device=self.device)
            for r, g, k in zip(R, G, ns):
                if k:
                    out[g[:k]] = r[:k]
            return out[: self.n_atoms].cpu().numpy(), np.arange(self.n_atoms, dtype=np.int64)
        rows = np.concatenate([r[:k].cpu().numpy() for r, k in zip(R, ns)])
        gids = np.concatenate([g[:k].cpu().numpy() for g, k in zip(G, ns)])
        o = np.argsort(gids, kind="stable")
        return rows[o], gids[o]

    def gather(self):
        """(pos, vel, gid) of all ranks' owned atoms in global-id order, on every rank (mdkk/domain.py:336-342)."""
        self.store.to_device()
        pos, gid = self._gather_rows(self.store.x, 3)
        vel, _ = self._gather_rows(self.store.v, 3)
        return pos, vel, gid

    def gather_positions(self) -> np.ndarray:
        self.store.to_device()
        return self._gather_rows(self.store.x, 3)[0]

    def gather_positions_async(self):
        """The collective gather runs now (every rank must take part at the same step)."""
        pos = self.gather_positions()
        return lambda: pos

    def gather_forces(self) -> np.ndarray:
        self.store.force.sync("b")
        f, _ = self._gather_rows(self.store.f, 3)
        return f

    def zero_forces(self) -> None:
        s = self.store
        s.force.sync("b")
        s.f.zero_()
        s.device_wrote(force=True)


class _CodeView:
    """Adapter so AtomStore.ghost_shift can read a receive lane's shift codes."""

    def __init__(self, ln: _RecvLane):
        self.start, self.count = ln.start, ln.count
        self.code = ln.codes if ln.codes is not None else torch.zeros(ln.count, dtype=torch.int8)
