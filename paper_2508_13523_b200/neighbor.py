"""Cell-list neighbour lists built on the GPU (drop-in for mdkk/neighbor.py).

`build` / `build_all` / `any_needs_rebuild` / `NeighborList` keep the
reference signatures (mdkk/neighbor.py:38-231).  The list lives in HBM as an
int32 table [cap][n_local] (atom index fastest — the reference's transposed
`layout_b`) plus counts; rows are produced in stencil order for the force
kernels, and `pairs()` returns the reference's canonical (row, partner gid,
z, y, x) order by sorting rows on device before the copy to host.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .domain import AtomStore, Box, RankedSystem, grid_args, shell_grid_args
from .memspace import DualArray, LayoutPolicy

DEFAULT_CAPACITY = 16
STYLES = {"full": 0, "half": 1}


class NeighborError(RuntimeError):
    pass


class StaleListError(NeighborError):
    """A neighbor list was used after atoms moved beyond the skin criterion."""


def grow_capacity(capacity: int, needed: int) -> int:
    """The reference's growth sequence: ceil(cap * 1.5) until >= needed (mdkk/neighbor.py:199-205)."""
    cap = max(int(capacity), 1)
    while cap < needed:
        cap = int(np.ceil(cap * 1.5))
    return cap


class NeighborList:
    """Device neighbour table + counts (mdkk/neighbor.py:38-80).

    `table_dev` is int32 cluster-blocked [ceil(n_local/32)][alloc_cap][32]
    (atom fastest within 32-row tiles — the reference's transposed layout_b);
    entries beyond counts[i] are undefined on device and -1 in the `table`
    DualArray view.
    """

    def __init__(self, store: AtomStore, style: str, newton: bool, cutoff: float, skin: float,
                 cap: int, table: torch.Tensor, counts: torch.Tensor, max_count: int, ref_buf=None,
                 ref_ready: bool = False):
        self.store = store
        self.style = style
        self.newton = bool(newton)
        self.cutoff = float(cutoff)
        self.skin = float(skin)
        self.n_local = store.n_local
        self.max_neighbors = int(cap)          # reference growth sequence from `capacity`
        self.alloc_cap = int(table.shape[1])   # physical slots per row (>= max_count)
        self.max_count = int(max_count)
        self.table_dev = table
        self.counts_dev = counts
        if ref_ready:   # the caller already holds the build-time positions in ref_buf
            self.ref_dev = ref_buf[: max(store.n_local, 1)]
        else:
            self.ref_dev = store.x[: max(store.n_local, 1)].clone() if ref_buf is None else _ref_into(ref_buf, store)
        self._d2 = torch.empty(1, dtype=torch.float64, device=store.device)   # written before every read
        self._pairs = None
        self._pending = None   # deferred capacity check: (device max count, build args)

    @property
    def pending(self) -> bool:
        return self._pending is not None

    def settle(self) -> "tuple[NeighborList, bool]":
        """Complete a deferred build (`build(..., defer=True)`): read the max count
        (one sync).  Returns (list, True) when the table held every row, else a
        list rebuilt with the grown capacity and False (a force launch gated on
        this list's count was a no-op and must be repeated)."""
        if self._pending is None:
            return self, True
        mc, box, capacity, pin, ready = self._pending
        self._pending = None
        ready.synchronize()
        need = int(pin[0])
        if need <= self.alloc_cap:
            self.max_count = need
            self.max_neighbors = grow_capacity(capacity, need)
            return self, True
        nl = build(self.store, box, self.cutoff, self.skin, self.style, self.newton, capacity,
                   cap_hint=grow_capacity(self.alloc_cap, need), recycle=self, rebin=False)
        return nl, False

    @property
    def build_cutoff(self) -> float:
        return self.cutoff + self.skin

    @property
    def counts(self) -> np.ndarray:
        return self.counts_dev[: self.n_local].cpu().numpy()

    def expanded(self, cap: int | None = None) -> torch.Tensor:
        """int32 [cap][n_local] table, -1 padded (device copy)."""
        cap = cap or self.max_neighbors
        ncl = self.table_dev.shape[0]
        t = self.table_dev.permute(1, 0, 2).reshape(self.alloc_cap, ncl * 32)[:cap, : max(self.n_local, 1)]
        t = t.contiguous()
        if self.n_local:
            k = torch.arange(cap, device=t.device)[:, None]
            t[:, : self.n_local][k >= self.counts_dev[None, : self.n_local]] = -1
        else:
            t.fill_(-1)
        return t

    @property
    def table(self) -> DualArray:
        """(n_local, cap) int32 DualArray, -1 padded; device storage [cap][n_local] (layout_b transposed)."""
        t = self.expanded()
        n = max(self.n_local, 1)
        d = DualArray((n, self.max_neighbors), layout_b=LayoutPolicy.transposed(2), dtype=np.int32,
                      device=t.device, storage_b=t)
        d.mark_modified("b")
        return d

    def pairs(self):
        """Directed entries (rows, cols, weight, write_j) in canonical order (mdkk/neighbor.py:62-64,192-197)."""
        if self._pairs is None:
            self._pairs = self._host_pairs()
        return self._pairs

    def _host_pairs(self):
        st = self.store
        n = self.n_local
        if n == 0:
            z = np.zeros(0, np.int64)
            return z, z, np.zeros(0), np.zeros(0, bool)
        cap = self.max_neighbors
        t = self.expanded(cap)
        st.to_device()
        _lib.call("mdkk_nbr_canonicalize", st.x.data_ptr(), st.gid.data_ptr(), n, cap, t.data_ptr(),
                  self.counts_dev.data_ptr(), _lib.stream(st.device))
        tab = t[:, :n].cpu().numpy().T
        cnt = self.counts
        rows = np.repeat(np.arange(n, dtype=np.int64), cnt)
        cols = tab[np.arange(cap)[None, :] < cnt[:, None]].astype(np.int64)
        local = cols < n
        if self.style == "full":
            w, wj = np.full(len(rows), 0.5), np.zeros(len(rows), bool)
        elif self.newton:
            w, wj = np.ones(len(rows)), np.ones(len(rows), bool)
        else:
            w, wj = np.where(local, 1.0, 0.5), local.copy()
        return rows, cols, w, wj

    # -- skin test (mdkk/neighbor.py:66-80) ---------------------------------
    def max_disp2_dev(self) -> torch.Tensor:
        st = self.store
        st.to_device()
        _lib.call("mdkk_max_disp2", st.x.data_ptr(), self.ref_dev.data_ptr(), self.n_local,
                  self._d2.data_ptr(), _lib.stream(st.device))
        return self._d2

    def max_displacement(self) -> float:
        if self.n_local == 0:
            return 0.0
        return math.sqrt(float(self.max_disp2_dev().item()))

    def needs_rebuild(self) -> bool:
        return self.max_displacement() > 0.5 * self.skin

    def check_current(self) -> None:
        if self.needs_rebuild():
            raise StaleListError(
                f"neighbor list stale: max displacement {self.max_displacement():.4g} "
                f"exceeds skin/2 = {0.5 * self.skin:.4g}")


def _ref_into(buf: torch.Tensor, store: AtomStore) -> torch.Tensor:
    n = max(store.n_local, 1)
    if buf.shape[0] < n or buf.device != store.device:
        return store.x[:n].clone()
    out = buf[:n]
    out.copy_(store.x[:n])
    return out


def _recycled(t: torch.Tensor | None, shape, dtype, device) -> torch.Tensor:
    """View of a dead list's storage when it is large enough (engine rebuilds), else a new tensor."""
    if t is not None and t.shape == shape and t.dtype == dtype and t.device == device:
        return t   # the usual engine rebuild: same rows, same capacity (no view ops on the host path)
    numel = 1
    for d in shape:
        numel *= d
    if t is not None and t.dtype == dtype and t.device == device and t.is_contiguous() and t.numel() >= numel:
        return t.reshape(-1)[:numel].view(shape)
    return torch.empty(shape, dtype=dtype, device=device)


class _BuildCache:
    """Per-store reusable device buffers for binning / building."""

    def __init__(self):
        self.bufs = {}
        self.last = None   # ((n_total, bc), (grid args)) of the last binning

    def get(self, name, n, dtype, device):
        t = self.bufs.get(name)
        if t is None or t.numel() < n or t.device != device:
            t = self.bufs[name] = torch.empty(max(int(n * 1.1), 1), dtype=dtype, device=device)
        return t


_cache: dict = {}


def build(store: AtomStore, box: Box, cutoff: float, skin: float, style: str = "full",
          newton: bool = True, capacity: int = DEFAULT_CAPACITY, cap_hint: int | None = None,
          recycle: NeighborList | None = None, defer: bool = False, rebin: bool = True,
          ref_ready: bool = False, **_unused) -> NeighborList:
    """One rank's list from its local + ghost rows (mdkk/neighbor.py:182-219).

    Owned rows must be cell-sorted for compact clusters (RankedSystem keeps
    them so); any order is still correct.  `cap_hint`
    (engine-internal) sizes the first launch; the reported `max_neighbors`
    always follows the reference growth sequence from `capacity`.
    `recycle` (engine-internal) is a list that is dead after this call: its
    device buffers are reused instead of allocating a new ~GB table.
    `defer` (engine-internal, with `cap_hint`): one launch, no host sync; the
    capacity check waits for `NeighborList.settle()` so that work gated on the
    device-side count (mdkk_lj_force_gated) can be queued first.
    `rebin=False` (engine-internal, a regrow right after a build of the same rows)
    reuses that build's cell lists, so the table comes out in the same order.
    `ref_ready` (engine-internal, with `recycle`): the recycled list's reference
    buffer already holds the current owned positions (the engine copies them
    while the host is still preparing the build).
    """
    if style not in STYLES:
        raise NeighborError(f"unknown list style {style!r}")
    bc = cutoff + skin
    if bc > 0.5 * box.min_periodic_length():
        raise NeighborError(f"cutoff+skin {bc} exceeds half the shortest periodic box length")
    dev = store.device
    lib, stream = _lib.lib(), _lib.stream(dev)
    ctx = _lib.ctx(dev)
    store.to_device()
    n_local, n_total = store.n_local, store.n_total
    lo = store.lo if store.lo is not None else np.zeros(3)
    hi = store.hi if store.hi is not None else box.lengths
    bins = getattr(store, "_bins", None)
    merged = bins is not None and bins[0] == bc and bins[1] == n_local and store.lo is not None
    store._bins = None   # one-shot: valid only for the build right after the sort (positions move)
    cache = _cache.setdefault((str(dev), store.rank), _BuildCache())
    if not rebin and getattr(cache, "last", None) is not None and cache.last[0] == (n_total, bc):
        merged = None                       # the previous build's cell lists, as they are
        garr, narr, ncell = cache.last[1]
    elif merged:   # owned rows come sorted from the spatial sort on this grid: bin only the ghosts
        _, _, garr, narr, ncell = shell_grid_args(lo, hi, bc)
    else:
        _, _, garr, narr, ncell = grid_args(lo, hi, bc, bc)
    cache.last = ((n_total, bc), (garr, narr, ncell))
    keys = cache.get("keys", n_total, torch.int32, dev)
    cstart = cache.get("cstart", ncell + 1, torch.int32, dev)
    catoms = cache.get("catoms", n_total, torch.int32, dev)
    if cap_hint is None and n_local:
        # first build: size the table from the density (mean partners 4/3 pi bc^3 rho,
        # halved for half lists, +25 % for fluctuations) instead of growing by retries
        vol = float(np.prod(np.asarray(hi, dtype=np.float64) - np.asarray(lo, dtype=np.float64)))
        mean = n_local / max(vol, 1e-300) * (4.0 / 3.0) * math.pi * bc ** 3 * (0.5 if style == "half" else 1.0)
        cap_hint = grow_capacity(capacity, int(1.25 * mean) + 8)
    alloc = max(grow_capacity(capacity, 0), int(cap_hint or 0))
    # the binning is queued first (on a rebuild the device is idle until it arrives); the
    # list buffers are prepared while it runs, in less host time than its ~70 us of device
    # work, so the build launch still follows it back to back
    if merged is None:
        pass
    elif merged:
        _lib.check(lib.mdkk_bin_merge(ctx, store.x.data_ptr(), n_local, n_total, garr, narr, bins[2].data_ptr(),
                                      keys.data_ptr(), cstart.data_ptr(), catoms.data_ptr(), stream),
                   "mdkk_bin_merge")
    else:
        _lib.check(lib.mdkk_bin_atoms(ctx, store.x.data_ptr(), n_total, garr, narr, keys.data_ptr(),
                                      cstart.data_ptr(), catoms.data_ptr(), stream), "mdkk_bin_atoms")
    old_t = recycle.table_dev if recycle is not None else None
    counts = _recycled(recycle.counts_dev if recycle is not None else None, (max(n_local, 1),), torch.int32, dev)
    mc = cache.get("mc", 1, torch.int32, dev)   # one element; stream-ordered reuse across builds
    mc.zero_()
    deferred = defer and cap_hint is not None
    if deferred:
        table = _recycled(old_t, ((n_local + 31) // 32 or 1, alloc, 32), torch.int32, dev)
    if deferred:
        _lib.check(lib.mdkk_nbr_build(ctx, store.x.data_ptr(), n_local, n_total, garr, narr, cstart.data_ptr(),
                                      catoms.data_ptr(), store.gid.data_ptr(), store.orank.data_ptr(),
                                      store.rank, bc, STYLES[style], int(bool(newton)), alloc,
                                      table.data_ptr(), counts.data_ptr(), mc.data_ptr(), stream),
                   "mdkk_nbr_build")
        # the count read-back is queued right behind the build (pinned, async): settle()
        # then waits on this event only, not on the work queued after it
        pin = cache.bufs.get("mc_pin")
        if pin is None:
            pin = cache.bufs["mc_pin"] = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        pin.copy_(mc, non_blocking=True)
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(dev))
        nl = NeighborList(store, style, newton, cutoff, skin, alloc, table, counts, alloc,
                          ref_buf=recycle.ref_dev if recycle is not None else None,
                          ref_ready=ref_ready and recycle is not None)
        nl._pending = (mc, box, capacity, pin, ready)
        return nl
    while True:
        table = _recycled(old_t, ((n_local + 31) // 32 or 1, alloc, 32), torch.int32, dev)
        mc.zero_()
        _lib.check(lib.mdkk_nbr_build(ctx, store.x.data_ptr(), n_local, n_total, garr, narr, cstart.data_ptr(),
                                      catoms.data_ptr(), store.gid.data_ptr(), store.orank.data_ptr(),
                                      store.rank, bc, STYLES[style], int(bool(newton)), alloc,
                                      table.data_ptr(), counts.data_ptr(), mc.data_ptr(), stream),
                   "mdkk_nbr_build")
        need = int(mc.item())
        if need <= alloc:
            break
        alloc = grow_capacity(alloc, need)  # never truncate: grow and rebuild
    cap = grow_capacity(capacity, need)
    return NeighborList(store, style, newton, cutoff, skin, cap, table, counts, need,
                        ref_buf=recycle.ref_dev if recycle is not None else None,
                          ref_ready=ref_ready and recycle is not None)


def build_all(system: RankedSystem, cutoff: float, skin: float, style: str = "full",
              newton: bool = True, capacity: int = DEFAULT_CAPACITY) -> list[NeighborList]:
    """Exchange ghosts, then per-rank builds (mdkk/neighbor.py:222-227)."""
    if system.sort_width is None:
        system.sort_width = cutoff + skin
        system.sort_local(cutoff + skin)   # cell order -> compact 32-atom clusters
    system.exchange_ghosts(cutoff + skin)
    return [build(store, system.box, cutoff, skin, style, newton, capacity) for store in system.stores]


def any_needs_rebuild(lists: list[NeighborList]) -> bool:
    """Global OR of the skin test (mdkk/neighbor.py:230-231): one device max per rank, one sync."""
    if not lists:
        return False
    d2 = [nl.max_disp2_dev() for nl in lists if nl.n_local]
    if not d2:
        return False
    worst = float(torch.stack([t[0] for t in d2]).max().item())
    return math.sqrt(worst) > 0.5 * lists[0].skin


def brute_force_pairs(pos, box: Box, cutoff: float, device=None) -> set[tuple[int, int]]:
    """O(N^2) minimum-image pair set, unordered index pairs (i, j), i < j (mdkk/neighbor.py:234-245).

    The test oracle the reference exports, evaluated on the GPU in row blocks
    with the reference's operations (min image L*floor(d/L + 0.5), r^2 in the
    einsum order (dx^2 + dz^2) + dy^2, strict <)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    x = torch.as_tensor(np.asarray(pos, dtype=np.float64), device=dev)
    n = int(x.shape[0])
    L = torch.as_tensor(np.asarray(box.lengths, dtype=np.float64), device=dev)
    per = torch.as_tensor(np.asarray(box.periodic, dtype=bool), device=dev)
    out: set[tuple[int, int]] = set()
    cut2 = float(cutoff) * float(cutoff)
    step = max(1, (1 << 24) // max(n, 1))
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        d = x[None, :, :] - x[lo:hi, None, :]
        d = torch.where(per, d - L * torch.floor(d / L + 0.5), d)
        r2 = (d[..., 0] * d[..., 0] + d[..., 2] * d[..., 2]) + d[..., 1] * d[..., 1]
        j = torch.arange(n, device=dev)[None, :]
        i = torch.arange(lo, hi, device=dev)[:, None]
        hit = torch.nonzero((r2 < cut2) & (j > i)).cpu().numpy()
        out.update((int(a) + lo, int(b)) for a, b in hit)
    return out
