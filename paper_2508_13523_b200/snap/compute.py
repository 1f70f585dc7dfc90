"""SNAP pipeline drop-ins on the GPU (mirror of mdkk/snap/compute.py).

`build_neighbor_map`, `SnapState`, `compute_ui`, `compute_yi`,
`compute_fused_deidrj`, `compute_energy`, `energy_from_y` keep the reference
signatures (mdkk/snap/compute.py:105-436).  U lives in HBM as complex128
row-major [n_atoms][n_flat] (the reference's layout "a"); the engine keeps Y
as its half set, transposed (`Yh_dev[e][i]`, atoms fastest), and expands the
reference-layout `state.Y` only when it is read.  The `layout` / `batch_u` /
`batch_y` / `tile_v` knobs are real schedule parameters of the GPU kernels
(storage layout; pairs in flight per warp in compute_ui; atoms per lane in
compute_yi; atom tiles of yi / bi) and, as the reference guarantees
(mdkk/snap/compute.py:238-276), change results only at rounding level.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from .. import _lib
from ..memspace import DualArray, LayoutPolicy
from .coupling import CouplingTables, bi_entries, device_product_list


class SnapError(RuntimeError):
    pass


def cutoff_switch(r, r_c: float):
    """f_c(r) = (1 + cos(pi r / r_c)) / 2 and its derivative (mdkk/snap/compute.py:27-32).

    Element-wise on the input's own side: numpy in, numpy out; a device tensor
    stays on the device.  The kernels evaluate the same switch inline
    (snap_common.cuh pair_geometry)."""
    if torch.is_tensor(r):
        x = r.to(torch.float64)
        return 0.5 * (1.0 + torch.cos(np.pi * x / r_c)), -np.pi / (2.0 * r_c) * torch.sin(np.pi * x / r_c)
    x = np.asarray(r, dtype=np.float64)
    return 0.5 * (1.0 + np.cos(np.pi * x / r_c)), -np.pi / (2.0 * r_c) * np.sin(np.pi * x / r_c)


def pair_u_flat(a, b, twojmax: int, device=None) -> np.ndarray:
    """Unweighted levels u_0..u_2J of each (a, b), flattened to (n, n_flat)
    (mdkk/snap/compute.py:165-184), computed on the GPU (mdkk_snap_pair_u, the
    reference's four-term recursion; (a, b) need not be unitary)."""
    a = np.atleast_1d(np.asarray(a, dtype=np.complex128))
    b = np.atleast_1d(np.asarray(b, dtype=np.complex128))
    twojmax = int(twojmax)
    nf = sum((t + 1) ** 2 for t in range(twojmax + 1))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    at = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    bt = torch.from_numpy(np.ascontiguousarray(b)).to(dev)
    out = torch.empty((max(len(a), 1), nf), dtype=torch.complex128, device=dev)
    _lib.check(_lib.lib().mdkk_snap_pair_u(len(a), twojmax, at.data_ptr(), bt.data_ptr(), out.data_ptr(),
                                           _lib.stream(dev)), "mdkk_snap_pair_u")
    return out[: len(a)].cpu().numpy()


class NeighborMap:
    """The pairs of a full list with r < r_c (mdkk/snap/compute.py:66-119).

    The engine kernels evaluate the pairs on the fly from the list; the
    reference's per-pair arrays (`rows`, `cols`, `dr`, `r`, `a`, `b`, `fc`,
    `dfc`, (row, dz, dy, dx) order) are materialised on the device on first
    access (mdkk_snap_pair_count / _fill) for the staged path and for callers
    that inspect them.
    """

    _FIELDS = ("rows", "cols", "dr", "r", "a", "b", "fc", "dfc")

    def __init__(self, store, nlist, r_c: float):
        self.store, self.nlist, self.r_c = store, nlist, float(r_c)
        self._dev = None
        self._host = {}

    def device_arrays(self) -> dict:
        """Per-pair device tensors (int32 rows/cols, f64 dr (P,3), r, complex128 a/b, fc, dfc)."""
        if self._dev is None:
            st, nl = self.store, self.nlist
            dev = st.device
            st.to_device()
            n = st.n_local
            npair = torch.zeros(n + 1, dtype=torch.int32, device=dev)
            offs = torch.zeros(n + 1, dtype=torch.int32, device=dev)
            flags = torch.zeros(1, dtype=torch.int32, device=dev)
            lib, stream = _lib.lib(), _lib.stream(dev)
            _lib.check(lib.mdkk_snap_pair_count(_lib.ctx(dev), st.x.data_ptr(), n, nl.table_dev.data_ptr(),
                                                nl.counts_dev.data_ptr(), nl.alloc_cap, self.r_c,
                                                npair.data_ptr(), offs.data_ptr(), flags.data_ptr(), stream),
                       "mdkk_snap_pair_count")
            if int(flags.item()) & _lib.FLAG_COINCIDENT:
                raise SnapError("neighbor at zero distance")
            P = int(offs[n].item())
            m = max(P, 1)
            d = dict(rows=torch.empty(m, dtype=torch.int32, device=dev),
                     cols=torch.empty(m, dtype=torch.int32, device=dev),
                     dr=torch.empty((m, 3), dtype=torch.float64, device=dev),
                     r=torch.empty(m, dtype=torch.float64, device=dev),
                     a=torch.empty(m, dtype=torch.complex128, device=dev),
                     b=torch.empty(m, dtype=torch.complex128, device=dev),
                     fc=torch.empty(m, dtype=torch.float64, device=dev),
                     dfc=torch.empty(m, dtype=torch.float64, device=dev))
            _lib.check(lib.mdkk_snap_pair_fill(st.x.data_ptr(), n, nl.table_dev.data_ptr(), nl.counts_dev.data_ptr(),
                                               nl.alloc_cap, self.r_c, offs.data_ptr(),
                                               *[d[k].data_ptr() for k in self._FIELDS], stream),
                       "mdkk_snap_pair_fill")
            self._dev = {k: v[:P] for k, v in d.items()}
        return self._dev

    @property
    def n_pairs(self) -> int:
        return int(self.device_arrays()["rows"].shape[0])

    def deriv_params(self, sel: slice):
        """(da, db), each (n, 3) complex, for one pair block (mdkk/snap/compute.py:98-102),
        from the device geometry the force kernels use (mdkk_snap_pair_grads)."""
        d = self.device_arrays()
        dr = d["dr"][sel].contiguous()
        n = int(dr.shape[0])
        da = torch.empty((max(n, 1), 3), dtype=torch.complex128, device=dr.device)
        db = torch.empty_like(da)
        _lib.check(_lib.lib().mdkk_snap_pair_grads(n, dr.data_ptr(), self.r_c, da.data_ptr(), db.data_ptr(),
                                                   _lib.stream(dr.device)), "mdkk_snap_pair_grads")
        return da[:n].cpu().numpy(), db[:n].cpu().numpy()

    def __getattr__(self, name):
        if name in NeighborMap._FIELDS:
            h = self._host.get(name)
            if h is None:
                t = self.device_arrays()[name].cpu().numpy()
                h = self._host[name] = t.astype(np.int64) if name in ("rows", "cols") else t
            return h
        raise AttributeError(name)


def build_neighbor_map(store, nlist, r_c: float) -> NeighborMap:
    """Validate the list for the descriptor pipeline (mdkk/snap/compute.py:105-119)."""
    if nlist.style != "full":
        raise SnapError("descriptor pipeline requires a full-style neighbor list")
    if r_c > nlist.build_cutoff:
        raise SnapError(f"cutoff {r_c} exceeds neighbor build cutoff {nlist.build_cutoff}")
    if not getattr(nlist, "_geo_order", False):
        # the reference's pair order (row, dz, dy, dx) on the device table, once per list:
        # the U accumulation order then follows geometry, not atom labels
        # (mdkk tests/test_snap.py:502-520)
        store.to_device()
        _lib.check(_lib.lib().mdkk_nbr_geo_order(store.x.data_ptr(), store.n_local, nlist.alloc_cap,
                                                 nlist.table_dev.data_ptr(), nlist.counts_dev.data_ptr(),
                                                 _lib.stream(store.device)), "mdkk_nbr_geo_order")
        nlist._geo_order = True
    return NeighborMap(store, nlist, r_c)


class _Handle:
    """Device copy of the Z-list product table (mdkk_snap_create)."""

    def __init__(self, tables: CouplingTables, beta: np.ndarray, device):
        coef, code, n_half, fmap = device_product_list(tables, beta)
        out = C.c_void_p()
        with torch.cuda.device(device):
            _lib.check(_lib.lib().mdkk_snap_create(
                _lib.ctx(device), tables.index.twojmax, len(coef), coef.ctypes.data, code.ctypes.data,
                n_half, fmap.ctypes.data, C.byref(out)), "mdkk_snap_create")
        self.ptr = out.value
        self.n_half = n_half
        self.n_products = int((coef != 0).sum())

    def __del__(self):
        try:
            _lib.lib().mdkk_snap_destroy(self.ptr)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


class SnapState:
    """Per-atom U and Y fields in HBM plus the schedule knobs (mdkk/snap/compute.py:238-276).

    `layout` is the device storage of U and the reference-layout Y: "a" =
    row-major [n][n_flat] (ui writes one atom's row), "b" = transposed
    [n_flat][ld] with atoms fastest (the yi / bi tile loads read whole
    rows).  `tile_v` > 0 runs yi and bi over atom tiles of that size (one
    launch per tile: bounded shared work per launch).  `batch_u` is the
    number of neighbour pairs compute_ui expands concurrently per two warps
    (<= 3, 4..7, >= 8 -> 32-, 16-, 8-lane teams per pair; the paper's
    ComputeUi work batching, Table 2; the default 4 is the fastest on B200);
    `batch_y` the atoms per lane of compute_yi (1, >= 2 -> 2: every Z-list
    broadcast serves two atoms).  No knob changes results
    beyond rounding (mdkk tests/test_snap.py:482-499).
    """

    def __init__(self, tables: CouplingTables, n_atoms: int, beta, batch_u: int = 4, batch_y: int = 1,
                 tile_v: int = 0, layout: str = "a", device=None):
        self.tables = tables
        self.index = tables.index
        self.n_atoms = int(n_atoms)
        self.beta = np.asarray(beta, dtype=np.float64)
        if self.beta.shape != (len(tables.triples),):
            raise SnapError(f"beta has {self.beta.shape} entries; expected {len(tables.triples)} "
                            f"(one per coupled triple)")
        if layout not in ("a", "b"):
            raise SnapError(f"layout must be 'a' or 'b', got {layout!r}")
        self.layout = layout
        self.batch_u, self.batch_y, self.tile_v = max(1, int(batch_u)), max(1, int(batch_y)), int(tile_v)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        nf = self.index.n_flat
        shape = (max(1, self.n_atoms), nf)
        n_half = sum((t + 1) ** 2 // 2 if t & 1 else (t // 2) * (t + 1) + t // 2 + 1
                     for t in range(self.index.twojmax + 1))
        self.ld = max(32, (self.n_atoms + 31) // 32 * 32)
        self._lay = 1 if layout == "b" else 0
        if self._lay:
            rm = LayoutPolicy.transposed(2)
            self.U_dev = torch.zeros((nf, self.ld), dtype=torch.complex128, device=self.device)
        else:
            rm = LayoutPolicy.row_major(2)   # device rows are atoms: one warp streams one atom's entries
            self.U_dev = torch.zeros(shape, dtype=torch.complex128, device=self.device)
        self.Yh_dev = torch.zeros((n_half, self.ld), dtype=torch.complex128, device=self.device)
        self._y_expanded = True   # the reference-layout Y (if any) agrees with Yh_dev
        self.U = DualArray(shape, layout_b=rm, dtype=np.complex128, device=self.device, storage_b=self.U_dev)
        # the reference-layout Y (n x n_flat, as large as U) exists only once something reads
        # or writes it: the engine itself works on the half set Yh
        self._shape, self._rm = shape, rm
        self._Y = None
        self.Y_dev = None
        self.energy_dev = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.flags = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._handle = None

    @property
    def Y(self) -> DualArray:
        if self._Y is None:
            self.Y_dev = torch.zeros_like(self.U_dev)
            self._Y = DualArray(self._shape, layout_b=self._rm, dtype=np.complex128, device=self.device,
                                storage_b=self.Y_dev)
        return self._Y

    def handle(self) -> _Handle:
        if self._handle is None:
            self._handle = _Handle(self.tables, self.beta, self.device)
        return self._handle

    def scheduled(self) -> int:
        """The handle pointer with this state's batch_u / batch_y applied (handles are
        shared between the states of one style, so the knobs are set per call)."""
        h = self.handle().ptr
        _lib.check(_lib.lib().mdkk_snap_set_schedule(h, self.batch_u, self.batch_y), "mdkk_snap_set_schedule")
        return h

    def u_view(self) -> np.ndarray:
        return self.U.read("a")[: self.n_atoms]

    def y_view(self) -> np.ndarray:
        self.expand_y()
        return self.Y.read("a")[: self.n_atoms]

    def expand_y(self) -> None:
        """Reference layout Y (n, n_flat) from the engine's half/transposed Yh (after compute_yi)."""
        if self._y_expanded and self._Y is not None:
            return
        Y = self.Y   # allocated on first use
        _lib.check(_lib.lib().mdkk_snap_y_expand(self.handle().ptr, self.Yh_dev.data_ptr(), self.ld, self.n_atoms,
                                                 self.Y_dev.data_ptr(), self._lay, self.ld, _lib.stream(self.device)),
                   "mdkk_snap_y_expand")
        Y.modified_a = False
        Y.mark_modified("b")
        self._y_expanded = True

    def sync_yh(self) -> None:
        """Engine Yh current: a host-written reference-layout Y is compressed into it."""
        if self._Y is not None and self._Y.modified_a:
            self.Y.sync("b")
            _lib.check(_lib.lib().mdkk_snap_y_compress(self.handle().ptr, self.Y_dev.data_ptr(), self.n_atoms,
                                                       self.Yh_dev.data_ptr(), self.ld, self._lay, self.ld,
                                                       _lib.stream(self.device)),
                       "mdkk_snap_y_compress")


def compute_ui(nmap: NeighborMap, state: SnapState) -> None:
    """U_i = sum_k f_c u(a_k, b_k) on the GPU (mdkk/snap/compute.py:279-292)."""
    st, nl = nmap.store, nmap.nlist
    st.to_device()
    state.flags.zero_()
    _lib.check(_lib.lib().mdkk_snap_ui(state.scheduled(), st.x.data_ptr(), st.n_local, nl.table_dev.data_ptr(),
                                       nl.counts_dev.data_ptr(), nl.alloc_cap, nmap.r_c, state.U_dev.data_ptr(),
                                       state._lay, state.ld, state.flags.data_ptr(), _lib.stream(st.device)),
               "mdkk_snap_ui")
    state.U.modified_a = False
    state.U.mark_modified("b")


def check_flags(state: SnapState) -> None:
    if int(state.flags.item()) & _lib.FLAG_COINCIDENT:
        raise SnapError("neighbor at zero distance")


def compute_yi(state: SnapState) -> None:
    """Full three-slot adjoint Y and the per-atom energy sum (mdkk/snap/compute.py:303-340, :376-387)."""
    state.U.sync("b")
    tiles = _tiles(state)
    h = state.scheduled()
    e_t = state.energy_dev if len(tiles) == 1 else torch.zeros(len(tiles), dtype=torch.float64, device=state.device)
    for k, (a0, n) in enumerate(tiles):
        _lib.check(_lib.lib().mdkk_snap_yi(_lib.ctx(state.device), h, _u_at(state, a0), n,
                                           state.Yh_dev.data_ptr() + 16 * a0, state.ld, e_t.data_ptr() + 8 * k,
                                           state._lay, state.ld, _lib.stream(state.device)), "mdkk_snap_yi")
    if len(tiles) > 1:
        state.energy_dev.copy_(e_t.sum().reshape(1))
    if state._Y is not None:
        state._Y.modified_a = False
        state._Y.modified_b = False
    state._y_expanded = False


def _tiles(state: SnapState):
    """Atom tiles (offset, count) of the tile_v knob (mdkk/snap/compute.py:295-299)."""
    n, t = state.n_atoms, state.tile_v
    if t <= 0 or t >= n:
        return [(0, n)]
    return [(a0, min(t, n - a0)) for a0 in range(0, n, t)]


def _u_at(state: SnapState, a0: int) -> int:
    """Device address of atom a0's U entries in the state's layout."""
    return state.U_dev.data_ptr() + 16 * (a0 if state._lay else a0 * state.index.n_flat)


def compute_zi(state: SnapState, it: int) -> np.ndarray:
    """Dense Z block of coupled triple `it` for every atom, (n, tj+1, tj+1)
    (mdkk/snap/compute.py:343-351; an oracle helper there): Z[iz] += c U[iu1] U[iu2]
    over the triple's terms, formed on the device from the resident U."""
    tt = state.tables.terms[it]
    tj = tt.tj
    n = state.n_atoms
    state.U.sync("b")
    u = state.U_dev[:, :n].T if state._lay else state.U_dev[:n]
    dev = state.device
    iz = torch.from_numpy(tt.iz - state.index.block_offset[tj]).to(dev)
    i1, i2 = torch.from_numpy(tt.iu1).to(dev), torch.from_numpy(tt.iu2).to(dev)
    c = torch.from_numpy(tt.coeff).to(dev).to(torch.complex128)
    z = torch.zeros(((tj + 1) * (tj + 1), max(n, 1)), dtype=torch.complex128, device=dev)
    z.index_add_(0, iz, (c[:, None] * u[:, i1].T * u[:, i2].T))
    return z[:, :n].T.reshape(n, tj + 1, tj + 1).cpu().numpy()


def compute_bi_complex(state: SnapState) -> np.ndarray:
    """Scalar invariants per atom and triple, complex (mdkk/snap/compute.py:354-367), on the GPU."""
    B = _bi_device(state)
    return B.cpu().numpy()


def compute_bi(state: SnapState) -> np.ndarray:
    """Descriptor vector: real part of the invariants (mdkk/snap/compute.py:370-373)."""
    return compute_bi_complex(state).real


def _bi_device(state: SnapState) -> torch.Tensor:
    n_tri = len(state.tables.triples)
    B = torch.zeros((max(state.n_atoms, 1), n_tri), dtype=torch.complex128, device=state.device)
    if state.n_atoms == 0:
        return B[:0]
    tab = getattr(state, "_bi_tab", None)
    if tab is None:
        coef, code, tri, chunk = bi_entries(state.tables, int(_lib.lib().mdkk_snap_bi_warps()))
        tab = state._bi_tab = [torch.from_numpy(v).to(state.device) for v in (coef, code, tri, chunk)]
    state.U.sync("b")
    for a0, n in _tiles(state):
        _lib.check(_lib.lib().mdkk_snap_bi(state.handle().ptr, _u_at(state, a0), n, *[t.data_ptr() for t in tab],
                                           n_tri, B.data_ptr() + 16 * n_tri * a0, state._lay, state.ld,
                                           _lib.stream(state.device)), "mdkk_snap_bi")
    return B[: state.n_atoms]


def energy_from_y(state: SnapState) -> float:
    """Re(sum Y : conj(U)) / 3, accumulated by the yi kernel (mdkk/snap/compute.py:376-387)."""
    return float(state.energy_dev.item()) if state.n_atoms else 0.0


def compute_energy(state: SnapState) -> float:
    """E = sum over atoms of beta . B, the descriptor route (mdkk/snap/compute.py:376-380)."""
    if not state.n_atoms:
        return 0.0
    beta = torch.from_numpy(state.beta).to(state.device)
    return float((_bi_device(state).real @ beta).sum().item())


def deidrj_device(nmap: NeighborMap, state: SnapState, f: torch.Tensor) -> None:
    """Launch the fused force kernel, accumulating into device rows f (n_total, 4) (must be zeroed)."""
    st, nl = nmap.store, nmap.nlist
    state.sync_yh()
    _lib.check(_lib.lib().mdkk_snap_deidrj(state.handle().ptr, st.x.data_ptr(), st.n_local, nl.table_dev.data_ptr(),
                                           nl.counts_dev.data_ptr(), nl.alloc_cap, nmap.r_c,
                                           state.Yh_dev.data_ptr(), state.ld, f.data_ptr(), _lib.stream(st.device)),
               "mdkk_snap_deidrj")


def compute_fused_deidrj(nmap: NeighborMap, state: SnapState, n_total: int) -> np.ndarray:
    """All three force components in one pass over pairs (mdkk/snap/compute.py:390-409); host copy returned."""
    f = torch.zeros((max(n_total, 1), 4), dtype=torch.float64, device=state.device)
    deidrj_device(nmap, state, f)
    return f[:n_total, :3].cpu().numpy()


def compute_duidrj(nmap: NeighborMap, state: SnapState) -> np.ndarray:
    """Staged path: d(f_c u)/d dr for every pair, (n_pairs, 3, n_flat) (mdkk/snap/compute.py:412-422)."""
    return _duidrj_device(nmap, state).cpu().numpy()


def _duidrj_device(nmap: NeighborMap, state: SnapState) -> torch.Tensor:
    d = nmap.device_arrays()
    P = d["rows"].shape[0]
    out = torch.empty((max(P, 1), 3, state.index.n_flat), dtype=torch.complex128, device=state.device)
    _lib.check(_lib.lib().mdkk_snap_duidrj(state.handle().ptr, P, d["dr"].data_ptr(), nmap.r_c, out.data_ptr(),
                                           _lib.stream(state.device)), "mdkk_snap_duidrj")
    return out[:P]


def compute_deidrj(nmap: NeighborMap, state: SnapState, du, n_total: int) -> np.ndarray:
    """Staged contraction of the derivatives against Y (mdkk/snap/compute.py:425-436)."""
    d = nmap.device_arrays()
    P = d["rows"].shape[0]
    du_t = du if isinstance(du, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(du))
    du_t = du_t.to(device=state.device, dtype=torch.complex128).contiguous()
    if du_t.shape != (P, 3, state.index.n_flat):
        raise SnapError(f"derivative block has shape {tuple(du_t.shape)}; expected {(P, 3, state.index.n_flat)}")
    state.expand_y()
    state.Y.sync("b")
    y_rows = state.Y_dev if not state._lay else state.Y.view("b").contiguous()   # kernel reads [n][n_flat]
    f = torch.zeros((max(n_total, 1), 4), dtype=torch.float64, device=state.device)
    _lib.check(_lib.lib().mdkk_snap_deidrj_staged(state.handle().ptr, P, d["rows"].data_ptr(), d["cols"].data_ptr(),
                                                  y_rows.data_ptr(), du_t.data_ptr(), f.data_ptr(),
                                                  _lib.stream(state.device)), "mdkk_snap_deidrj_staged")
    return f[:n_total, :3].cpu().numpy()
