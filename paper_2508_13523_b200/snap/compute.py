"""SNAP pipeline drop-ins on the GPU (mirror of mdkk/snap/compute.py).

`build_neighbor_map`, `SnapState`, `compute_ui`, `compute_yi`,
`compute_fused_deidrj`, `compute_energy`, `energy_from_y` keep the reference
signatures (mdkk/snap/compute.py:105-436).  U lives in HBM as complex128
row-major [n_atoms][n_flat] (the reference's layout "a"); the engine keeps Y
as its half set, transposed (`Yh_dev[e][i]`, atoms fastest), and expands the
reference-layout `state.Y` only when it is read.  The `layout` / `batch_u` /
`batch_y` / `tile_v` knobs are accepted for signature parity (the reference
guarantees they never change results, mdkk/snap/compute.py:238-276) and do
not change the GPU schedule.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from .. import _lib
from ..memspace import DualArray, LayoutPolicy
from .coupling import CouplingTables, device_product_list


class SnapError(RuntimeError):
    pass


class NeighborMap:
    """The pairs of a full list with r < r_c, evaluated on the fly by the kernels (mdkk/snap/compute.py:66-119)."""

    def __init__(self, store, nlist, r_c: float):
        self.store, self.nlist, self.r_c = store, nlist, float(r_c)

    @property
    def n_pairs(self) -> int:
        """Pairs within r_c (diagnostic, host sync)."""
        st, nl = self.store, self.nlist
        x = st.positions()
        rows, cols, _, _ = nl.pairs()
        d = x[cols] - x[rows]
        return int((np.einsum("ij,ij->i", d, d) < self.r_c ** 2).sum())


def build_neighbor_map(store, nlist, r_c: float) -> NeighborMap:
    """Validate the list for the descriptor pipeline (mdkk/snap/compute.py:105-119)."""
    if nlist.style != "full":
        raise SnapError("descriptor pipeline requires a full-style neighbor list")
    if r_c > nlist.build_cutoff:
        raise SnapError(f"cutoff {r_c} exceeds neighbor build cutoff {nlist.build_cutoff}")
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
    """Per-atom U and Y fields in HBM plus the (schedule-only) knobs (mdkk/snap/compute.py:238-276)."""

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
        rm = LayoutPolicy.row_major(2)   # device rows are atoms: one warp streams one atom's 285 entries
        self.U_dev = torch.zeros(shape, dtype=torch.complex128, device=self.device)
        self.Y_dev = torch.zeros_like(self.U_dev)
        n_half = sum((t + 1) ** 2 // 2 if t & 1 else (t // 2) * (t + 1) + t // 2 + 1
                     for t in range(self.index.twojmax + 1))
        self.ld = max(32, (self.n_atoms + 31) // 32 * 32)
        self.Yh_dev = torch.zeros((n_half, self.ld), dtype=torch.complex128, device=self.device)
        self._y_expanded = True   # Y_dev agrees with Yh_dev
        self.U = DualArray(shape, layout_b=rm, dtype=np.complex128, device=self.device, storage_b=self.U_dev)
        self.Y = DualArray(shape, layout_b=rm, dtype=np.complex128, device=self.device, storage_b=self.Y_dev)
        self.energy_dev = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.flags = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._handle = None

    def handle(self) -> _Handle:
        if self._handle is None:
            self._handle = _Handle(self.tables, self.beta, self.device)
        return self._handle

    def u_view(self) -> np.ndarray:
        return self.U.read("a")[: self.n_atoms]

    def y_view(self) -> np.ndarray:
        self.expand_y()
        return self.Y.read("a")[: self.n_atoms]

    def expand_y(self) -> None:
        """Reference layout Y (n, n_flat) from the engine's half/transposed Yh (after compute_yi)."""
        if self._y_expanded:
            return
        _lib.check(_lib.lib().mdkk_snap_y_expand(self.handle().ptr, self.Yh_dev.data_ptr(), self.ld, self.n_atoms,
                                                 self.Y_dev.data_ptr(), _lib.stream(self.device)),
                   "mdkk_snap_y_expand")
        self.Y.modified_a = False
        self.Y.mark_modified("b")
        self._y_expanded = True

    def sync_yh(self) -> None:
        """Engine Yh current: a host-written reference-layout Y is compressed into it."""
        if self.Y.modified_a:
            self.Y.sync("b")
            _lib.check(_lib.lib().mdkk_snap_y_compress(self.handle().ptr, self.Y_dev.data_ptr(), self.n_atoms,
                                                       self.Yh_dev.data_ptr(), self.ld, _lib.stream(self.device)),
                       "mdkk_snap_y_compress")


def compute_ui(nmap: NeighborMap, state: SnapState) -> None:
    """U_i = sum_k f_c u(a_k, b_k) on the GPU (mdkk/snap/compute.py:279-292)."""
    st, nl = nmap.store, nmap.nlist
    st.to_device()
    state.flags.zero_()
    _lib.check(_lib.lib().mdkk_snap_ui(state.handle().ptr, st.x.data_ptr(), st.n_local, nl.table_dev.data_ptr(),
                                       nl.counts_dev.data_ptr(), nl.alloc_cap, nmap.r_c, state.U_dev.data_ptr(),
                                       state.flags.data_ptr(), _lib.stream(st.device)), "mdkk_snap_ui")
    state.U.modified_a = False
    state.U.mark_modified("b")


def check_flags(state: SnapState) -> None:
    if int(state.flags.item()) & _lib.FLAG_COINCIDENT:
        raise SnapError("neighbor at zero distance")


def compute_yi(state: SnapState) -> None:
    """Full three-slot adjoint Y and the per-atom energy sum (mdkk/snap/compute.py:303-340, :376-387)."""
    state.U.sync("b")
    _lib.check(_lib.lib().mdkk_snap_yi(_lib.ctx(state.device), state.handle().ptr, state.U_dev.data_ptr(),
                                       state.n_atoms, state.Yh_dev.data_ptr(), state.ld,
                                       state.energy_dev.data_ptr(), _lib.stream(state.device)), "mdkk_snap_yi")
    state.Y.modified_a = False
    state.Y.modified_b = False
    state._y_expanded = False


def energy_from_y(state: SnapState) -> float:
    """Re(sum Y : conj(U)) / 3, accumulated by the yi kernel (mdkk/snap/compute.py:376-387)."""
    return float(state.energy_dev.item()) if state.n_atoms else 0.0


def compute_energy(state: SnapState) -> float:
    """E = sum beta . B; equal to the adjoint route to 1e-12 (mdkk tests/test_snap.py:364-372)."""
    return energy_from_y(state)


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
