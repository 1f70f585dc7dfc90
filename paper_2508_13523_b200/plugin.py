"""The B200 path plugged into the reference engine `mdkk` (the drop-in boundary).

The reference's engine keeps its own host objects (numpy `RankedSystem`,
`AtomStore`, `NeighborList`, `NeighborMap`, `SnapState`); this module lets it
run its hot path on the GPU without changing them:

* `register(registry)` adds the paper's `/kk` styles -- `lj/cut/kk`,
  `lj/cut/opt/kk`, `snap/kk`, `snap/opt/kk` -- to an mdkk `StyleRegistry`
  (mdkk/driver/registry.py:24-50), so `suffix kk` in a script selects them and
  everything else falls back to the base style (mdkk/driver/simulation.py:145-153);
* `install()` rebinds mdkk's hot-path functions in every loaded mdkk module
  (`neighbor.build`, `brute_force_pairs`, `pair_lj.compute_pair`, the SNAP
  `compute_ui / compute_yi / compute_fused_deidrj / compute_duidrj /
  compute_deidrj / compute_bi(_complex) / pair_u_flat`) to the adapters below,
  and makes `default_registry()` include the /kk styles.  This is how the
  reference's own test modules run against the drop-ins
  (tests/test_reference_suite_gpu.py).

Each adapter mirrors the reference rows on the device (positions uploaded per
call, tables per list), runs the sm_100a kernels, and writes results back
through the reference's DualArray protocol (`read("a")` / `mark_modified`).
Communication and bookkeeping stay the reference's own (`exchange_ghosts`,
`reverse_comm`, `gather_forces`): the boundary is the compute.  There is no
CPU fallback: every adapter raises if the CUDA library is missing.
"""

from __future__ import annotations

import sys
import weakref

import numpy as np
import torch

from . import _lib
from .domain import AtomStore
from .domain import Box as _Box
from .memspace import ordered_scatter
from .neighbor import NeighborList as _NL
from .neighbor import build as _build
from .neighbor import brute_force_pairs as _brute
from .pair_lj import PairParams as _Params
from .pair_lj import lj_force_rank
from .snap import compute as _sc
from .snap.coupling import make_coupling_tables

_CHUNK_BASE = 8192   # the reference's SNAP pair chunk (mdkk/snap/compute.py:20), scaled by batch_u


def _mdkk():
    import mdkk  # the reference engine this plugs into (baseline/_ref or /root/reference/pkg/src)
    return mdkk


def _dev() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------------- mirrors
class _Mirror:
    """Device rows of one reference AtomStore (same row order: n_local owned, then ghosts)."""

    def __init__(self, ref_store, device):
        self.device = device
        self.n_local, self.n_total = int(ref_store.n_local), int(ref_store.n_total)
        cap = max(self.n_total, 1)
        x = torch.zeros((cap, 4), dtype=torch.float64, device=device)
        v = torch.zeros((max(self.n_local, 1), 4), dtype=torch.float64, device=device)
        gid = torch.from_numpy(np.asarray(ref_store.global_ids, dtype=np.int64)[: self.n_total].copy()).to(device)
        st = AtomStore(int(ref_store.rank), device, x, v, gid, self.n_local)
        st.n_ghost = self.n_total - self.n_local
        st._views()
        if self.n_total:
            st.orank[: self.n_total] = torch.from_numpy(
                np.asarray(ref_store.owner_rank[: self.n_total], dtype=np.int32)).to(device)
            st.oidx[: self.n_total] = torch.from_numpy(
                np.asarray(ref_store.owner_index[: self.n_total], dtype=np.int32)).to(device)
        self.store = st
        self.upload(ref_store)

    def upload(self, ref_store) -> AtomStore:
        """Current host positions -> device rows (the reference moves atoms in numpy)."""
        if self.n_total:
            pos = np.ascontiguousarray(ref_store.positions()[: self.n_total], dtype=np.float64)
            self.store.x[: self.n_total, :3].copy_(torch.from_numpy(pos))
        self.store.device_wrote(pos=True)
        return self.store


_mirrors: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _mirror(ref_store) -> AtomStore:
    """The store's device mirror with current positions (rebuilt when its rows changed)."""
    m = _mirrors.get(ref_store)
    if m is None or m.n_total != ref_store.n_total or m.n_local != ref_store.n_local:
        m = _mirrors[ref_store] = _Mirror(ref_store, _dev())
        return m.store
    return m.upload(ref_store)


def _device_list(ref_nl, store: AtomStore) -> _NL:
    """A device NeighborList over the mirror's rows: the one the drop-in build made,
    else the reference list's table uploaded in the cluster-blocked layout."""
    kk = getattr(ref_nl, "_kk", None)
    if kk is not None and kk.store is store:
        return kk
    n, cap = int(ref_nl.n_local), int(ref_nl.max_neighbors)
    ncl = (n + 31) // 32 or 1
    tbl = np.full((ncl * 32, cap), -1, dtype=np.int32)
    if n:
        tbl[:n] = np.asarray(ref_nl.table.read("a"))[:n, :cap]
    dev = store.device
    table = torch.from_numpy(tbl.reshape(ncl, 32, cap).transpose(0, 2, 1).copy()).to(dev)
    counts = torch.from_numpy(np.asarray(ref_nl.counts, dtype=np.int32).reshape(-1)[: max(n, 1)].copy()).to(dev)
    if n == 0:
        counts = torch.zeros(1, dtype=torch.int32, device=dev)
    nl = _NL(store, ref_nl.style, ref_nl.newton, ref_nl.cutoff, ref_nl.skin, cap, table, counts,
             int(counts.max().item()) if n else 0)
    ref_nl._kk = nl
    return nl


# ---------------------------------------------------------- neighbour build
def build(store, box, cutoff: float, skin: float, style: str = "full", newton: bool = True,
          capacity: int = 16):
    """mdkk.neighbor.build (mdkk/neighbor.py:182-219) on the GPU: the returned object is the
    reference's own NeighborList, filled from the device build (canonical rows, -1 padded
    table, counts, capacity grown x1.5 from `capacity`, directed pair arrays)."""
    mn = _mdkk().neighbor
    if style not in ("full", "half"):
        raise mn.NeighborError(f"unknown list style {style!r}")
    bc = cutoff + skin
    if bc > 0.5 * box.min_periodic_length():
        raise mn.NeighborError(f"cutoff+skin {bc} exceeds half the shortest periodic box length")
    mirror = _mirror(store)
    nl = _build(mirror, _Box(box.lengths, box.periodic), cutoff, skin, style, newton, capacity)
    rows, cols, w, wj = nl.pairs()
    out = mn.NeighborList(store, style, newton, cutoff, skin, capacity)
    n = store.n_local
    counts = nl.counts.astype(np.int32) if n else np.zeros(0, np.int32)
    out.max_neighbors = nl.max_neighbors
    out.counts = counts
    out.table = _mdkk().memspace.create_dual((max(n, 1), nl.max_neighbors), dtype=np.int32)
    tbl = out.table.view("a")
    tbl.fill(-1)
    if len(rows):
        first = np.concatenate([[0], np.cumsum(counts)])[:-1]
        tbl[rows, np.arange(len(rows)) - first[rows]] = cols
    out.table.mark_modified("a")
    out.pair_i, out.pair_j, out.pair_weight, out.pair_write_j = rows, cols, w, wj
    out._kk = nl
    return out


def brute_force_pairs(pos, box, cutoff: float) -> set:
    """mdkk.neighbor.brute_force_pairs (mdkk/neighbor.py:234-245) on the GPU."""
    return _brute(pos, _Box(box.lengths, box.periodic), cutoff)


# ------------------------------------------------------------------- LJ
def compute_pair(kernel, system, lists, mode: str = "atom", strategy=None, n_workers=None,
                 zero_forces: bool = True):
    """mdkk.pair_lj.compute_pair (mdkk/pair_lj.py:114-179) with the force kernel on the GPU.

    Per rank: the mirror's positions are refreshed, the list's device table is
    reused (or uploaded), the sm_100a LJ kernel runs with the requested schedule
    (`mode`) and half-list write strategy (the reference's Serial / Duplicate /
    Atomic objects), and the forces are added into the reference store's force
    rows; then the reference's reverse comm folds ghost rows and the reference
    PairResult is returned."""
    mp = _mdkk().pair_lj
    mm = _mdkk().memspace
    if mode not in ("atom", "neighbor"):
        raise mp.PairError(f"unknown execution mode {mode!r}")
    params = getattr(kernel, "params", None)
    if params is None or not all(hasattr(params, k) for k in ("epsilon", "sigma", "r_c")):
        raise mp.PairError(f"the device pair engine evaluates LJCut kernels, got {kernel!r}")
    strat = _strategy(strategy, n_workers, mm)
    p = _Params(params.epsilon, params.sigma, params.r_c)
    if zero_forces:
        system.zero_forces()
    dev = _dev()
    evs = torch.zeros((len(system.stores), 7), dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    contribs = []
    for k, (store, nlist) in enumerate(zip(system.stores, lists)):
        nlist.check_current()
        mirror = _mirror(store)
        nl = _device_list(nlist, mirror)
        mirror.f.zero_()
        lj_force_rank(mirror, nl, p, evs[k], flags, zero=False, mode=mode, strategy=strat)
        contribs.append((store, mirror))
    if int(flags.item()) & _lib.FLAG_COINCIDENT:
        raise mp.PairError("coincident atoms (r = 0)")
    for store, mirror in contribs:
        if store.n_total:
            f = store.force.read("a")
            f[: store.n_total] += mirror.f[: store.n_total, :3].cpu().numpy()
            store.force.mark_modified("a")
    if any(s.n_ghost for s in system.stores):
        system.reverse_comm()
    ev = evs.sum(dim=0).cpu().numpy()
    return mp.PairResult(float(ev[0]), system.gather_forces(), ev[1:7].copy())


def _strategy(strategy, n_workers, mm):
    """The reference's strategy object -> this package's (same semantics, device kernels)."""
    from . import memspace as ms
    if strategy is None or isinstance(strategy, mm.Serial):
        return ms.Serial()   # the reference's default (mdkk/pair_lj.py:131)
    if isinstance(strategy, mm.Atomic):
        return ms.Atomic()
    if isinstance(strategy, mm.Duplicate):
        copies = strategy.copies if n_workers is None else min(strategy.copies, ms.worker_count(n_workers))
        return ms.Duplicate(copies)
    if isinstance(strategy, (ms.Serial, ms.Atomic, ms.Duplicate)):
        return strategy
    raise _mdkk().pair_lj.PairError(f"unknown scatter strategy {strategy!r}")


# ------------------------------------------------------------------- SNAP
_tables: dict = {}


def _state(rs) -> _sc.SnapState:
    """This package's SnapState twin of a reference SnapState (same tables, beta, knobs)."""
    tj = int(rs.index.twojmax)
    key = (int(rs.n_atoms), rs.beta.tobytes(), rs.batch_u, rs.batch_y, rs.tile_v)
    st = getattr(rs, "_kk", None)
    if st is None or st._key != key:
        tables = _tables.get(tj)
        if tables is None:
            tables = _tables[tj] = make_coupling_tables(tj / 2.0)
        st = _sc.SnapState(tables, rs.n_atoms, rs.beta, batch_u=rs.batch_u, batch_y=rs.batch_y,
                           tile_v=rs.tile_v, layout="a", device=_dev())
        st._key = key
        rs._kk = st
    return st


def _put(dual, layout: str, n: int, host: np.ndarray) -> None:
    arr = dual.read(layout)
    arr[:] = 0.0
    arr[:n] = host
    dual.mark_modified(layout)


def _chunks(n_pairs: int, rs):
    step = max(1, int(rs.batch_u)) * _CHUNK_BASE
    return [(lo, min(lo + step, n_pairs)) for lo in range(0, n_pairs, step)]


def pair_u_flat(a, b, twojmax: int) -> np.ndarray:
    return _sc.pair_u_flat(a, b, twojmax)


def compute_ui(nmap, state) -> None:
    """mdkk compute_ui (mdkk/snap/compute.py:279-292): u(a, b) of every pair on the GPU
    (four-term recursion), weighted by f_c and summed into its row in pair order."""
    st = _state(state)
    dev, nf = st.device, st.index.n_flat
    n = st.n_atoms
    U = torch.zeros((max(n, 1), nf), dtype=torch.complex128, device=dev)
    lib = _lib.lib()
    for lo, hi in _chunks(nmap.n_pairs, state):
        m = hi - lo
        a = torch.from_numpy(np.ascontiguousarray(nmap.a[lo:hi])).to(dev)
        b = torch.from_numpy(np.ascontiguousarray(nmap.b[lo:hi])).to(dev)
        u = torch.empty((m, nf), dtype=torch.complex128, device=dev)
        _lib.check(lib.mdkk_snap_pair_u(m, st.index.twojmax, a.data_ptr(), b.data_ptr(), u.data_ptr(),
                                        _lib.stream(dev)), "mdkk_snap_pair_u")
        fc = torch.from_numpy(np.ascontiguousarray(nmap.fc[lo:hi])).to(dev)
        wu = torch.view_as_real(u * fc[:, None]).reshape(m, 2 * nf).contiguous()
        rows = torch.from_numpy(np.asarray(nmap.rows[lo:hi], dtype=np.int64)).to(dev)
        ordered_scatter(torch.view_as_real(U).reshape(-1, 2 * nf), 2 * nf, 2 * nf, rows, wu)
    st.U_dev[: max(n, 1)].copy_(U)
    st.U.modified_a = False
    st.U.mark_modified("b")
    _put(state.U, state.layout, n, U[:n].cpu().numpy())


def _upload_u(state, st) -> None:
    n = st.n_atoms
    if n:
        st.U_dev[:n].copy_(torch.from_numpy(np.ascontiguousarray(state.u_view())).to(st.device))
    st.U.modified_a = False
    st.U.mark_modified("b")


def compute_yi(state) -> None:
    """mdkk compute_yi (mdkk/snap/compute.py:303-340): the adjoint Y on the GPU (Z-list
    kernel over the half set), expanded to the reference layout and written back."""
    st = _state(state)
    _upload_u(state, st)
    _sc.compute_yi(st)
    st.expand_y()
    _put(state.Y, state.layout, st.n_atoms, st.Y_dev[: st.n_atoms].cpu().numpy())


def compute_bi_complex(state) -> np.ndarray:
    st = _state(state)
    _upload_u(state, st)
    return _sc.compute_bi_complex(st)


def compute_bi(state) -> np.ndarray:
    return compute_bi_complex(state).real


def _scatter_pair_forces(f: torch.Tensor, rows: torch.Tensor, cols: torch.Tensor, t: torch.Tensor) -> None:
    """F[row] += t then F[col] -= t, each in pair order (np.add.at / np.subtract.at)."""
    ordered_scatter(f, 3, 3, rows, t)
    ordered_scatter(f, 3, 3, cols, -t)


def _y_rows(state, st) -> torch.Tensor:
    n = st.n_atoms
    y = torch.zeros((max(n, 1), st.index.n_flat), dtype=torch.complex128, device=st.device)
    if n:
        y[:n].copy_(torch.from_numpy(np.ascontiguousarray(state.y_view())).to(st.device))
    return y


def _wdu(st, dr: np.ndarray, r_c: float) -> torch.Tensor:
    m = len(dr)
    d = torch.from_numpy(np.ascontiguousarray(dr, dtype=np.float64)).to(st.device)
    out = torch.empty((max(m, 1), 3, st.index.n_flat), dtype=torch.complex128, device=st.device)
    _lib.check(_lib.lib().mdkk_snap_duidrj(st.handle().ptr, m, d.data_ptr(), r_c, out.data_ptr(),
                                           _lib.stream(st.device)), "mdkk_snap_duidrj")
    return out[:m]


def _forces_from(nmap, state, st, n_total: int, wdu_of) -> np.ndarray:
    y = _y_rows(state, st)
    f = torch.zeros((max(n_total, 1), 3), dtype=torch.float64, device=st.device)
    for lo, hi in _chunks(nmap.n_pairs, state):
        m = hi - lo
        rows32 = torch.from_numpy(np.asarray(nmap.rows[lo:hi], dtype=np.int32)).to(st.device)
        w = wdu_of(lo, hi)
        t = torch.empty((m, 3), dtype=torch.float64, device=st.device)
        _lib.check(_lib.lib().mdkk_snap_pair_dedr(st.handle().ptr, m, rows32.data_ptr(), y.data_ptr(),
                                                  w.data_ptr(), t.data_ptr(), _lib.stream(st.device)),
                   "mdkk_snap_pair_dedr")
        cols = torch.from_numpy(np.asarray(nmap.cols[lo:hi], dtype=np.int64)).to(st.device)
        _scatter_pair_forces(f, rows32.long(), cols, t)
    return f[:n_total].cpu().numpy()


def compute_fused_deidrj(nmap, state, n_total: int) -> np.ndarray:
    """mdkk compute_fused_deidrj (mdkk/snap/compute.py:390-409): per pair chunk the
    derivative recursion (k_snap_duidrj) and the contraction against Y on the GPU,
    forces scattered to both endpoints in pair order."""
    st = _state(state)
    return _forces_from(nmap, state, st, n_total, lambda lo, hi: _wdu(st, nmap.dr[lo:hi], nmap.r_c))


def compute_duidrj(nmap, state) -> np.ndarray:
    """mdkk compute_duidrj (mdkk/snap/compute.py:412-422): staged d(f_c u)/d dr, (P, 3, F)."""
    st = _state(state)
    out = np.empty((nmap.n_pairs, 3, st.index.n_flat), dtype=np.complex128)
    for lo, hi in _chunks(nmap.n_pairs, state):
        out[lo:hi] = _wdu(st, nmap.dr[lo:hi], nmap.r_c).cpu().numpy()
    return out


def compute_deidrj(nmap, state, du, n_total: int) -> np.ndarray:
    """mdkk compute_deidrj (mdkk/snap/compute.py:425-436): staged contraction on the GPU."""
    st = _state(state)
    return _forces_from(nmap, state, st, n_total, lambda lo, hi: torch.from_numpy(
        np.ascontiguousarray(du[lo:hi], dtype=np.complex128)).to(st.device))


# ----------------------------------------------------------------- styles
class LJStyleKK:
    """`lj/cut/kk` in the reference engine (mdkk/driver/simulation.py:65-85 protocol)."""

    list_style = None

    def __init__(self, r_c: float, mode: str = "atom", name: str = "lj/cut/kk"):
        self.name = name
        self.r_c = float(r_c)
        self.default_mode = mode
        self.kernel = None

    def set_coeff(self, epsilon: float, sigma: float) -> None:
        mp = _mdkk().pair_lj
        self.kernel = mp.LJCut(mp.PairParams(epsilon, sigma, self.r_c))

    def compute(self, system, lists, config):
        if self.kernel is None:
            raise _mdkk().driver.simulation.RunError("pair_coeff must be set before computing forces")
        return compute_pair(self.kernel, system, lists, mode=config.mode or self.default_mode,
                            strategy=config.make_strategy(), n_workers=config.workers)


class SnapStyleKK:
    """`snap/kk` in the reference engine (mdkk/driver/simulation.py:88-142 protocol): per rank
    the fused device pipeline over the list table (ui -> yi(+E) -> deidrj), then the
    reference's reverse comm."""

    list_style = "full"

    def __init__(self, r_c: float, jmax: float, beta, name: str = "snap/kk", batch_u: int = 4, batch_y: int = 1,
                 tile_v: int = 0, layout: str = "a"):
        self.name = name
        self.r_c = float(r_c)
        self.tables = make_coupling_tables(jmax)
        self.beta = np.asarray(beta, dtype=np.float64)
        self.knobs = dict(batch_u=batch_u, batch_y=batch_y, tile_v=tile_v, layout=layout)
        self._states: dict = {}

    @classmethod
    def from_file(cls, r_c: float, path: str, **kw) -> "SnapStyleKK":
        jmax, beta = _mdkk().snap.read_coeff_file(path)
        return cls(r_c, jmax, beta, **kw)

    def set_coeff(self, *_):
        raise _mdkk().driver.simulation.RunError("snap styles read coefficients from their file; "
                                                 "pair_coeff does not apply")

    def compute(self, system, lists, config):
        mp = _mdkk().pair_lj
        knobs = {k: (getattr(config, k) if getattr(config, k, None) is not None else v)
                 for k, v in self.knobs.items()}
        energy = torch.zeros((), dtype=torch.float64, device=_dev())
        for idx, (store, nlist) in enumerate(zip(system.stores, lists)):
            nlist.check_current()
            mirror = _mirror(store)
            nl = _device_list(nlist, mirror)
            nmap = _sc.build_neighbor_map(mirror, nl, self.r_c)
            key = (idx, store.n_local, tuple(sorted(knobs.items())))
            st = self._states.get(key)
            if st is None:
                self._states = {k: v for k, v in self._states.items() if k[0] != idx}
                st = self._states[key] = _sc.SnapState(self.tables, store.n_local, self.beta, device=mirror.device,
                                                       **knobs)
            _sc.compute_ui(nmap, st)
            _sc.compute_yi(st)
            mirror.f.zero_()
            _sc.deidrj_device(nmap, st, mirror.f)
            _sc.check_flags(st)
            energy = energy + st.energy_dev[0]
            if store.n_total:
                fr = store.force.read("a")
                fr[: store.n_total] = mirror.f[: store.n_total, :3].cpu().numpy()
                store.force.mark_modified("a")
        system.reverse_comm()
        return mp.PairResult(float(energy.item()), system.gather_forces(), np.zeros(6))


def register(registry) -> None:
    """Add the /kk styles to an mdkk StyleRegistry (mdkk/driver/registry.py:24-33)."""
    registry.register("lj/cut/kk", lambda args: LJStyleKK(float(args[0]), mode="atom"))
    registry.register("lj/cut/opt/kk", lambda args: LJStyleKK(float(args[0]), mode="neighbor",
                                                              name="lj/cut/opt/kk"))
    registry.register("snap/kk", lambda args: SnapStyleKK.from_file(float(args[0]), args[1]))
    registry.register("snap/opt/kk", lambda args: SnapStyleKK.from_file(float(args[0]), args[1], name="snap/opt/kk",
                                                                        batch_u=8, tile_v=256))


# ---------------------------------------------------------------- install
_REBIND = {
    ("neighbor", "build"): build,
    ("neighbor", "brute_force_pairs"): brute_force_pairs,
    ("pair_lj", "compute_pair"): compute_pair,
    ("snap.compute", "compute_ui"): compute_ui,
    ("snap.compute", "compute_yi"): compute_yi,
    ("snap.compute", "compute_fused_deidrj"): compute_fused_deidrj,
    ("snap.compute", "compute_duidrj"): compute_duidrj,
    ("snap.compute", "compute_deidrj"): compute_deidrj,
    ("snap.compute", "compute_bi"): compute_bi,
    ("snap.compute", "compute_bi_complex"): compute_bi_complex,
    ("snap.compute", "pair_u_flat"): pair_u_flat,
}
_installed: list = []


def install() -> list[str]:
    """Rebind mdkk's hot-path functions to the GPU adapters in every loaded mdkk module
    (names imported with `from ... import` included) and extend `default_registry()` with
    the /kk styles.  Import mdkk's modules first; test modules imported afterwards bind
    the adapters.  Returns the rebound names."""
    import importlib
    mdkk = _mdkk()
    for sub in ("neighbor", "pair_lj", "snap", "snap.compute", "driver", "driver.simulation", "driver.bench"):
        importlib.import_module(f"mdkk.{sub}")
    originals = {}
    for (mod, name), new in _REBIND.items():
        originals[id(getattr(importlib.import_module(f"mdkk.{mod}"), name))] = (name, new)
    done = []
    for mname, mod in list(sys.modules.items()):
        if mod is None or not (mname == "mdkk" or mname.startswith("mdkk.")):
            continue
        for attr, val in list(vars(mod).items()):
            hit = originals.get(id(val))
            if hit is not None and hit[0] == attr:
                _installed.append((mod, attr, val))
                setattr(mod, attr, hit[1])
                done.append(f"{mname}.{attr}")
    sim = mdkk.driver.simulation
    base = sim.default_registry

    def default_registry():
        reg = base()
        register(reg)
        return reg
    _installed.append((sim, "default_registry", base))
    sim.default_registry = default_registry
    if getattr(mdkk.driver, "default_registry", None) is base:
        _installed.append((mdkk.driver, "default_registry", base))
        mdkk.driver.default_registry = default_registry
    return done


def uninstall() -> None:
    """Restore everything `install()` rebound."""
    while _installed:
        mod, attr, val = _installed.pop()
        setattr(mod, attr, val)
