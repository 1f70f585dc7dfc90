"""Lennard-Jones pair engine on the GPU (drop-in for mdkk/pair_lj.py).

`PairParams`, `LJCut`, `PairResult`, `u2_lj` and `compute_pair` keep the
reference signatures (mdkk/pair_lj.py:29-179).  `compute_pair` launches the
sm_100a kernel `mdkk_lj_force` per rank — owner-writes for full lists, FP64
atomics for half lists (or the Serial / Duplicate ScatterAccumulator
strategies, `mdkk_lj_force_strategy`) — then the device reverse comm; energy
and the six virial components come from a deterministic on-device reduction.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .domain import RankedSystem
from .memspace import STRATEGIES, Duplicate, Serial, combine_copies, ordered_scatter, worker_count
from .neighbor import STYLES, NeighborList


class PairError(RuntimeError):
    pass


class PairParams:
    """epsilon, sigma, r_c with the reference validation (mdkk/pair_lj.py:29-39)."""

    def __init__(self, epsilon: float, sigma: float, r_c: float):
        if epsilon <= 0 or sigma <= 0 or r_c <= 0:
            raise PairError("epsilon, sigma, r_c must all be positive")
        if r_c <= sigma:
            raise PairError(f"cutoff {r_c} must exceed sigma {sigma}")
        self.epsilon, self.sigma, self.r_c = float(epsilon), float(sigma), float(r_c)


def u2_lj(r: float, params: PairParams) -> tuple[float, float]:
    """Scalar closed form (energy, fpair) for one distance (mdkk/pair_lj.py:55-69)."""
    if r == 0:
        raise PairError("coincident atoms (r = 0)")
    if not (0 < r < params.r_c):
        raise PairError(f"r = {r} outside (0, r_c = {params.r_c})")
    s2 = (params.sigma * params.sigma) / (r * r)
    s6 = s2 * s2 * s2
    return 4.0 * params.epsilon * (s6 * s6 - s6), 24.0 * params.epsilon * (2.0 * s6 * s6 - s6) / (r * r)


class LJCut:
    """Truncated (not shifted) 12-6 kernel (mdkk/pair_lj.py:72-91); evaluated by csrc/lj.cu."""

    name = "lj/cut"

    def __init__(self, params: PairParams):
        self.params = params
        self.r_c = params.r_c

    def pair_energy_force(self, r2):
        """(e, fpair) on squared distances, all < r_c^2 (mdkk/pair_lj.py:81-91).

        Element-wise on whatever it is given: a numpy array returns numpy
        arrays, a device tensor stays on the device.  The force engine does not
        call this; csrc/lj.cu evaluates the same expressions in the same order."""
        is_t = torch.is_tensor(r2)
        x = r2 if is_t else np.asarray(r2, dtype=np.float64)
        if x.numel() if is_t else x.size:
            if float(x.min()) <= 0.0:
                raise PairError("coincident atoms (r = 0)")
        p = self.params
        s2 = (p.sigma * p.sigma) / x
        s6 = s2 * s2 * s2
        s12 = s6 * s6
        e = 4.0 * p.epsilon * (s12 - s6)
        fp = 24.0 * p.epsilon * (2.0 * s12 - s6) / x
        return e, fp


class PairResult:
    """Energy, gid-ordered forces, virial (xx,yy,zz,xy,xz,yz) — read lazily from the device."""

    def __init__(self, ev: torch.Tensor, system: RankedSystem | None, flags: torch.Tensor | None = None):
        self._ev = ev
        self._system = system
        self._flags = flags
        self._energy = self._virial = self._forces = None

    def _host_ev(self):
        if self._energy is None:
            if self._flags is not None and int(self._flags.item()) & _lib.FLAG_COINCIDENT:
                raise PairError("coincident atoms (r = 0)")
            ev = self._ev.cpu().numpy()
            self._energy, self._virial = float(ev[0]), ev[1:7].copy()

    @property
    def energy(self) -> float:
        self._host_ev()
        return self._energy

    @property
    def virial(self) -> np.ndarray:
        self._host_ev()
        return self._virial

    @property
    def forces(self) -> np.ndarray:
        if self._forces is None:
            self._forces = self._system.gather_forces()
        return self._forces

    def pressure(self, volume: float) -> float:
        return float(self.virial[:3].sum() / (3.0 * volume))


def lj_force_rank(store, nl: NeighborList, params: PairParams, ev: torch.Tensor, flags: torch.Tensor,
                  zero: bool = True, virial: bool = True, mode: str = "atom", gate: torch.Tensor | None = None,
                  gate_limit: float = 0.0, integ: dict | None = None, strategy=None) -> None:
    """One rank's kernel launch (no host sync).

    Ghost force rows are zero outside a force evaluation (migrate zeroes all
    rows, reverse comm zeroes ghosts, full-list kernels write owner rows
    only), so only the half list (owner rows accumulate with atomics) needs
    a clear.  `gate` (engine-internal, device double): the launch is
    speculative and does nothing when sqrt(gate) > gate_limit (a rebuilding
    step, which relaunches after its rebuild).
    """
    dev = store.device
    if zero and nl.style == "half":
        store.f.zero_()
    # mode "atom": one thread per owned atom; "neighbor": a team of lanes per atom
    # splitting its list (mdkk/pair_lj.py:118-143)
    pend = nl._pending
    if integ is not None and integ.get("pack") is not None:
        # ... + the next step's periodic ghost rows in the reduction's launch (one rank)
        ln, shifts = integ["pack"]
        _lib.check(_lib.lib().mdkk_lj_force_integrate_pack(
            _lib.ctx(dev), store.x.data_ptr(), store.n_local, nl.table_dev.data_ptr(), nl.counts_dev.data_ptr(),
            nl.alloc_cap, int(virial), params.epsilon, params.sigma, params.r_c, store.f.data_ptr(), ev.data_ptr(),
            flags.data_ptr(), gate.data_ptr() if gate is not None else None, gate_limit,
            pend[0].data_ptr() if pend is not None else None, nl.alloc_cap, store.v.data_ptr(),
            nl.ref_dev.data_ptr(), integ["x_next"].data_ptr(), integ["d2_next"].data_ptr(), integ["dt"], integ["h"],
            ln.idx.data_ptr(), ln.code.data_ptr(), shifts.data_ptr(), ln.count,
            integ["d2_zero"].data_ptr() if integ.get("d2_zero") is not None else None, _lib.stream(dev)),
            "mdkk_lj_force_integrate_pack")
        return
    if integ is not None:
        # full list + velocity-Verlet epilogue (engine advance loop; mdkk_lj_force_integrate)
        _lib.check(_lib.lib().mdkk_lj_force_integrate(
            _lib.ctx(dev), store.x.data_ptr(), store.n_local, nl.table_dev.data_ptr(), nl.counts_dev.data_ptr(),
            nl.alloc_cap, int(virial), params.epsilon, params.sigma, params.r_c, store.f.data_ptr(), ev.data_ptr(),
            flags.data_ptr(), gate.data_ptr() if gate is not None else None, gate_limit,
            pend[0].data_ptr() if pend is not None else None, nl.alloc_cap, integ["mode"], store.v.data_ptr(),
            nl.ref_dev.data_ptr(), integ["x_next"].data_ptr() if integ["mode"] == 2 else None,
            integ["d2_next"].data_ptr() if integ["mode"] == 2 else None, integ["dt"], integ["h"],
            integ["flags"].data_ptr() if integ.get("part") else None, int(integ.get("part", 0)),
            _lib.stream(dev)), "mdkk_lj_force_integrate")
        return
    if gate is not None or pend is not None:
        # speculative launch: skipped on the device if the step rebuilds (gate) or the
        # deferred build overflowed its table (count gate; see NeighborList.settle)
        _lib.check(_lib.lib().mdkk_lj_force_gated(
            _lib.ctx(dev), store.x.data_ptr(), store.n_local, nl.table_dev.data_ptr(), nl.counts_dev.data_ptr(),
            nl.alloc_cap, STYLES[nl.style], int(nl.newton), int(virial), int(mode == "neighbor"), params.epsilon,
            params.sigma, params.r_c, store.f.data_ptr(), ev.data_ptr(), flags.data_ptr(),
            gate.data_ptr() if gate is not None else None, gate_limit,
            pend[0].data_ptr() if pend is not None else None, nl.alloc_cap, _lib.stream(dev)),
            "mdkk_lj_force_gated")
        return
    if nl.style == "half" and isinstance(strategy, (Serial, Duplicate)):
        _half_with_strategy(store, nl, params, ev, flags, virial, strategy)
        return
    fn = "mdkk_lj_force_neighbor" if mode == "neighbor" else "mdkk_lj_force"
    _lib.check(getattr(_lib.lib(), fn)(
        _lib.ctx(dev), store.x.data_ptr(), store.n_local, nl.table_dev.data_ptr(), nl.counts_dev.data_ptr(),
        nl.alloc_cap, STYLES[nl.style], int(nl.newton), int(virial), params.epsilon, params.sigma, params.r_c,
        store.f.data_ptr(), ev.data_ptr(), flags.data_ptr(), _lib.stream(dev)), fn)


def _half_with_strategy(store, nl: NeighborList, params: PairParams, ev, flags, virial: bool, strategy) -> None:
    """Half-list force with the partner writes deconflicted by `strategy`
    (mdkk/pair_lj.py:138-165 through ScatterAccumulator, mdkk/memspace.py:198-254).

    Duplicate: the kernel's REDs go into `copies` staging copies (copy = block %
    copies), combined in a fixed order into f.  Serial: the kernel stores own rows
    and stages every partner contribution per table entry (no atomics); they are
    applied in (row, slot) order by the ordered scatter -- run-to-run deterministic.
    The strategy kernels run the atom-parallel schedule."""
    dev = store.device
    L = _lib.lib()
    f = store.f
    if isinstance(strategy, Duplicate):
        stage = torch.zeros((strategy.copies,) + tuple(f.shape), dtype=torch.float64, device=dev)
        _lib.check(L.mdkk_lj_force_strategy(
            _lib.ctx(dev), store.x.data_ptr(), store.n_local, nl.table_dev.data_ptr(), nl.counts_dev.data_ptr(),
            nl.alloc_cap, int(nl.newton), int(virial), params.epsilon, params.sigma, params.r_c, f.data_ptr(),
            ev.data_ptr(), flags.data_ptr(), 1, stage.data_ptr(), int(f.numel()), strategy.copies,
            _lib.stream(dev)), "mdkk_lj_force_strategy")
        combine_copies(stage, f)
        return
    ncl, cap = nl.table_dev.shape[0], nl.alloc_cap
    stage = torch.zeros((ncl, cap, 32, 4), dtype=torch.float64, device=dev)
    _lib.check(L.mdkk_lj_force_strategy(
        _lib.ctx(dev), store.x.data_ptr(), store.n_local, nl.table_dev.data_ptr(), nl.counts_dev.data_ptr(),
        cap, int(nl.newton), int(virial), params.epsilon, params.sigma, params.r_c, f.data_ptr(), ev.data_ptr(),
        flags.data_ptr(), 2, stage.data_ptr(), 0, 1, _lib.stream(dev)), "mdkk_lj_force_strategy")
    n = store.n_local * cap
    ent = stage.permute(0, 2, 1, 3).reshape(-1, 4)[:n]           # (row, slot) order
    tab = nl.table_dev.permute(0, 2, 1).reshape(-1)[:n]
    used = ent[:, 3] != 0
    ordered_scatter(f, 4, 3, tab[used].long(), ent[used, :3].contiguous())


def compute_pair(kernel, system: RankedSystem, lists: list[NeighborList], mode: str = "atom", strategy=None,
                 n_workers: int | None = None, zero_forces: bool = True, check: bool = True) -> PairResult:
    """Evaluate the LJ kernel over every rank's list (mdkk/pair_lj.py:114-179).

    `mode` picks the GPU schedule: "atom" = one thread per owned atom,
    "neighbor" = a team of lanes per atom over its list (the reference's
    mid-row split).  `strategy` deconflicts the half list's partner writes
    (Serial = staged + ordered, deterministic; Duplicate = staging copies;
    Atomic = FP64 RED; None = Atomic, the engine default); full lists write
    owner rows only, so every strategy is the same owner-write kernel there.
    `n_workers` (capped by MDKK_THREADS as in mdkk/parallel.py) sizes a
    Duplicate without an explicit copy count.  `check=False` (engine-internal) skips the
    synchronous stale-list and coincident-atom checks; the error word is then
    read when the result is first inspected.
    """
    if mode not in ("atom", "neighbor"):
        raise PairError(f"unknown execution mode {mode!r}")
    if strategy is not None and not isinstance(strategy, STRATEGIES):
        raise PairError(f"unknown scatter strategy {strategy!r}")
    workers = worker_count(n_workers)
    if isinstance(strategy, Duplicate) and n_workers is not None:
        strategy = Duplicate(min(strategy.copies, workers))
    params = kernel.params
    dev = system.device
    evs = torch.zeros((len(system.stores), 7), dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    prev = None
    if not zero_forces:
        prev = [s.f.clone() for s in system.stores]
    half = False
    for k, (store, nl) in enumerate(zip(system.stores, lists)):
        if check:
            nl.check_current()
        store.to_device()
        half |= nl.style == "half"
        lj_force_rank(store, nl, params, evs[k], flags, mode=mode, strategy=strategy)
        store.device_wrote(force=True)
    if half and any(s.n_ghost for s in system.stores):
        if isinstance(strategy, Serial):
            system.reverse_comm(ordered=True)
        else:
            system.reverse_comm()
    if prev is not None:
        for s, p in zip(system.stores, prev):
            s.f[: s.n_local] += p[: s.n_local]
    ev = evs.sum(dim=0) if len(system.stores) > 1 else evs[0]
    res = PairResult(ev, system, flags)
    if check:
        res._host_ev()  # raise PairError now, as the reference does
    return res
