"""`snap` / `snap/kk` pair style: the descriptor pipeline per rank + reverse comm (mdkk/driver/simulation.py:88-142)."""

from __future__ import annotations

import numpy as np
import torch

from ..pair_lj import PairResult
from .compute import SnapState, build_neighbor_map, check_flags, compute_ui, compute_yi, deidrj_device
from .coupling import make_coupling_tables, read_coeff_file


class SnapStyle:
    list_style = "full"  # the expansion needs every neighbour of every atom

    def __init__(self, r_c: float, jmax: float, beta, name: str = "snap/kk", batch_u: int = 4, batch_y: int = 2,
                 tile_v: int = 0, layout: str = "a"):
        self.name = name
        self.r_c = float(r_c)
        self.tables = make_coupling_tables(jmax)
        self.beta = np.asarray(beta, dtype=np.float64)
        self.knobs = dict(batch_u=batch_u, batch_y=batch_y, tile_v=tile_v, layout=layout)
        self._states: dict = {}

    @classmethod
    def from_file(cls, r_c: float, path: str, **kw) -> "SnapStyle":
        jmax, beta = read_coeff_file(path)
        return cls(r_c, jmax, beta, **kw)

    def set_coeff(self, *_):
        from ..driver.simulation import RunError
        raise RunError("snap styles read coefficients from their file; pair_coeff does not apply")

    def _knobs(self, config) -> dict:
        """RunConfig knobs override the style's own (mdkk/driver/simulation.py:115-121)."""
        k = dict(self.knobs)
        for name in ("batch_u", "batch_y", "tile_v", "layout"):
            v = getattr(config, name, None) if config is not None else None
            if v is not None:
                k[name] = v
        return k

    def _state(self, idx, store, config=None):
        knobs = self._knobs(config)
        key = (idx, store.n_local, tuple(sorted(knobs.items())))
        st = self._states.get(key)
        if st is None:
            self._states = {k: v for k, v in self._states.items() if k[0] != idx}
            # the coupling table handle is shared across states of the same style
            st = SnapState(self.tables, store.n_local, self.beta, device=store.device, **knobs)
            for other in self._states.values():
                st._handle = other._handle
                break
            self._states[key] = st
        return st

    def compute_device(self, system, lists, config):
        """Engine path (no host sync): U -> Y(+E) -> fused forces -> reverse comm."""
        e = torch.zeros((), dtype=torch.float64, device=system.device)
        states = []
        for idx, (store, nl) in enumerate(zip(system.stores, lists)):
            nmap = build_neighbor_map(store, nl, self.r_c)
            st = self._state(idx, store, config)
            compute_ui(nmap, st)
            compute_yi(st)
            store.f[: store.n_total].zero_()
            deidrj_device(nmap, st, store.f)
            store.device_wrote(force=True)
            e = e + st.energy_dev[0]
            states.append(st)
        system.reverse_comm()
        self._last = states
        return e, states[0].flags if states else torch.zeros(1, dtype=torch.int32, device=system.device)

    def compute(self, system, lists, config, check: bool = True) -> PairResult:
        if check:
            for nl in lists:
                nl.check_current()
        e, _ = self.compute_device(system, lists, config)
        if check:
            for st in self._last:
                check_flags(st)
        ev = torch.zeros(7, dtype=torch.float64, device=system.device)
        ev[0] = e
        return PairResult(ev, system)  # virial not computed for SNAP (mdkk/driver/simulation.py:142)
