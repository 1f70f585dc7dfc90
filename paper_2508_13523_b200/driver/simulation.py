"""Device-resident velocity-Verlet driver (mirror of mdkk/driver/simulation.py).

`RunConfig`, `LJStyle`, `SnapStyle`, `default_registry`, `Simulation`,
`run_script`, `RunResult`, `lattice_positions`, `seeded_velocities` keep the
reference names and semantics (mdkk/driver/simulation.py:36-488).  x, v, f
never leave HBM inside the loop: one step is

    verlet_first (kick + drift + max|x - x_ref|^2)  ->  1 scalar D2H (rebuild?)
    [migrate + rebuild | forward pack]  ->  force kernel (+ reverse fold)
    ->  verlet_second (kick)

and energies / kinetic energy / the non-finite check are read back only on
thermo steps.  Styles `lj/cut/kk` and `snap/kk` are the B200 drop-ins; the
base names resolve to the same GPU styles (there is no CPU path here).
"""

from __future__ import annotations

import gc
import math

import numpy as np
import torch

from .. import _lib
from ..domain import Box, RankedSystem
from ..memspace import Atomic, Duplicate, Serial, pinned_array
from ..neighbor import build, build_all
from ..pair_lj import LJCut, PairParams, PairResult, compute_pair, lj_force_rank
from .registry import StyleRegistry
from .script import parse_script


class RunError(RuntimeError):
    pass


class RunConfig:
    """Harness knobs (mdkk/driver/simulation.py:36-62) plus `device`."""

    def __init__(self, n_ranks: int = 1, strategy: str | None = None, mode: str | None = None,
                 list_style: str | None = None, newton: bool = True, skin: float = 0.3,
                 workers: int | None = None, batch_u: int | None = None, batch_y: int | None = None,
                 tile_v: int | None = None, layout: str | None = None, rng_seed: int | None = None,
                 device=None, distributed: bool = False):
        # None = the device default (owner writes for full lists, FP64 RED for half
        # lists); an explicit name selects that ScatterAccumulator strategy for the
        # half list's partner writes (the reference defaults to "serial")
        if strategy is not None and strategy not in ("serial", "duplicate", "atomic"):
            raise RunError(f"unknown strategy {strategy!r}; choose from ['atomic', 'duplicate', 'serial']")
        self.n_ranks = int(n_ranks)
        self.strategy = strategy
        self.mode = mode
        self.list_style = list_style
        self.newton = bool(newton)
        self.skin = float(skin)
        self.workers = workers
        self.batch_u, self.batch_y, self.tile_v, self.layout = batch_u, batch_y, tile_v, layout
        self.rng_seed = rng_seed
        self.device = device
        # one brick per process over torch.distributed (NCCL) instead of in-process logical ranks
        self.distributed = bool(distributed)

    def make_strategy(self):
        """The strategy object compute_pair receives (mdkk/driver/simulation.py:58-59)."""
        if self.strategy is None:
            return None
        return {"serial": Serial, "atomic": Atomic}.get(self.strategy, lambda: Duplicate(self.workers))()


class LJStyle:
    """Truncated 12-6 pair style on the GPU (mdkk/driver/simulation.py:65-85)."""

    list_style = None
    supports_gate = True     # compute_device can be launched speculatively (see Simulation._half_kick_drift)

    def __init__(self, r_c: float, mode: str = "atom", name: str = "lj/cut/kk"):
        self.name = name
        self.r_c = float(r_c)
        self.default_mode = mode
        self.kernel = None

    def set_coeff(self, epsilon: float, sigma: float) -> None:
        self.kernel = LJCut(PairParams(epsilon, sigma, self.r_c))

    def compute(self, system, lists, config: RunConfig, check: bool = True) -> PairResult:
        if self.kernel is None:
            raise RunError("pair_coeff must be set before computing forces")
        return compute_pair(self.kernel, system, lists, mode=config.mode or self.default_mode,
                            strategy=config.make_strategy(), n_workers=config.workers, check=check)

    def compute_device(self, system, lists, config, gate=None, gate_limit: float = 0.0, integ=None
                       ) -> tuple[torch.Tensor, torch.Tensor]:
        """Engine path: no host sync; returns (device energy scalar, device flag word).
        With `gate` the launch is speculative (a no-op when sqrt(gate) > gate_limit)."""
        if self.kernel is None:
            raise RunError("pair_coeff must be set before computing forces")
        dev = system.device
        # persistent per-system buffers: the kernels overwrite ev; the flag word is
        # sticky (checked on thermo steps: "at or before step N")
        key = (id(system), len(system.stores), str(dev))
        if getattr(self, "_bufkey", None) != key:
            self._bufkey = key
            self._evs = torch.zeros((2, len(system.stores), 7), dtype=torch.float64, device=dev)
            self._flags = torch.zeros(1, dtype=torch.int32, device=dev)
            self._slot = 0
        # two energy slots used in turn: a step's returned energy stays valid while the
        # next step's (speculative) launch is already queued (the per-step non-finite check);
        # a halo-overlap part 1 writes no energy (part 2 reduces both) and keeps the slot
        if integ is None or integ.get("part", 0) != 1:
            self._slot ^= 1
        evs, flags = self._evs[self._slot], self._flags
        half = False
        for k, (s, nl) in enumerate(zip(system.stores, lists)):
            lj_force_rank(s, nl, self.kernel.params, evs[k], flags, virial=False,
                          mode=config.mode or self.default_mode, gate=gate, gate_limit=gate_limit, integ=integ,
                          strategy=config.make_strategy())
            half |= nl.style == "half"
        if half:   # collective in the distributed system: every rank calls it
            system.reverse_comm(ordered=config.strategy == "serial")
        for s in system.stores:
            s.device_wrote(force=True, vel=integ is not None)
        return (evs[:, 0].sum() if len(system.stores) > 1 else evs[0, 0]), flags


def default_registry() -> StyleRegistry:
    """lj/cut, lj/cut/opt, lj/cut/kk, snap, snap/opt, snap/kk -> GPU styles (mdkk/driver/simulation.py:145-153)."""
    reg = StyleRegistry()
    for name in ("lj/cut", "lj/cut/opt", "lj/cut/kk"):
        reg.register(name, lambda args, _n=name: LJStyle(float(args[0]),
                                                         mode="neighbor" if _n.endswith("opt") else "atom",
                                                         name=_n))
    try:
        from ..snap.style import SnapStyle
    except ImportError:  # SNAP kernels not built into this library version
        SnapStyle = None
    if SnapStyle is not None:
        for name in ("snap", "snap/kk"):
            reg.register(name, lambda args, _n=name: SnapStyle.from_file(float(args[0]), args[1], name=_n))
        # the reference's opt preset (mdkk/driver/simulation.py:151-152)
        reg.register("snap/opt", lambda args: SnapStyle.from_file(float(args[0]), args[1], name="snap/opt",
                                                                  batch_u=8, tile_v=256))
    return reg


def lattice_positions(style: str, rho: float, cells) -> tuple[np.ndarray, Box]:
    """fcc/sc sites in meshgrid(ij) cell x basis order (mdkk/driver/simulation.py:156-178).

    `bcc` (absent from the reference) takes the lattice constant a as `rho`.
    """
    if rho <= 0:
        raise RunError("lattice density must be positive")
    if style == "fcc":
        a = (4.0 / rho) ** (1.0 / 3.0)
        base = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]])
    elif style == "sc":
        a = (1.0 / rho) ** (1.0 / 3.0)
        base = np.zeros((1, 3))
    elif style == "bcc":
        a = float(rho)
        base = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.5]])
    else:
        raise RunError(f"unknown lattice style {style!r}")
    nx, ny, nz = (int(c) for c in cells)
    if min(nx, ny, nz) < 1:
        raise RunError("create_box needs at least one cell per direction")
    ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    corners = np.stack([ii, jj, kk], axis=-1).reshape(-1, 3).astype(np.float64)
    pos = (corners[:, None, :] + base[None, :, :]).reshape(-1, 3) * a
    return pos, Box((a * nx, a * ny, a * nz))


def seeded_velocities(n: int, temperature: float, mass: float, seed: int) -> np.ndarray:
    """Gaussian, zero momentum, exact-T rescale (mdkk/driver/simulation.py:181-194)."""
    if temperature < 0:
        raise RunError("temperature must be non-negative")
    if temperature == 0.0 or n == 0:
        return np.zeros((n, 3))
    v = np.random.default_rng(seed).normal(0.0, np.sqrt(temperature / mass), (n, 3))
    v -= v.mean(axis=0)
    t_now = mass * float(np.sum(v * v)) / (3.0 * n)
    if t_now > 0:
        v *= np.sqrt(temperature / t_now)
    return v


class RunResult:
    """Thermo rows, per-logged-step gid-ordered snapshots (mdkk/driver/simulation.py:197-210)."""

    def __init__(self):
        self.rows = []
        self.snapshots = {}
        self.qeq_log = []         # (step, iters_s, iters_t, sum_q, energy) (mdkk/driver/simulation.py:203)
        self.lines = []
        self.n_rebuilds = 0

    def log(self, step, e_pot, e_kin, temperature):
        e_total = e_pot + e_kin
        self.rows.append((step, e_pot, e_kin, e_total, temperature))
        self.lines.append(f"{step} {e_pot:.17g} {e_kin:.17g} {e_total:.17g} {temperature:.17g}")


class Simulation:
    """Executes a parsed script; the NVE loop runs device-resident (mdkk/driver/simulation.py:213-481)."""

    def __init__(self, config: RunConfig | None = None, registry: StyleRegistry | None = None, log=print):
        self.config = config or RunConfig()
        self.registry = registry or default_registry()
        self.log = log or (lambda *_: None)
        self.suffix = None
        self.lattice_spec = None
        self.cells = None
        self.box = None
        self.mass = 1.0
        self._positions = None
        self._velocities = None
        self.style = None
        self.dt = 0.005
        self.thermo_every = 100
        self.system: RankedSystem | None = None
        self.lists = None
        self.results: list[RunResult] = []
        self.n_rebuilds = 0
        self._cap_hint = None
        self.snapshots = True
        dev = self.config.device
        self.device = torch.device(dev) if dev is not None else torch.device("cuda", torch.cuda.current_device())
        self._d2 = None
        self._d2_host = None
        self._d2_ready = None      # event after the skin-test read-back
        self._spec_e = None        # energy of a speculatively launched force evaluation
        self._packed = False
        self._kick_pending = False
        self.qeq = None
        self._e_dev = None
        self._flags = None
        self._run_step = 0         # steps taken in the current run (the non-finite abort names them)
        self._e_prev = None        # device energy of the last completed step

    # ------------------------------------------------------------ commands
    def execute(self, script) -> "Simulation":
        cmds = parse_script(script) if isinstance(script, str) else script
        for cmd in cmds:
            handler = getattr(self, f"_cmd_{cmd.name}", None)
            if handler is None:
                raise RunError(f"line {cmd.line_no}: no handler for {cmd.name!r}")
            try:
                handler(cmd.args)
            except (RunError, ValueError) as exc:
                raise RunError(f"line {cmd.line_no} ({cmd.name}): {exc}") from exc
        return self

    def _cmd_units(self, a):
        if a[0] != "lj":
            raise RunError("only reduced units are supported")

    def _cmd_boundary(self, a):
        if tuple(a) != ("p", "p", "p"):
            raise RunError("only fully periodic boundaries are supported")

    def _cmd_lattice(self, a):
        self.lattice_spec = (a[0], float(a[1]))

    def _cmd_create_box(self, a):
        if self.lattice_spec is None:
            raise RunError("lattice must be set before create_box")
        self.cells = tuple(int(v) for v in a)
        _, self.box = lattice_positions(self.lattice_spec[0], self.lattice_spec[1], self.cells)

    def _cmd_create_atoms(self, a):
        if self.cells is None:
            raise RunError("create_box must run before create_atoms")
        pos, self.box = lattice_positions(self.lattice_spec[0], self.lattice_spec[1], self.cells)
        self._positions = pinned_array(pos)   # the run's upload is then one DMA per array
        self._velocities = pinned_array(np.zeros_like(pos))
        self.system = None

    def _cmd_mass(self, a):
        m = float(a[0])
        if m <= 0:
            raise RunError("mass must be positive")
        self.mass = m

    def _cmd_velocity(self, a):
        if self._positions is None:
            raise RunError("create_atoms must run before velocity")
        t, seed = float(a[0]), int(a[1])
        if self.config.rng_seed is not None:
            seed = self.config.rng_seed
        self._velocities = pinned_array(seeded_velocities(len(self._positions), t, self.mass, seed))
        self.system = None

    def _cmd_pair_style(self, a):
        self.style = self.registry.resolve(a[0], self.suffix)(a[1:])
        self.lists = None

    def _cmd_pair_coeff(self, a):
        if self.style is None:
            raise RunError("pair_style must be set before pair_coeff")
        self.style.set_coeff(float(a[0]), float(a[1]))

    def _cmd_qeq(self, a):
        """`qeq off` | `qeq on gamma eta chi cutoff` (mdkk/driver/simulation.py:306-311)."""
        from ..qeq import QeqParams
        if a[0] == "off":
            self.qeq = None
            return
        gamma, eta, chi, cutoff = (float(v) for v in a[1:])
        self.qeq = QeqParams(gamma=gamma, eta=eta, chi=chi, cutoff=cutoff)

    def _qeq_diagnostic(self, step: int, result: RunResult) -> None:
        """Charges on a one-rank copy at thermo steps (mdkk/driver/simulation.py:417-429), solved on the GPU."""
        if self.qeq is None:
            return
        from ..qeq import QeqSystem, build_matrix, qeq_energy, solve_qeq
        gp, gv, _ = self.system.gather()
        solo = RankedSystem.distribute(self.system.box, 1, gp, gv, device=self.device)
        qlists = build_all(solo, self.qeq.cutoff, self.config.skin, style="full", newton=False)
        store = solo.stores[0]
        H = build_matrix(store, qlists[0], self.qeq)
        qsys = QeqSystem(H, np.full(store.n_local, self.qeq.chi))
        q = solve_qeq(qsys)
        result.qeq_log.append((step, *qsys.iterations, float(q.sum()), qeq_energy(qsys)))

    def _cmd_suffix(self, a):
        self.suffix = None if a[0] == "off" else a[0]

    def _cmd_timestep(self, a):
        dt = float(a[0])
        if dt <= 0:
            raise RunError("timestep must be positive")
        self.dt = dt

    def _cmd_thermo(self, a):
        n = int(a[0])
        if n <= 0:
            raise RunError("thermo interval must be positive")
        self.thermo_every = n

    def _cmd_run(self, a):
        self.run_nve(int(a[0]))

    # --------------------------------------------------------- integration
    def _ensure_system(self):
        if self.style is None:
            raise RunError("pair_style must be set before run")
        if self._positions is None:
            raise RunError("create_atoms must run before run")
        if self.system is None:
            with torch.cuda.device(self.device):
                if self.config.distributed:
                    from ..dist import DistSystem
                    self.system = DistSystem.distribute(self.box, self._positions, self._velocities,
                                                        device=self.device)
                else:
                    self.system = RankedSystem.distribute(self.box, self.config.n_ranks, self._positions,
                                                          self._velocities, device=self.device)
            self.lists = None
        if self.lists is None:
            style_list = self.style.list_style or self.config.list_style or "half"
            if self.style.list_style and self.config.list_style and self.config.list_style != self.style.list_style:
                raise RunError(f"style {self.style.name} requires {self.style.list_style} lists")
            self._list_style = style_list
            self.lists = build_all(self.system, self.style.r_c, self.config.skin, style=style_list,
                                   newton=self.config.newton)
            self._cap_hint = max(nl.alloc_cap for nl in self.lists)
        if self._d2 is None:
            self._d2 = torch.zeros(max(self.config.n_ranks, 1), dtype=torch.float64, device=self.device)

    def _rebuild_lists(self, defer: bool = False):
        """migrate + build (mdkk/driver/simulation.py:368-373).  `defer`: the capacity
        check is left to `_settle_lists` (after a count-gated force launch)."""
        halo = self.style.r_c + self.config.skin
        # forces are recomputed right after (full lists overwrite every owned row, half
        # lists and SNAP clear the rows they accumulate into): no reset pass
        old = self.lists if self.lists is not None and len(self.lists) == len(self.system.stores) else None
        # one rank: the sort's position gather also fills the recycled skin-test reference
        ready = bool(self.system.migrate(halo, zero_forces=False,
                                         ref_out=old[0].ref_dev if old is not None and len(old) == 1 else None))
        old = self.lists if self.lists is not None and len(self.lists) == len(self.system.stores) else None
        if ready and old is None:
            ready = False
        if not ready and old is not None and all(o.ref_dev.shape[0] >= max(s.n_local, 1)
                                                 for o, s in zip(old, self.system.stores)):
            # the new lists' skin-test reference = the owned positions now: copied here, so the
            # device does it while the host prepares the build (not after the build kernel)
            for o, s in zip(old, self.system.stores):
                n = max(s.n_local, 1)
                o.ref_dev[:n].copy_(s.x[:n])
            ready = True
        self.lists = None   # the old lists are dead: their buffers are recycled
        self.lists = [build(s, self.system.box, self.style.r_c, self.config.skin, style=self._list_style,
                            newton=self.config.newton, cap_hint=self._cap_hint,
                            recycle=old[k] if old is not None else None, defer=defer, ref_ready=ready)
                      for k, s in enumerate(self.system.stores)]
        if not defer:
            self._cap_hint = max(nl.alloc_cap for nl in self.lists)
        self.n_rebuilds += 1

    def _settle_lists(self) -> bool:
        """Finish deferred builds; False when a table overflowed and was regrown."""
        ok = True
        for k, nl in enumerate(self.lists):
            self.lists[k], good = nl.settle()
            ok &= good
        self._cap_hint = max(nl.alloc_cap for nl in self.lists)
        return ok

    def _forces_device(self, gate=None, gate_limit: float = 0.0, integ=None):
        if gate is not None or integ is not None:
            e, flags = self.style.compute_device(self.system, self.lists, self.config, gate, gate_limit, integ)
        else:
            e, flags = self.style.compute_device(self.system, self.lists, self.config)
        self._e_dev, self._flags = e, flags
        return e

    def _compute_forces(self) -> float:
        return float(self._forces_device().item())

    def _kinetic(self) -> tuple[float, float]:
        lib, st = _lib.lib(), _lib.stream(self.device)
        ke = torch.zeros(len(self.system.stores), dtype=torch.float64, device=self.device)
        n = 0
        for k, s in enumerate(self.system.stores):
            s.to_device()
            _lib.check(lib.mdkk_kinetic(_lib.ctx(self.device), s.v.data_ptr(), s.n_local, self.mass,
                                        ke[k:].data_ptr(), st), "mdkk_kinetic")
            n += s.n_local
        tot = torch.stack([ke.sum(), torch.tensor(float(n), dtype=torch.float64, device=self.device)])
        k, n = (float(v) for v in self._global_sum(tot).cpu().numpy())
        return k, (2.0 * k / (3.0 * n) if n else 0.0)

    def _global_sum(self, t: torch.Tensor) -> torch.Tensor:
        if self.config.distributed:
            return self.system.allreduce_sum(t.clone())
        return t

    def _half_kick_drift(self) -> bool:
        """v += dt/2m f; x += dt v; returns whether any rank moved beyond skin/2 (one sync)."""
        lib, st = _lib.lib(), _lib.stream(self.device)
        ctx = _lib.ctx(self.device)
        h = 0.5 * self.dt / self.mass
        for k, (s, nl) in enumerate(zip(self.system.stores, self.lists)):
            s.to_device()
            _lib.check(lib.mdkk_verlet_first(ctx, s.x.data_ptr(), s.v.data_ptr(), s.f.data_ptr(),
                                             nl.ref_dev.data_ptr(), s.n_local, self.dt, h,
                                             self._d2[k:].data_ptr(), int(self._kick_pending), st),
                       "mdkk_verlet_first")
            s.device_wrote(pos=True, vel=True)
        self._kick_pending = False
        n = len(self.system.stores)
        worst = self._d2[0:1] if n == 1 else self._d2[:n].max().reshape(1)
        if self.config.distributed:   # any rank over skin/2 -> every rank rebuilds (mdkk/neighbor.py:230)
            worst = self.system.allreduce_max(worst)
        # the step's one host sync: a pinned 8-byte read-back, no reduction kernel for one rank
        if self._d2_host is None:
            self._d2_host = torch.zeros(1, dtype=torch.float64, pin_memory=True)
        # (distributed: `worst` is the all-reduced maximum, the same on every rank, so
        # the speculative halo exchange and force launch below stay collective-matched)
        # the read-back runs on a side stream: the compute stream goes straight on to the
        # speculative pack + force launch instead of waiting out the copy-engine round
        # trip (the next step's verlet_first, which rewrites the maximum, is only issued
        # after the host has waited for this copy)
        main = torch.cuda.current_stream(self.device)
        if self._d2_ready is None:
            self._d2_ready = torch.cuda.Event()
            self._d2_kicked = torch.cuda.Event()
            self._side = torch.cuda.Stream(self.device)
        self._d2_kicked.record(main)
        self._side.wait_event(self._d2_kicked)
        with torch.cuda.stream(self._side):
            self._d2_host.copy_(worst, non_blocking=True)
        self._d2_ready.record(self._side)
        # speculative halo refresh, queued behind the read-back: a plain step needs
        # it next, and a rebuild simply overwrites the ghost rows
        self.system.forward_comm()
        self._packed = True
        if self._speculative():
            # speculative force launch, gated on the device by the same skin test:
            # the GPU runs it while the host reads the decision (no idle gap), and
            # it is a no-op on a rebuilding step (relaunched after the rebuild)
            self._gate = worst
            self._spec_e = self._forces_device(gate=worst, gate_limit=0.5 * self.config.skin)
        self._d2_ready.synchronize()
        d2 = float(self._d2_host[0])
        if not math.isfinite(d2):
            self._nonfinite_abort(self._run_step - 1)
        return math.sqrt(d2) > 0.5 * self.config.skin

    def _half_kick(self):
        lib, st = _lib.lib(), _lib.stream(self.device)
        h = 0.5 * self.dt / self.mass
        for s in self.system.stores:
            _lib.check(lib.mdkk_verlet_second(_lib.ctx(self.device), s.v.data_ptr(), s.f.data_ptr(), s.n_local,
                                              h, self.mass, None, st), "mdkk_verlet_second")
            s.device_wrote(vel=True)

    def step_device(self, defer_kick: bool = False) -> torch.Tensor:
        """One velocity-Verlet step (mdkk/driver/simulation.py:431-450); energy stays on device.

        `defer_kick` leaves the closing half-kick pending: the next step's
        opening pass applies it (one fewer pass over v and f per step inside
        `advance`); `flush_kick()` completes it before velocities are read.
        """
        self._packed = False
        self._spec_e = None
        self._run_step += 1
        if self._half_kick_drift():
            # with a gated style the build's capacity check is deferred: the force launch
            # (gated on the device-side count) queues behind the build without a host
            # round trip, and only an overflow (rare: cap grows x1.5) repeats it
            # (distributed half lists excepted: a regrow on one rank would re-run the
            # reverse-comm collective on that rank alone)
            defer = (self._speculative() and self._cap_hint is not None
                     and not (self.config.distributed and self._list_style == "half"))
            self._rebuild_lists(defer=defer)
            e = self._forces_device()
            if defer and not self._settle_lists():
                e = self._forces_device()
        else:
            if not self._packed:
                self.system.forward_comm()
            e = self._spec_e if self._spec_e is not None else self._forces_device()
        self._spec_e = None
        self._e_prev = e
        if defer_kick:
            self._kick_pending = True
        else:
            self._half_kick()
        return e

    def flush_kick(self) -> None:
        """Apply a deferred closing half-kick (velocities complete afterwards)."""
        if self._kick_pending:
            self._half_kick()
            self._kick_pending = False

    def step_once(self) -> float:
        return float(self.step_device().item())

    def advance(self, n_steps: int) -> torch.Tensor | None:
        """n velocity-Verlet steps without thermo; returns the last step's device energy.

        The cyclic garbage collector is paused for the loop: the per-step host
        objects are acyclic (freed by reference counting), and a full
        collection over the interpreter's heap would stall the launch queue
        for milliseconds.
        """
        was = gc.isenabled()
        gc.disable()
        try:
            if n_steps >= 2 and self._fusable():
                return self._advance_fused(n_steps)
            e = None
            for _ in range(n_steps):
                e = self.step_device(defer_kick=True)
            self.flush_kick()
            return e
        finally:
            if was:
                gc.enable()

    def _speculative(self) -> bool:
        """Gated (speculative) force launches: LJ with the default or Atomic half-list
        writes; an explicit Serial / Duplicate strategy runs the staged kernels unguarded."""
        return (getattr(self.style, "supports_gate", False)
                and not (self._list_style == "half" and self.config.strategy in ("serial", "duplicate")))

    def _fusable(self) -> bool:
        """The integration fuses into the force kernel for full-list LJ (atom mode) with one
        store per process (one in-process rank, or one rank per GPU): the epilogue needs
        each owned atom's complete force."""
        return (isinstance(self.style, LJStyle) and self._speculative()
                and self._list_style == "full" and (self.config.mode or self.style.default_mode) == "atom"
                and len(self.system.stores) == 1)

    def _advance_fused(self, n_steps: int) -> torch.Tensor:
        """`advance` with velocity-Verlet fused into the force epilogue.

        Step s's force kernel also closes step s and opens + drifts step s+1 into a
        second position buffer, taking the next skin-test maximum; the last step
        only closes.  The pipeline keeps the speculative shape of `step_device`:
        the pack and the force launch for step s are queued, gated on step s's
        device-side maximum, before the host has read it; a rebuilding step
        relaunches after the rebuild.  Positions swap buffers after every drift.
        Bit-identical to the unfused loop (tests/test_pipeline_gpu.py).
        """
        lib, stream = _lib.lib(), _lib.stream(self.device)
        ctx = _lib.ctx(self.device)
        s = self.system.stores[0]
        h = 0.5 * self.dt / self.mass
        half = 0.5 * self.config.skin
        main = torch.cuda.current_stream(self.device)
        if getattr(self, "_fz", None) is None:
            # drift maxima in a three-slot ring: step s writes slot s+1 and its (pack-fused)
            # reduction clears slot s+2, whose previous read-back the host has already waited on
            self._fz = dict(d2=torch.zeros(3, dtype=torch.float64, device=self.device),
                            pin=torch.zeros(3, dtype=torch.float64, pin_memory=True),
                            ready=[torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()],
                            kicked=torch.cuda.Event(), side=torch.cuda.Stream(self.device), x_alt=None)
        fz = self._fz
        d2 = fz["d2"]

        def read_back(k):   # d2[k] -> pin[k] on the side stream, behind the work queued so far
            fz["kicked"].record(main)
            fz["side"].wait_event(fz["kicked"])
            with torch.cuda.stream(fz["side"]):
                fz["pin"][k:k + 1].copy_(d2[k:k + 1], non_blocking=True)
            fz["ready"][k].record(fz["side"])

        def x_alt():        # the drift target: same capacity, never aliasing a live buffer
            a = fz["x_alt"]
            live = {s.x.data_ptr()} | ({s._alt[0].data_ptr()} if s._alt is not None else set())
            if a is None or a.shape[0] != s.x.shape[0] or a.data_ptr() in live:
                a = fz["x_alt"] = torch.zeros_like(s.x)   # once per buffer; pads defined
            return a

        dist_ = self.config.distributed
        # one rank per GPU with other ranks across some faces: overlap the halo exchange
        overlap = bool(dist_ and getattr(self.system, "world", 1) > 1 and self.system.remote_dims())
        overlap_halo = self.style.r_c + self.config.skin + 0.5 * self.config.skin * (1.0 + 1e-9) + 1e-12

        def global_max(k):   # one rank per GPU: every rank gates and decides on the same maximum
            if dist_:
                self.system.allreduce_max(d2[k:k + 1])

        fuse_pack = (not dist_) and isinstance(self.system, RankedSystem) and self.system.n_ranks == 1
        packed = False   # the ghost rows of the current x were written by the previous launch
        cleared = None   # the d2 slot the previous launch's reduction cleared
        # opening of step 1: the classic pass (with any deferred closing kick)
        s.to_device()
        _lib.check(lib.mdkk_verlet_first(ctx, s.x.data_ptr(), s.v.data_ptr(), s.f.data_ptr(),
                                         self.lists[0].ref_dev.data_ptr(), s.n_local, self.dt, h, d2.data_ptr(),
                                         int(self._kick_pending), stream), "mdkk_verlet_first")
        global_max(0)
        self._kick_pending = False
        s.device_wrote(pos=True, vel=True)
        cur = 0
        read_back(cur)
        e = None
        d2[1:].zero_()
        for step in range(1, n_steps + 1):
            self._run_step += 1
            mode = 2 if step < n_steps else 1
            nxt, aft = (cur + 1) % 3, (cur + 2) % 3
            xa = x_alt() if mode == 2 else None

            def launch(gated, part=0):
                nonlocal packed, cleared
                integ = dict(mode=mode, x_next=xa, d2_next=d2[nxt:nxt + 1], dt=self.dt, h=h, part=part)
                if part:
                    integ["flags"] = self.system.cluster_flags(self.lists[0], overlap_halo)
                packed = False
                if mode == 2 and fuse_pack:
                    # one rank: step s+1's periodic ghost rows are written from x(s+1) in the
                    # force launch's reduction blocks (the separate pack of the next step is skipped)
                    lanes = self.system.lanes
                    if not lanes:
                        packed = True
                    elif len(lanes) == 1 and lanes[0].start == s.n_local:
                        integ["pack"] = (lanes[0], self.system._shift_dev)
                        integ["d2_zero"] = d2[aft:aft + 1]   # the slot step s+2 writes
                        packed = True
                if mode == 2 and part != 2 and cleared != nxt:
                    d2[nxt:nxt + 1].zero_()
                e_ = self._forces_device(gate=d2[cur:cur + 1] if gated else None, gate_limit=half, integ=integ)
                # the slot this launch's reduction cleared (a relaunch of this step refills d2[nxt])
                cleared = aft if "d2_zero" in integ else None
                return e_

            if overlap:
                # halo overlap: the clusters that list no exchanged ghost run while the
                # exchange is in flight, the boundary clusters once it has landed
                pending = self.system.forward_comm_begin()
                launch(True, part=1)
                self.system.forward_comm_end(pending)
                e = launch(True, part=2)
            else:
                if not packed:
                    self.system.forward_comm()         # speculative halo refresh
                e = launch(True)                       # speculative force + integration
            if mode == 2:
                global_max(nxt)
                read_back(nxt)
            fz["ready"][cur].synchronize()
            d2h = float(fz["pin"][cur])
            if not math.isfinite(d2h):   # the drift of this step saw a non-finite x / v / f
                self._nonfinite_abort(self._run_step - 1)
            if math.sqrt(d2h) > half:
                defer = self._cap_hint is not None
                self._rebuild_lists(defer=defer)
                s = self.system.stores[0]               # a distributed migrate makes a new store
                xa = x_alt() if mode == 2 else None     # the rebuild may have rotated buffers
                e = launch(False)
                if defer and not self._settle_lists():
                    e = launch(False)
                if mode == 2:
                    global_max(nxt)
                    read_back(nxt)                     # the relaunch rewrote the maximum
            if mode == 2:
                fz["x_alt"] = s.x                      # swap: x(s+1) becomes current
                s.x = xa
                s._views()
                s.device_wrote(pos=True, vel=True, force=True)
                cur = nxt
            else:
                s.device_wrote(vel=True, force=True)
            self._e_prev = e
        return e

    def _nonfinite_abort(self, step: int):
        """The per-step drift maximum came back non-finite: the forces (or energy) of
        `step` were not finite (mdkk/driver/simulation.py:459-464, checked every step
        there).  Raise the reference's RunError naming that step."""
        torch.cuda.synchronize(self.device)
        if self._flags is not None and int(self._flags.item()) & _lib.FLAG_COINCIDENT:
            from ..pair_lj import PairError
            raise PairError("coincident atoms (r = 0)")   # what the reference's kernel raises (pair_lj.py:83-84)
        e = getattr(self, "_e_prev", None)
        if e is not None and not math.isfinite(float(self._global_sum(e.reshape(1)).item())):
            raise RunError(f"non-finite potential energy at step {step}")
        raise RunError(f"non-finite force at step {step}")

    def _check_finite(self, step, e_pot):
        if not np.isfinite(e_pot):
            raise RunError(f"non-finite potential energy at step {step}")
        for s in self.system.stores:
            if s.n_local and not bool(torch.isfinite(s.f[: s.n_local, :3]).all().item()):
                raise RunError(f"non-finite force at step {step}")
        if self._flags is not None and int(self._flags.item()) & _lib.FLAG_COINCIDENT:
            from ..pair_lj import PairError
            raise PairError("coincident atoms (r = 0)")   # the reference kernel's error (pair_lj.py:83-84)

    def run_nve(self, n_steps: int) -> RunResult:
        """NVE with thermo at 0, every `thermo`, and the last step (mdkk/driver/simulation.py:452-481).

        Non-finite values abort at the first bad step, as in the reference: the
        per-step skin-test read-back the loop already waits on carries it (the
        kernels turn a non-finite drift into +inf), so step t's check sees step
        t-1's forces; logged steps also scan energy, forces and the error word.
        """
        if n_steps < 0:
            raise RunError("run expects a non-negative step count")
        with torch.cuda.device(self.device):
            self._ensure_system()
            result = RunResult()
            self.results.append(result)
            rebuilds0 = self.n_rebuilds

            pending = []     # (step, finish): snapshots whose read-back overlaps the next stretch

            def settle_snapshots(keep: int = 0):
                while len(pending) > keep:
                    at, finish = pending.pop(0)
                    result.snapshots[at] = finish()

            def log(step, e_dev, last):
                e_pot = float(self._global_sum(e_dev.reshape(1)).item())
                self._check_finite(step, e_pot)
                ke, t = self._kinetic()
                result.log(step, e_pot, ke, t)
                if self.snapshots:
                    # queued on the copy stream; the host copy of an earlier snapshot overlaps it
                    pending.append((step, self.system.gather_positions_async()))
                self._qeq_diagnostic(step, result)
                self.log(result.lines[-1])

            self._run_step = 0
            self._e_prev = None
            log(0, self._forces_device(), n_steps == 0)
            step = 0
            while step < n_steps:   # device-resident stretches between thermo steps
                k = min(self.thermo_every - step % self.thermo_every, n_steps - step)
                e = self.advance(k)
                step += k
                log(step, e, step == n_steps)
                settle_snapshots(keep=1)   # earlier snapshots finish while this one is in flight
            settle_snapshots()
            result.n_rebuilds = self.n_rebuilds - rebuilds0
        return result


def run_script(text: str, config: RunConfig | None = None, log=print) -> Simulation:
    """Parse and execute a script (mdkk/driver/simulation.py:484-488)."""
    sim = Simulation(config, log=log)
    sim.execute(parse_script(text))
    return sim
