#!/usr/bin/env python
"""Benchmark: LJ melt (and SNAP) atom-steps/s on B200, one JSON line on rank 0.

Workload at N=1 (BASELINE.json configs[1]): LJ 12-6 melt, 2,048,000 atoms fcc
rho*=0.8442 (80^3 cells), rc=2.5, skin=0.3, T=1.44 (seed 87287), dt=0.005,
velocity-Verlet NVE with skin rebuilds — both the full/newton-off list (no
atomics, headline `value`) and the half/newton-on list (FP64 atomics).  A
"step" is one full velocity-Verlet step (kick+drift+skin test, halo refresh
or rebuild, force, kick).  Inputs (x, v, f, table: ~1 GB) exceed the 126 MB L2.
At N = 1 the configs[2] melt (16,384,000 atoms) is timed too, as a variant:
the baseline of the strong-scaling curve.  Under torchrun (N > 1) the headline
is configs[2] split over the N GPUs (strong scaling; `--weak` = an 80^3 brick
per GPU) and the SNAP line is configs[4] (1,024,000 atoms) over the N GPUs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Matom-steps/s for LJ & SNAP at 1/2/4/8 B200; % of HBM / FP64 roofline"
UNIT = "Matom-steps/s"
LJ = dict(rho=0.8442, cells=80, rc=2.5, skin=0.3, T=1.44, seed=87287, dt=0.005)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def lj_script(cells, style_newton_thermo=10 ** 9, steps=0):
    cx, cy, cz = cells if isinstance(cells, tuple) else (cells, cells, cells)
    return (f"units lj\nboundary p p p\nlattice fcc {LJ['rho']}\ncreate_box {cx} {cy} {cz}\n"
            f"create_atoms\nmass 1.0\nvelocity {LJ['T']} {LJ['seed']}\npair_style lj/cut {LJ['rc']}\n"
            f"pair_coeff 1.0 1.0\ntimestep {LJ['dt']}\nthermo {style_newton_thermo}\n")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi -lms 100 in a child process while running (the recipe's clocks line).

    A separate process, not a Python thread: a sampler thread would contend
    for the GIL with the launch loop and perturb the timed region.
    """

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._p = None

    def __enter__(self):
        import subprocess
        import tempfile
        self._out = tempfile.TemporaryFile(mode="w+")
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                        "--format=csv,noheader,nounits", "-lms", "100"],
                                       stdout=self._out, stderr=subprocess.DEVNULL)
        except OSError:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        import time as _t
        _t.sleep(0.15)   # at least one sample after the timed region's tail
        self._p.terminate()
        self._p.wait()
        self._out.seek(0)
        for line in self._out.read().splitlines():
            parts = [v.strip() for v in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                self.samples.append(float(parts[0]))
                self.max_mhz = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:]):
                if v.lower() == "active":
                    self.reasons.add(name)

    def summary(self):
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------- CPU oracle
def cpu_lj_sample(steps=3, cells=40, style="full"):
    """Oracle (numpy port of mdkk) on a bounded sample of configs[1]: the same melt at 40^3 cells
    (256,000 atoms, 1/8 of configs[1]), initial build untimed, `steps` timed NVE steps.  The
    per-atom CPU rate grows with N up to ~256k (numpy overheads amortise: 32k runs 1.33x slower
    per atom here), so this sample is the closest bounded stand-in for the 2M configuration."""
    from oracle import md
    pos, L = md.lattice("fcc", LJ["rho"], (cells, cells, cells))
    vel = md.seeded_velocities(len(pos), LJ["T"], 1.0, LJ["seed"])
    run = md.LJRun(pos, vel, L, rc=LJ["rc"], skin=LJ["skin"], style=style, newton=(style == "half"), dt=LJ["dt"])
    run.forces()
    t0 = time.perf_counter()
    for _ in range(steps):
        run.step()
    dt = time.perf_counter() - t0
    return len(pos) * steps / dt / 1e6, dt, len(pos)


def _reference_replica(cells, steps, warmup, out):
    """One single-threaded replica of the reference arm's bounded sample (child process)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:
        pass
    from oracle import md
    pos, L = md.lattice("fcc", LJ["rho"], (cells, cells, cells))
    vel = md.seeded_velocities(len(pos), LJ["T"], 1.0, LJ["seed"])
    run = md.LJRun(pos, vel, L, rc=LJ["rc"], skin=LJ["skin"], style="full", newton=False, dt=LJ["dt"])
    run.forces()
    for _ in range(warmup):
        run.step()
    t = []
    for _ in range(steps):
        t0 = time.perf_counter()
        run.step()
        t.append(time.perf_counter() - t0)
    out.put((len(pos), t))


def run_reference(args):
    """The reference arm: mdkk's algorithm (the numpy port in oracle/, mdkk being pure Python and
    single-threaded by construction) on every host core -- one replica per core of the bounded
    sample, aggregate throughput (the SURVEY's "nproc concurrent replica processes")."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    # bounded sample: 20^3 cells (32,000 atoms, ~0.3 s per step on one core) for up to
    # 200 timed steps, smaller cubes beyond so the whole run stays within a few minutes
    # bounded sample of configs[1]: 40^3 cells (256,000 atoms, ~4 s per step on one core) for runs
    # of up to 60 steps, 20^3 (32,000 atoms, ~0.6 s per step) up to 400, smaller cubes beyond,
    # so the whole run stays within a few minutes
    total = max(1, args.steps + args.warmup)
    cells = 40 if total <= 60 else 20 if total <= 400 else max(6, int(20 * (400.0 / total) ** (1.0 / 3.0)))
    n_rep = max(1, min(os.cpu_count() or 1, 32))
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    procs = [ctx.Process(target=_reference_replica, args=(cells, args.steps, args.warmup, q)) for _ in range(n_rep)]
    for p_ in procs:
        p_.start()
    res = [q.get() for _ in procs]
    for p_ in procs:
        p_.join()
    n_atoms = res[0][0]
    rates = [n_atoms * args.steps / sum(t) / 1e6 for _, t in res]
    value = float(sum(rates))
    ms = 1e3 * float(np.mean([sum(t) for _, t in res])) / args.steps
    sample = (f"numpy oracle port of mdkk (oracle/md.py), LJ melt {n_atoms:,} atoms fcc rho 0.8442 rc 2.5 "
              f"skin 0.3 T 1.44 dt 0.005 full list, {args.steps} steps after {args.warmup} warm-up, "
              f"{n_rep} concurrent single-threaded replicas (one per host core), aggregate rate "
              f"(one replica alone: {max(rates):.4f})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"LJ melt, bounded CPU sample of configs[1] ({n_atoms:,} atoms per replica)",
                   "n_atoms": n_atoms, "replicas": n_rep},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": n_rep, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


# -------------------------------------------------------------------- GPU
def lj_run(style, cells, steps, warmup, device, profile=True, distributed=False):
    import torch
    from paper_2508_13523_b200 import _lib
    from paper_2508_13523_b200.driver import RunConfig, Simulation
    sim = Simulation(RunConfig(list_style=style, newton=(style == "half"), skin=LJ["skin"], device=device,
                               distributed=distributed), log=None)
    sim.execute(lj_script(cells))
    sim._ensure_system()
    sim._forces_device()
    # warm-up through the same loop as the timed region (its buffers, pinned read-back
    # slots and side stream are created here, not inside the timing)
    sim.advance(max(warmup, 2))
    torch.cuda.synchronize()
    rebuild0, l0 = sim.n_rebuilds, _lib.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if distributed:
        import torch.distributed as dist
        dist.barrier()
    start.record()
    sim.advance(steps)
    end.record()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    ms = start.elapsed_time(end) / steps
    launches = _lib.launch_count() - l0
    rebuilds = sim.n_rebuilds - rebuild0
    fms = None
    if profile:
        # force-kernel time, measured after (not inside) the timed region: CUDA events
        # around every force launch of a further stretch, the gated no-op launches of
        # rebuilding steps (a few us) dropped
        fev = []
        orig = sim._forces_device

        def timed_forces(**kw):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            e = orig(**kw)
            b.record()
            fev.append((a, b))
            return e
        sim._forces_device = timed_forces
        sim.advance(min(steps, 30))
        sim._forces_device = orig
        torch.cuda.synchronize()
        t = np.array([a.elapsed_time(b) for a, b in fev])
        fms = float(t[t > 0.5 * np.median(t)].mean()) if len(t) else None
    st = sim.system.stores[0]
    nn = float(sim.lists[0].counts_dev[: st.n_local].double().mean().item())
    e = float(sim._e_dev.item())
    return dict(ms=ms, force_ms=fms, n_atoms=sim.system.n_atoms, rebuilds=rebuilds,
                launches=launches, nn=nn, e_pot=e, n_ghost=st.n_ghost, fused=sim._fusable())


SNAP = dict(a=3.1803, cells=80, rc=4.73, skin=0.3, T=0.01, seed=4928459, dt=0.001, twojmax=8)
SNAP_TERMS = 32578   # coupling terms at 2J = 8


def snap_flops_per_atom_step(nn):
    """Canonical mdkk-formulation FLOPs: nn*(9260 + 60518) + 36*T."""
    return nn * (9260.0 + 60518.0) + 36.0 * SNAP_TERMS


def fp64_peak(device):
    """Live FP64 FMA peak (TFLOP/s) from the library's DFMA probe, timed with CUDA events."""
    import torch
    from paper_2508_13523_b200 import _lib
    out = torch.zeros(1, dtype=torch.float64, device=device)
    blocks, iters = 148 * 8, 20000
    _lib.call("mdkk_fp64_probe", blocks, 100, out.data_ptr(), _lib.stream(device))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.call("mdkk_fp64_probe", blocks, iters, out.data_ptr(), _lib.stream(device))
    b.record()
    torch.cuda.synchronize()
    return blocks * 256 * iters * 8 * 2 / (a.elapsed_time(b) * 1e-3) / 1e12


def snap_run(cells, steps, warmup, device, distributed=False):
    import tempfile
    import torch
    from paper_2508_13523_b200 import _lib
    from paper_2508_13523_b200.driver import RunConfig, Simulation
    coeff = os.path.join(tempfile.mkdtemp(), "w_2j8.coeff")
    with open(coeff, "w") as fh:
        fh.write("4\n" + "\n".join(repr(float(b)) for b in np.linspace(0.05, 0.1, 55)) + "\n")
    # batch_y=2: compute_yi serves two atoms per lane (the fastest schedule on B200; batch_u keeps
    # the reference default 4 = 16-lane teams, also the fastest)
    sim = Simulation(RunConfig(skin=SNAP["skin"], device=device, distributed=distributed, batch_y=2), log=None)
    sim.execute(f"units lj\nboundary p p p\nlattice bcc {SNAP['a']}\ncreate_box {cells} {cells} {cells}\n"
                f"create_atoms\nmass 1.0\nvelocity {SNAP['T']} {SNAP['seed']}\nsuffix kk\n"
                f"pair_style snap {SNAP['rc']} {coeff}\ntimestep {SNAP['dt']}\nthermo 1000000000\n")
    sim._ensure_system()
    sim._forces_device()
    for _ in range(warmup):
        sim.step_device()
    torch.cuda.synchronize()
    fev = []
    orig = sim._forces_device

    def timed_forces(**kw):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        e = orig(**kw)
        b.record()
        if not kw and fev and fev[-1][2]:
            fev.pop()    # a rebuilding step: its speculative (gated, no-op) launch is replaced
        fev.append((a, b, bool(kw)))
        return e
    sim._forces_device = timed_forces
    l0 = _lib.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if distributed:
        import torch.distributed as dist
        dist.barrier()
    start.record()
    sim.advance(steps)
    end.record()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    ms = start.elapsed_time(end) / steps
    st, nl = sim.system.stores[0], sim.lists[0]
    # pairs within rc per atom (the descriptor neighbours), counted on device from the list
    ncl = nl.table_dev.shape[0]
    tab = nl.table_dev.permute(1, 0, 2).reshape(nl.alloc_cap, ncl * 32)[:, : st.n_local].long()
    cnt = nl.counts_dev[: st.n_local].long()
    valid = torch.arange(nl.alloc_cap, device=device)[:, None] < cnt[None, :]
    xj = st.x[torch.where(valid, tab, 0), :3]
    d = xj - st.x[: st.n_local, :3][None]
    nn = float((((d * d).sum(-1) < SNAP["rc"] ** 2) & valid).sum().item()) / st.n_local
    return dict(ms=ms, force_ms=float(np.mean([a.elapsed_time(b) for a, b, _ in fev])), n_atoms=sim.system.n_atoms,
                nn=nn, launches=_lib.launch_count() - l0, e_pot=float(sim._e_dev.item()))


def lj_e2e(style, cells, steps, device, distributed=False):
    """Public API end to end: host arrays -> distribute/build -> run_nve(steps) -> thermo + gid-ordered D2H."""
    import torch
    from paper_2508_13523_b200.driver import RunConfig, Simulation
    sim = Simulation(RunConfig(list_style=style, newton=(style == "half"), skin=LJ["skin"], device=device,
                               distributed=distributed), log=None)
    sim.execute(lj_script(cells, style_newton_thermo=steps))
    import gc
    gc.collect()               # earlier runs' buffers back to the caching allocator
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.run_nve(steps)          # upload, build, steps, thermo at 0 and `steps` (+ gid-ordered snapshots)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    n = sim.system.n_atoms
    h2d = n * 2 * 3 * 8                         # positions + velocities uploaded once
    d2h = 2 * (n * 3 * 8 + 2 * 8)               # two thermo snapshots (positions) + E, KE
    return dict(value=n * steps / dt / 1e6, h2d=h2d / steps, d2h=d2h / steps)


def ncu_metrics():
    """Per-kernel ncu figures committed under profiles/ (tools/ncu_metrics.py): DRAM bytes,
    L1TEX wavefront %, executed FP64 instructions, per launch, with the launch's atom count."""
    p = os.path.join(ROOT, "profiles", "ncu_metrics.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def build_block(prof, peak):
    """The neighbour build's HBM / L2 figures from its committed ncu capture (one melt-state
    rebuild of the 2M-atom system, tools/ncu_metrics.py): the north star asks for both."""
    b = prof.get("k_nbr_build_full")
    if not b:
        return None
    sec = b["duration_us"] * 1e-6
    return {"kernel": "k_nbr_build_full (streaming cluster build, full list)", "ms_ncu": b["duration_us"] * 1e-3,
            "dram_gbs": b["dram_bytes"] / sec / 1e9, "dram_frac": b["dram_bytes"] / sec / 1e9 / peak,
            "l2_gbs": b.get("l2_bytes", 0.0) / sec / 1e9 or None, "l1_wavefront_pct": b.get("l1tex_wavefront_pct"),
            "warps_active_pct": b.get("warps_active_pct"),
            "note": "issue bound (one rebuild per ~6 steps): ~530 union candidates tested per listed atom; "
                    "the DRAM bytes are the table write (0.73 GB) + position reads; L2 bytes include the "
                    "table's sector-granular 4-byte stores",
            "source": b.get("source")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cells", type=int, default=LJ["cells"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-snap", action="store_true")
    ap.add_argument("--no-16m", action="store_true", help="skip the configs[2] point at N=1")
    ap.add_argument("--snap-cells", type=int, default=SNAP["cells"])
    ap.add_argument("--snap-steps", type=int, default=5)
    ap.add_argument("--strong", action="store_true",
                    help="configs[2] headline: the fixed 160^3-cell (16,384,000-atom) melt over the N GPUs "
                         "(the default when WORLD_SIZE > 1)")
    ap.add_argument("--weak", action="store_true", help="N > 1: an 80^3-cell brick per GPU instead")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)

    from paper_2508_13523_b200.domain import Box as _Box, decompose as _decompose
    grid = _decompose(_Box((1.0, 1.0, 1.0)), world).grid
    # N = 1: configs[1] (2,048,000 atoms) headline + the configs[2] point (16,384,000 atoms) as a
    # variant; N > 1: configs[2] strong scaling (the north star's 80 % target), or --weak bricks
    strong = args.strong or (world > 1 and not args.weak)
    cells = (160, 160, 160) if strong else tuple(args.cells * g for g in grid)
    scaling = "strong" if strong else "weak"
    workload = ("LJ 12-6 melt fcc rho*=0.8442, rc=2.5, skin=0.3, T=1.44, dt=0.005, full list newton-off "
                + ("(configs[2]: 16,384,000 atoms, strong scaling over the GPUs)" if strong else
                   "(configs[1]: 2,048,000 atoms per GPU)"))
    distributed = world > 1

    def max_over_ranks(v):
        if not distributed or v is None:
            return v
        import torch.distributed as dist
        t = torch.tensor([v], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with ClockSampler(local) as clk:   # sampled in a child process across the timed LJ runs
        full = lj_run("full", cells, args.steps, args.warmup, device, distributed=distributed)
        half = lj_run("half", cells, args.steps, args.warmup, device, distributed=distributed)
        big = None
        if world == 1 and not strong and not args.no_16m:
            big = lj_run("full", (160, 160, 160), min(args.steps, 20), max(args.warmup, 3), device, profile=False)
    ms = max_over_ranks(full["ms"])
    half_ms = max_over_ranks(half["ms"])
    force_ms = max_over_ranks(full["force_ms"])
    n_atoms = full["n_atoms"]           # global atom count (all bricks)
    value = n_atoms / (ms * 1e-3) / 1e6
    peak, peak_kind = _peaks()
    nn = full["nn"]
    prof = ncu_metrics()
    # pair-stream model per launch: 28 B per listed partner + 52 B per atom;
    # the fused integration epilogue adds v read+write, x_ref read, x_next write (128 B)
    fused = bool(full.get("fused"))
    per_atom = 28.0 * nn + 52.0 + (128.0 if fused else 0.0)
    n_rank = full["n_atoms"] / world
    bytes_per_launch = n_rank * per_atom
    achieved = bytes_per_launch / (force_ms * 1e-3) / 1e9
    kname = "k_lj_fused" if fused else "k_lj"
    kp = prof.get(kname, {})
    traffic = kp.get("dram_bytes") * n_rank / kp["n_atoms"] if kp.get("dram_bytes") else None
    # e2e: the user's call `run 100` (the configs' run length) from host arrays, thermo + snapshots back
    e2e_steps = 100
    if not args.no_e2e:
        lj_e2e("full", cells, 5, device, distributed)   # untimed: first-call allocations
    e2e = lj_e2e("full", cells, e2e_steps, device, distributed) if not args.no_e2e else None
    if e2e is not None and distributed:
        e2e["value"] = n_atoms * e2e_steps / max_over_ranks(n_atoms * e2e_steps / e2e["value"])
    snapr, fp64 = None, None
    if not args.no_snap:
        fp64 = fp64_peak(device)
        snapr = snap_run(args.snap_cells, args.snap_steps, 2, device, distributed)
        snapr["ms"] = max_over_ranks(snapr["ms"])
        snapr["force_ms"] = max_over_ranks(snapr["force_ms"])
    cpu = None
    if rank == 0 and not args.no_cpu:
        v, secs, n = cpu_lj_sample()
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"numpy oracle port of mdkk (oracle/md.py), the configs[1] melt at 40^3 cells ({n:,} "
                         f"atoms; same rho/rc/skin/T/dt, full list), 3 NVE steps after the initial build, "
                         f"{secs:.1f} s, 1 thread of {os.cpu_count()}"}
    if rank == 0:
        snap_block = None
        if snapr is not None:
            flop_model = snap_flops_per_atom_step(snapr["nn"]) * snapr["n_atoms"] / (snapr["force_ms"] * 1e-3) / 1e12
            ex = prof.get("snap_pipeline", {})
            executed = (ex["dflop_per_atom"] * snapr["n_atoms"] / (snapr["force_ms"] * 1e-3) / 1e12
                        if ex.get("dflop_per_atom") else None)
            snap_block = {
                "workload": f"SNAP W bcc a=3.1803, 2J=8, rc=4.73, skin 0.3, T=0.01, dt=0.001, "
                            f"{snapr['n_atoms']:,} atoms (configs[4]"
                            + (f", strong scaling over {world} GPUs)" if distributed else " at N=1)"),
                "value": snapr["n_atoms"] / (snapr["ms"] * 1e-3) / 1e6, "unit": UNIT,
                "scaling": "strong" if distributed else None,
                "ms_per_step": snapr["ms"], "force_ms": snapr["force_ms"], "steps": args.snap_steps,
                "pairs_within_rc_per_atom": snapr["nn"],
                "roofline": {"bound": "fp64", "kernel": "ui + yi + fused deidrj (+ reverse comm)",
                             "achieved": flop_model, "peak": fp64 * world,
                             "peak_kind": "measured live (DFMA probe) x GPUs", "unit": "TFLOP/s",
                             "frac": flop_model / (fp64 * world),
                             "flops_model": "canonical mdkk formulation nn*(9260+60518)+36*32578 per atom",
                             "executed_tflops": executed,
                             "executed_frac": executed / (fp64 * world) if executed else None,
                             "executed_source": ex.get("source")}}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload,
                       "n_atoms": full["n_atoms"], "n_ghost_rank0": full["n_ghost"], "list": "full",
                       "grid": list(grid),
                       "rebuilds_in_timed_steps": full["rebuilds"], "mean_neighbors": nn,
                       "l2": "inputs (x,v,f,table ~%.0f MB per GPU) larger than L2"
                             % (n_rank * (nn * 4 + 96) / 1e6),
                       "parallelism": (f"spatial DD {grid[0]}x{grid[1]}x{grid[2]}, NCCL halo exchange"
                                       if world > 1 else "1 GPU")},
            "variants": {
                "lj_full_newton_off": {"value": value, "ms_per_step": ms, "force_ms": force_ms,
                                       "rebuilds": full["rebuilds"]},
                "lj_half_newton_on_atomics": {"value": half["n_atoms"] / (half_ms * 1e-3) / 1e6,
                                              "ms_per_step": half_ms, "force_ms": half["force_ms"],
                                              "rebuilds": half["rebuilds"], "mean_neighbors": half["nn"]},
            },
            "roofline": {"bound": "hbm",
                         "kernel": ("k_lj<full> + fused velocity-Verlet epilogue (+ partial reduce)" if fused
                                    else "k_lj<full> (+ partial reduce)"),
                         "achieved": achieved,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic,
                         "bytes_model": (f"n_local*(28*nn+52+128), nn={nn:.2f} measured" if fused
                                         else f"n_local*(28*nn+52), nn={nn:.2f} measured"),
                         "dram_frac": traffic / (force_ms * 1e-3) / 1e9 / peak if traffic else None,
                         "l1_wavefront_pct": kp.get("l1tex_wavefront_pct"),
                         "l2_gbs": (kp["l2_bytes"] / (force_ms * 1e-3) / 1e9) if kp.get("l2_bytes") else None,
                         "fp64_pipe_pct": kp.get("fp64_pipe_pct"),
                         "profile_source": kp.get("source"),
                         "note": ("frac = SURVEY 8(d) pair-stream model (x_j reuse in L1/L2 lets it exceed 1); "
                                  "dram_frac = the kernel's ncu DRAM bytes per launch over the live launch time; "
                                  "the binding limiter is the L1TEX data pipe (l1_wavefront_pct)")},
            "neighbor_build": build_block(prof, peak),
            "snap": snap_block,
            "cpu_baseline": cpu,
            "e2e": ({"value": e2e["value"], "unit": UNIT, "h2d_bytes_per_step": e2e["h2d"],
                     "d2h_bytes_per_step": e2e["d2h"],
                     "what": f"Simulation.run_nve({e2e_steps}) from host positions/velocities: upload, distribute, "
                             "first build, steps, thermo at 0 and end with gid-ordered position snapshots"}
                    if e2e else None),
            "gpu_launches": full["launches"],
            "clocks": clk.summary(),
        }
        if big is not None:
            out["variants"]["lj_16m_full_configs2_n1"] = {
                "value": big["n_atoms"] / (big["ms"] * 1e-3) / 1e6, "ms_per_step": big["ms"],
                "n_atoms": big["n_atoms"], "rebuilds": big["rebuilds"],
                "what": "configs[2] on one GPU: the strong-scaling baseline for bench.py --gpus N"}
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
