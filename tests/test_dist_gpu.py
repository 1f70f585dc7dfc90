"""World-size-2 run of the one-brick-per-process engine (dist.DistSystem) on one GPU.

Two processes share cuda:0 and talk over gloo (the collectives and P2P are
staged through the host; on a multi-GPU box the same code uses NCCL on device
buffers).  Every device kernel of the distributed path runs: owner partition,
halo select / pack / fold, migration, lists, LJ (full and half) and SNAP.
The thermo log must match the in-process two-rank run (mdkk's rank
invariance, tests/test_driver.py:252-260).
"""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

LJ = ("units lj\nboundary p p p\nlattice fcc 0.8442\ncreate_box 16 16 16\ncreate_atoms\nmass 1.0\n"
      "velocity 1.44 87287\npair_style lj/cut 2.5\npair_coeff 1.0 1.0\ntimestep 0.005\nthermo 10\nrun 40\n")


def _snap_script(coeff):
    return ("units lj\nboundary p p p\nlattice bcc 3.1803\ncreate_box 6 6 6\ncreate_atoms\nmass 1.0\n"
            f"velocity 0.01 4928459\nsuffix kk\npair_style snap 4.73 {coeff}\ntimestep 0.001\nthermo 5\nrun 10\n")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, coeff, out):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_13523_b200.driver import RunConfig, run_script
        res = {}
        for style in ("full", "half"):
            sim = run_script(LJ, RunConfig(list_style=style, newton=(style == "half"),
                                                                   distributed=True, device="cuda:0"), log=None)
            res[f"lj_{style}"] = np.array(sim.results[-1].rows)
            if style == "full":   # the halo-overlap path ran: interior clusters, then boundary ones
                fl = getattr(sim.lists[0], "_part_flags", None)
                res["overlap"] = np.array([-1.0 if fl is None else float(fl.float().mean().item())])
        sim = run_script(_snap_script(coeff), RunConfig(distributed=True, device="cuda:0"), log=None)
        res["snap"] = np.array(sim.results[-1].rows)
        if rank == 0:
            np.savez(out, **res)
    finally:
        dist.destroy_process_group()


def test_distributed_two_ranks_on_one_gpu(gpu, tmp_path):
    import torch.multiprocessing as mp
    from paper_2508_13523_b200.driver import RunConfig, run_script
    coeff = tmp_path / "w.coeff"
    coeff.write_text("4\n" + "\n".join(repr(float(b)) for b in np.linspace(0.05, 0.1, 55)) + "\n")
    out = str(tmp_path / "dist.npz")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(coeff), out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    got = np.load(out)
    # full-list LJ took the split (interior while the exchange is in flight, then boundary)
    # launch: flags exist and both parts are non-empty for the 16^3-cell brick pair
    assert 0.0 < got["overlap"][0] < 1.0, got["overlap"]
    for style in ("full", "half"):
        ref = np.array(run_script(LJ, RunConfig(n_ranks=2, list_style=style,
                                                                        newton=(style == "half")),
                                  log=None).results[-1].rows)
        assert np.allclose(got[f"lj_{style}"][:, 1:], ref[:, 1:], rtol=1e-9), style
    ref = np.array(run_script(_snap_script(str(coeff)), RunConfig(n_ranks=2), log=None).results[-1].rows)
    assert np.allclose(got["snap"][:, 1:], ref[:, 1:], rtol=1e-9)
