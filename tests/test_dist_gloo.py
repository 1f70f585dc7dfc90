"""Host logic of the one-rank-per-GPU halo exchange, world_size 2 over gloo on CPU.

`DistSystem` (paper_2508_13523_b200/dist.py) is driven with a torch-CPU test
double of its kernel layer (the product always uses the CUDA library); the
ghost sets, forward positions, reverse folds and migration are compared with
the oracle's in-process 2-rank RankedSystem (mdkk/domain.py:246-334).
"""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class TorchOps:
    """CPU stand-in for dist.CudaOps (same semantics: stable, combo-major halo order)."""

    def __init__(self, device):
        self.device = device

    def halo_select(self, x, n, tab, C_):
        p = x[:n, :3]
        out, totals = [], []
        for c in range(C_):
            lo, hi, sh = tab[c, :3], tab[c, 3:6], tab[c, 6:9]
            q = p + sh
            m = ((q >= lo) & (q < hi)).all(dim=1)
            idx = torch.nonzero(m).flatten().to(torch.int32)
            out.append(idx)
            totals.append(len(idx))
        idx = torch.cat(out) if out else torch.zeros(0, dtype=torch.int32)
        return torch.cat([idx, torch.zeros(1, dtype=torch.int32)]), np.array(totals, dtype=np.int64)

    def pack(self, x, idx, code, shifts, n, out):
        if n:
            out[:n, :3] = x[idx[:n].long(), :3] + shifts[code[:n].long()]
            out[:n, 3] = 0.0

    def fold(self, f, idx, buf, n):
        if n:
            f.index_add_(0, idx[:n].long(), buf[:n].clone())

    def gather_rows(self, src, idx, n, out):
        if n:
            out[:n] = src[idx[:n].long()]

    def gather_i64(self, src, idx, n, out):
        if n:
            out[:n] = src[idx[:n].long()]

    def wrap(self, x, n, lengths):
        L = torch.as_tensor(lengths)
        x[:n, :3] = x[:n, :3] - L * torch.floor(x[:n, :3] / L)

    def owner_partition(self, x, n, lengths, grid, R):
        g = torch.as_tensor(grid)
        c = torch.floor(x[:n, :3] / torch.as_tensor(lengths) * g.double()).long()
        c = torch.minimum(torch.clamp(c, min=0), g - 1)
        key = (c[:, 0] * g[1] + c[:, 1]) * g[2] + c[:, 2]
        order = torch.argsort(key, stable=True).to(torch.int32)
        start = np.concatenate([[0], np.cumsum(np.bincount(key.numpy(), minlength=R))])
        return start.astype(np.int64), order

    def cell_order(self, x, n, lo, hi, width):
        return torch.arange(max(n, 1), dtype=torch.int32)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import md
        from paper_2508_13523_b200 import Box
        from paper_2508_13523_b200.dist import DistSystem
        pos, L = md.random_config(200, 0.7, seed=5)
        vel = np.random.default_rng(6).normal(size=pos.shape)
        cpu = torch.device("cpu")
        ds = DistSystem.distribute(Box(L), pos, vel, device=cpu, ops=TorchOps(cpu))
        ds.exchange_ghosts(1.3)
        s = ds.store
        ghosts = {(int(g), tuple(np.rint(sh / L).astype(int)), tuple(np.round(p, 12)))
                  for g, sh, p in zip(s.global_ids[s.n_local:], s.ghost_shift[s.n_local:],
                                      s.positions()[s.n_local:])}
        # move owned atoms a little, forward, check ghost = owner + shift
        s.x[: s.n_local, :3] += 0.01
        s.device_wrote(pos=True)
        ds.forward_comm()
        fwd = {(int(g), tuple(np.round(p, 12))) for g, p in zip(s.global_ids[s.n_local:], s.positions()[s.n_local:])}
        # reverse: unit force on every ghost row -> owners receive one per ghost copy
        s.f.zero_()
        s.f[s.n_local:s.n_total, :3] = 1.0
        s.device_wrote(force=True)
        ds.reverse_comm()
        folded = ds.gather_forces()
        # migrate after a large move, then gather
        s.x[: s.n_local, 0] += 3.0
        s.device_wrote(pos=True)
        ds.migrate(1.3)
        gp, gv, gid = ds.gather()
        q.put((rank, ghosts, fwd, folded, gp, gv, gid, ds.store.n_local))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(400)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_dist_system_matches_oracle(world):
    """World 2, 4 and 8: grids (2,1,1), (2,2,1), (2,2,2) -- with two bricks along an axis the
    left and right neighbour are the same rank under different periodic shifts."""
    from oracle import md
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=360)
        res[r[0]] = r
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    pos, L = md.random_config(200, 0.7, seed=5)
    vel = np.random.default_rng(6).normal(size=pos.shape)
    osys = md.Ranked(L, world, pos, vel)
    osys.exchange_ghosts(1.3)
    for r, ork in enumerate(osys.ranks):
        ref = {(int(g), tuple(np.rint(sh / L).astype(int)), tuple(np.round(p, 12)))
               for g, sh, p in zip(ork.gid[ork.n_local:], ork.shift[ork.n_local:], ork.x[ork.n_local:])}
        assert res[r][1] == ref
    # forward comm: ghost = (owner + 0.01) + shift, exactly as the oracle computes it
    for rk in osys.ranks:
        rk.x[: rk.n_local] += 0.01
    osys.forward()
    for r, ork in enumerate(osys.ranks):
        ref = {(int(g), tuple(np.round(p, 12))) for g, p in zip(ork.gid[ork.n_local:], ork.x[ork.n_local:])}
        assert res[r][2] == ref
    # reverse comm: each owner gets +1 per ghost image of it anywhere
    for rk in osys.ranks:
        rk.f[:] = 0.0
        rk.f[rk.n_local:] = 1.0
    osys.reverse()
    for r in range(world):
        assert np.allclose(res[r][3], osys.gather_forces())
    # migration: same owned sets and gid-ordered state on every rank
    for rk in osys.ranks:
        rk.x[: rk.n_local, 0] += 3.0
    osys.migrate(1.3)
    gp, gv, gid = osys.gather()
    for r in range(world):
        assert np.array_equal(res[r][6], gid)
        assert np.allclose(res[r][4], gp, atol=1e-12) and np.allclose(res[r][5], gv)
    assert sum(res[r][7] for r in range(world)) == 200
    assert [res[r][7] for r in range(world)] == [rk.n_local for rk in osys.ranks]
