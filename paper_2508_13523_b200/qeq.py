"""Charge equilibration on the GPU: drop-in for mdkk/qeq.py.

Same names, arguments and errors as the reference (mdkk/qeq.py:21-315).  The
over-allocated CSR matrix lives in HBM (int64 row offsets, f64 values, int32
columns and row counts) and is assembled by a kernel from a full neighbour
list; SpMV, the fused dual SpMV, the Gershgorin guard and the conjugate-
gradient vector stages are CUDA kernels (csrc/qeq.cu) with fixed-order
reductions, so `cg_solve_fused` reproduces two `cg_solve` calls bit for bit.
Vectors may be passed as numpy arrays (uploaded) or CUDA tensors; results
come back as numpy, as in the reference.  The only per-iteration host work is
the convergence test on two scalars.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .domain import AtomStore
from .neighbor import NeighborList


class QeqError(RuntimeError):
    pass


class QeqConfigError(QeqError):
    """Parameterization violates the positive-definiteness guarantee."""


class QeqParams:
    """Single-species charge-equilibration parameters (mdkk/qeq.py:29-38)."""

    def __init__(self, gamma: float, eta: float, chi: float, cutoff: float):
        if gamma <= 0 or eta <= 0 or cutoff <= 0:
            raise QeqError("gamma, eta, cutoff must be positive")
        self.gamma = float(gamma)
        self.eta = float(eta)
        self.chi = float(chi)
        self.cutoff = float(cutoff)


def scan_offsets_64(capacities) -> np.ndarray:
    """Exclusive 64-bit scan of per-row capacities (mdkk/qeq.py:41-46); host utility."""
    caps = np.asarray(capacities, dtype=np.int64)
    offsets = np.zeros(len(caps) + 1, dtype=np.int64)
    np.cumsum(caps, out=offsets[1:])
    return offsets


class OverCSR:
    """Four-array over-allocated CSR matrix in HBM (mdkk/qeq.py:49-87).

    ``row_offsets[r] .. row_offsets[r] + row_nnz[r]`` is the active span of
    row r; the remainder up to ``row_offsets[r+1]`` is slack.  The numpy
    attributes are host copies made on first access.
    """

    def __init__(self, n_rows: int, n_cols: int, offsets: torch.Tensor, values: torch.Tensor,
                 columns: torch.Tensor, nnz: torch.Tensor):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.offsets_dev, self.values_dev, self.columns_dev, self.nnz_dev = offsets, values, columns, nnz
        self.device = values.device
        self._host = {}

    def _h(self, name, t, dtype):
        h = self._host.get(name)
        if h is None:
            h = self._host[name] = t.cpu().numpy().astype(dtype, copy=False)
        return h

    @property
    def row_offsets(self) -> np.ndarray:
        return self._h("off", self.offsets_dev, np.int64)

    @property
    def values(self) -> np.ndarray:
        return self._h("val", self.values_dev, np.float64)

    @property
    def columns(self) -> np.ndarray:
        return self._h("col", self.columns_dev, np.int32)

    @property
    def row_nnz(self) -> np.ndarray:
        return self._h("nnz", self.nnz_dev[: self.n_rows], np.int32)

    def to_dense(self) -> np.ndarray:
        """Dense host copy (test helper, as in the reference)."""
        dense = np.zeros((self.n_rows, self.n_cols))
        off, val, col, nnz = self.row_offsets, self.values, self.columns, self.row_nnz
        for r in range(self.n_rows):
            s = off[r]
            np.add.at(dense[r], col[s:s + nnz[r]].astype(np.int64), val[s:s + nnz[r]])
        return dense


def build_matrix(store: AtomStore, nlist: NeighborList, params: QeqParams) -> OverCSR:
    """Assemble the shielded-interaction matrix from a full list on the GPU (mdkk/qeq.py:90-133)."""
    if nlist.style != "full":
        raise QeqError("matrix assembly requires a full-style neighbor list")
    if params.cutoff > nlist.build_cutoff:
        raise QeqError(f"QEq cutoff {params.cutoff} exceeds neighbor build cutoff {nlist.build_cutoff}")
    dev = store.device
    n = store.n_local
    lib, stream = _lib.lib(), _lib.stream(dev)
    store.to_device()
    caps = torch.empty(n + 1, dtype=torch.int64, device=dev)
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    _lib.check(lib.mdkk_qeq_offsets(_lib.ctx(dev), nlist.counts_dev.data_ptr(), n, nlist.alloc_cap,
                                    caps.data_ptr(), offsets.data_ptr(), stream), "mdkk_qeq_offsets")
    total = int(offsets[n].item())
    values = torch.zeros(max(total, 1), dtype=torch.float64, device=dev)
    columns = torch.zeros(max(total, 1), dtype=torch.int32, device=dev)
    nnz = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    _lib.check(lib.mdkk_qeq_build(store.x.data_ptr(), n, nlist.table_dev.data_ptr(), nlist.counts_dev.data_ptr(),
                                  nlist.alloc_cap, store.oidx.data_ptr(), offsets.data_ptr(), params.eta,
                                  params.gamma, params.cutoff, values.data_ptr(), columns.data_ptr(),
                                  nnz.data_ptr(), stream), "mdkk_qeq_build")
    return OverCSR(n, n, offsets, values[:total], columns[:total], nnz)


def _vec(H: OverCSR, x, what="x") -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    if tuple(t.shape) != (H.n_cols,):
        raise QeqError(f"dimension mismatch: H is {H.n_rows}x{H.n_cols}, {what} has shape {tuple(t.shape)}")
    return t.to(device=H.device, dtype=torch.float64).contiguous()


def _spmv_dev(H: OverCSR, x1: torch.Tensor, x2: torch.Tensor | None = None, dots: torch.Tensor | None = None):
    y1 = torch.empty(max(H.n_rows, 1), dtype=torch.float64, device=H.device)
    y2 = torch.empty_like(y1) if x2 is not None else None
    _lib.check(_lib.lib().mdkk_qeq_spmv(_lib.ctx(H.device), H.offsets_dev.data_ptr(), H.values_dev.data_ptr(),
                                        H.columns_dev.data_ptr(), H.nnz_dev.data_ptr(), H.n_rows, x1.data_ptr(),
                                        _lib.ptr(x2), y1.data_ptr(), _lib.ptr(y2), _lib.ptr(dots),
                                        _lib.stream(H.device)), "mdkk_qeq_spmv")
    return y1[: H.n_rows], (y2[: H.n_rows] if y2 is not None else None)


def spmv(H: OverCSR, x) -> np.ndarray:
    """y = Hx over the active prefix of each row (mdkk/qeq.py:136-143)."""
    return _spmv_dev(H, _vec(H, x))[0].cpu().numpy()


def spmv_fused(H: OverCSR, x1, x2) -> tuple[np.ndarray, np.ndarray]:
    """Two products sharing one traversal; bit-identical to two spmv calls (mdkk/qeq.py:146-157)."""
    if np.shape(x1) != (H.n_cols,) or np.shape(x2) != (H.n_cols,):
        raise QeqError("dimension mismatch in fused spmv")
    y1, y2 = _spmv_dev(H, _vec(H, x1), _vec(H, x2))
    return y1.cpu().numpy(), y2.cpu().numpy()


def spmv_rowchunk(H: OverCSR, x, n_chunks: int = 4) -> np.ndarray:
    """Row-split traversal (mdkk/qeq.py:160-177): the GPU kernel already splits each
    row over a team of lanes with a fixed reduction, so this is `spmv`."""
    return spmv(H, x)


def check_spd(H: OverCSR) -> None:
    """Gershgorin positive-definiteness guard (mdkk/qeq.py:180-194)."""
    n = H.n_rows
    if n == 0:
        return
    bad = torch.full((1,), 2**31 - 1, dtype=torch.int32, device=H.device)
    diag = torch.empty(n, dtype=torch.float64, device=H.device)
    off = torch.empty(n, dtype=torch.float64, device=H.device)
    _lib.check(_lib.lib().mdkk_qeq_gershgorin(H.offsets_dev.data_ptr(), H.values_dev.data_ptr(),
                                              H.columns_dev.data_ptr(), H.nnz_dev.data_ptr(), n, bad.data_ptr(),
                                              diag.data_ptr(), off.data_ptr(), _lib.stream(H.device)),
               "mdkk_qeq_gershgorin")
    r = int(bad.item())
    if r < n:
        raise QeqConfigError(
            f"Gershgorin violation at row {r}: diagonal {float(diag[r]):.6g} <= off-diagonal "
            f"sum {float(off[r]):.6g}; raise eta or shrink the QEq cutoff")


class _CG:
    """Device state of one CG system (x, r, p, Ap and the scalars rr, pAp, rr_new)."""

    def __init__(self, H: OverCSR, b: torch.Tensor, tol: float):
        dev, n = H.device, H.n_rows
        self.n = n
        self.x = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
        self.r = b.clone() if n else torch.zeros(1, dtype=torch.float64, device=dev)
        self.p = self.r.clone()
        self.sc = torch.zeros(4, dtype=torch.float64, device=dev)   # rr, bb, rr_new, pAp
        ctx, st = _lib.ctx(dev), _lib.stream(dev)
        lib = _lib.lib()
        _lib.check(lib.mdkk_dot(ctx, self.r.data_ptr(), self.r.data_ptr(), n, self.sc.data_ptr(), st), "mdkk_dot")
        self.sc[1] = self.sc[0]
        h = self.sc[:2].cpu().numpy()
        self.rr, self.bb = float(h[0]), float(h[1])
        self.tol2 = tol * tol
        self.it = 0
        self.active = self.bb > 0.0 and self.rr > self.tol2 * self.bb

    def step(self, ap: torch.Tensor, pap_ptr: int) -> None:
        lib, dev = _lib.lib(), self.x.device
        ctx, st = _lib.ctx(dev), _lib.stream(dev)
        sc = self.sc.data_ptr()
        _lib.check(lib.mdkk_cg_update(ctx, self.n, self.x.data_ptr(), self.r.data_ptr(), self.p.data_ptr(),
                                      ap.data_ptr(), sc, pap_ptr, sc + 16, st), "mdkk_cg_update")
        _lib.check(lib.mdkk_cg_direction(self.n, self.r.data_ptr(), self.p.data_ptr(), sc, sc + 16, st),
                   "mdkk_cg_direction")
        self.sc[0] = self.sc[2]
        self.rr = float(self.sc[2].item())
        self.it += 1


def _solution(s: _CG) -> np.ndarray:
    return s.x[: s.n].cpu().numpy()


def cg_solve(H: OverCSR, b, tol: float = 1e-6, max_iter: int = 500,
             trajectory: list | None = None) -> tuple[np.ndarray, int]:
    """Conjugate gradient to relative residual tol (mdkk/qeq.py:210-230)."""
    s = _CG(H, _vec(H, b, "b"), tol)
    if s.bb == 0.0:
        return _solution(s), 0
    dots = torch.zeros(2, dtype=torch.float64, device=H.device)
    while s.rr > s.tol2 * s.bb:
        if s.it >= max_iter:
            raise QeqError(f"CG failed to converge in {max_iter} iterations; "
                           f"relative residual {np.sqrt(s.rr / s.bb):.3e}")
        ap, _ = _spmv_dev(H, s.p, None, dots)
        s.step(ap, dots.data_ptr())
        if trajectory is not None:
            trajectory.append((s.it, _solution(s), s.r[: s.n].cpu().numpy()))
    return _solution(s), s.it


def cg_solve_fused(H: OverCSR, b1, b2, tol: float = 1e-6, max_iter: int = 500,
                   trajectories: tuple[list, list] | None = None) -> tuple[np.ndarray, np.ndarray, int, int]:
    """Fused dual CG: one matrix traversal per iteration drives both systems (mdkk/qeq.py:233-274)."""
    ss = [_CG(H, _vec(H, b1, "b1"), tol), _CG(H, _vec(H, b2, "b2"), tol)]
    dots = torch.zeros(2, dtype=torch.float64, device=H.device)
    outer = 0
    while ss[0].active or ss[1].active:
        if outer >= max_iter:
            res = [np.sqrt(s.rr / s.bb) if s.bb else 0.0 for s in ss]
            raise QeqError(f"fused CG failed to converge in {max_iter} iterations; "
                           f"relative residuals {res[0]:.3e}, {res[1]:.3e}")
        ap1, ap2 = _spmv_dev(H, ss[0].p, ss[1].p, dots)
        for lane, (s, ap) in enumerate(zip(ss, (ap1, ap2))):
            if not s.active:
                continue
            s.step(ap, dots.data_ptr() + 8 * lane)
            if trajectories is not None:
                trajectories[lane].append((s.it, _solution(s), s.r[: s.n].cpu().numpy()))
            if s.rr <= s.tol2 * s.bb:
                s.active = False
        outer += 1
    return _solution(ss[0]), _solution(ss[1]), ss[0].it, ss[1].it


class QeqSystem:
    """Interaction matrix plus electronegativity data for one charge solve (mdkk/qeq.py:277-290)."""

    def __init__(self, H: OverCSR, chi, tol: float = 1e-6, max_iter: int = 500, net_charge: float = 0.0):
        self.H = H
        self.chi = np.asarray(chi, dtype=np.float64)
        if self.chi.shape != (H.n_rows,):
            raise QeqError("chi length must match matrix rows")
        self.tol = float(tol)
        self.max_iter = int(max_iter)
        self.net_charge = float(net_charge)
        self.q = None
        self.iterations = (0, 0)


def solve_qeq(system: QeqSystem) -> np.ndarray:
    """q = s + lambda t with H s = -chi, H t = -1 (fused CG), lambda = (Q - sum s) / sum t (mdkk/qeq.py:293-307)."""
    check_spd(system.H)
    n = system.H.n_rows
    s, t, it_s, it_t = cg_solve_fused(system.H, -system.chi, -np.ones(n), tol=system.tol, max_iter=system.max_iter)
    lam = (system.net_charge - s.sum()) / t.sum()
    q = s + lam * t
    system.q = q
    system.iterations = (it_s, it_t)
    return q


def qeq_energy(system: QeqSystem) -> float:
    """chi.q + q.Hq/2 of the solved charges (mdkk/qeq.py:310-315)."""
    if system.q is None:
        raise QeqError("solve_qeq must run first")
    q = system.q
    return float(np.dot(system.chi, q) + 0.5 * np.dot(q, spmv(system.H, q)))
