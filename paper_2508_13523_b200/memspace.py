"""Dual-space arrays: space "a" = host numpy, space "b" = device (torch CUDA) storage.

Mirror of mdkk/memspace.py:26-162 with the reference's protocol unchanged
(single writer, copy only when stale, `transfer_count` counts physical
copies), but space "b" is real HBM.  Device rows may be padded: positions and
forces are stored as AoS double4 (x, y, z, pad) so one neighbour gather is one
32-byte sector, while the logical (n, 3) view is what both spaces expose.

Scatter strategies (Serial / Duplicate / Atomic) and `ScatterAccumulator`
(mdkk/memspace.py:165-257) run on the device (csrc/scatter.cu): Serial is an
ordered segmented sum (bit-identical to sequential np.add.at), Atomic is
FP64 RED, Duplicate stages one copy per worker and combines them in a fixed
order.  `compute_pair` maps the same strategies onto the half-list force
kernel's partner writes (full lists write owner rows only: nothing to
deconflict).
"""

from __future__ import annotations

import os

import numpy as np
import torch

SPACES = ("a", "b")

_TORCH_DTYPE = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32,
                np.dtype(np.int64): torch.int64, np.dtype(np.complex128): torch.complex128,
                np.dtype(np.int8): torch.int8}


class MemspaceError(RuntimeError):
    """Protocol violation on a dual-space array (mdkk/memspace.py:21-22)."""


class LayoutPolicy:
    """Logical -> storage dimension order, slowest first (mdkk/memspace.py:26-74)."""

    __slots__ = ("order",)

    def __init__(self, order):
        order = tuple(int(d) for d in order)
        if sorted(order) != list(range(len(order))):
            raise ValueError(f"order must be a permutation of 0..{len(order) - 1}, got {order}")
        self.order = order

    @classmethod
    def row_major(cls, ndim: int) -> "LayoutPolicy":
        return cls(range(ndim))

    @classmethod
    def transposed(cls, ndim: int) -> "LayoutPolicy":
        return cls(range(ndim - 1, -1, -1))

    def storage_shape(self, shape) -> tuple[int, ...]:
        return tuple(shape[d] for d in self.order)

    def flat_index(self, idx, shape) -> int:
        if len(idx) != len(self.order):
            raise ValueError("index rank mismatch")
        off = 0
        for d in self.order:
            off = off * shape[d] + idx[d]
        return off

    def view(self, flat, shape):
        """Logical-index view of flat storage (numpy or torch) laid out in this order."""
        shape = tuple(int(s) for s in shape)
        st = flat.reshape(self.storage_shape(shape))
        axes = self.logical_axes()
        return st.transpose(axes) if isinstance(st, np.ndarray) else st.permute(*axes)

    def logical_axes(self) -> tuple[int, ...]:
        return tuple(self.order.index(d) for d in range(len(self.order)))

    def __eq__(self, other):
        return isinstance(other, LayoutPolicy) and self.order == other.order

    def __repr__(self):
        return f"LayoutPolicy(order={self.order})"


_STAGE_MIN = 1 << 20   # bytes: larger host<->device copies go through pinned staging


def pinned_array(a: np.ndarray) -> np.ndarray:
    """A copy of `a` in page-locked host memory (a numpy view of a pinned torch block), so
    that `upload` DMAs it directly; `a` itself when it is small or there is no GPU.  The
    engine keeps the host-side state it generates (lattice positions, seeded velocities)
    this way: the run's first upload is then a plain DMA."""
    a = np.ascontiguousarray(a)
    if a.nbytes < _STAGE_MIN or a.dtype not in _TORCH_DTYPE or not torch.cuda.is_available():
        return a
    pin = torch.empty(a.shape, dtype=_TORCH_DTYPE[a.dtype], pin_memory=True)
    out = pin.numpy()
    torch.from_numpy(out).copy_(torch.from_numpy(a))
    return out


def upload(a: np.ndarray, device) -> torch.Tensor:
    """Host array -> device tensor.  Pinned arrays (`pinned_array`) are one DMA; large
    pageable arrays are staged through pinned memory with torch's multi-threaded host
    copy, then DMA'd asynchronously (the caching host allocator keeps the staging block
    until the copy completes): ~2x the pageable path, whose single-threaded staging is
    the bottleneck."""
    src = torch.from_numpy(np.ascontiguousarray(a))
    if src.numel() * src.element_size() < _STAGE_MIN or torch.device(device).type != "cuda":
        return src.to(device)
    if src.is_pinned():
        # direct DMA; blocking, so the caller may free or rewrite the host array on return
        return src.to(device)
    # staged in ~8 MB chunks: chunk k's DMA overlaps the host copy of chunk k+1
    pin = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
    dst = torch.empty(src.shape, dtype=src.dtype, device=device)
    fs, fp, fd = src.reshape(-1), pin.reshape(-1), dst.reshape(-1)
    step = max(1, (8 << 20) // src.element_size())
    for a0 in range(0, fs.numel(), step):
        a1 = min(fs.numel(), a0 + step)
        fp[a0:a1].copy_(fs[a0:a1])
        fd[a0:a1].copy_(fp[a0:a1], non_blocking=True)
    return dst


def download(t: torch.Tensor) -> np.ndarray:
    """Device tensor (any strides) -> fresh host array: one DMA into a pinned block that
    the returned array then owns (no second host copy: copying 50 MB into fresh pageable
    memory costs ~1.6 ms of page faults even multi-threaded; the block returns to torch's
    caching host allocator when the array is freed)."""
    if t.numel() * t.element_size() < _STAGE_MIN or not t.is_cuda:
        return t.cpu().numpy()
    pin = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    pin.copy_(t)
    return pin.numpy()


_COPY_STREAMS: dict = {}


def download_async(t: torch.Tensor):
    """`download(t)` started now, finished by the returned callable: the DMA into a pinned
    block is queued on a copy stream behind the work already on the current stream, so
    kernels queued next overlap it; the callable waits for it and returns the array.
    The caller must not write `t` afterwards (pass a private buffer)."""
    if t.numel() * t.element_size() < _STAGE_MIN or not t.is_cuda:
        host = t.cpu().numpy()
        return lambda: host
    side = _COPY_STREAMS.get(t.device)
    if side is None:
        side = _COPY_STREAMS[t.device] = torch.cuda.Stream(t.device)
    side.wait_stream(torch.cuda.current_stream(t.device))
    pin = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    with torch.cuda.stream(side):
        pin.copy_(t, non_blocking=True)
        done = torch.cuda.Event()
        done.record(side)
    t.record_stream(side)

    def finish() -> np.ndarray:
        done.synchronize()
        return pin.numpy()   # the array owns the pinned block (see download)
    return finish



class DualArray:
    """Host/device mirrored array with staleness flags (mdkk/memspace.py:77-156).

    ``pad_last`` pads the fastest logical dimension of the device storage
    (used for double4 rows).  ``storage_b`` adopts an existing device tensor.
    """

    def __init__(self, shape, layout_a: LayoutPolicy | None = None, layout_b: LayoutPolicy | None = None,
                 dtype=np.float64, device=None, pad_last: int | None = None, storage_b=None):
        shape = tuple(int(s) for s in shape)
        if not shape or any(s <= 0 for s in shape):
            raise ValueError(f"all extents must be > 0, got {shape}")
        self.shape = shape
        self.dtype = np.dtype(dtype)
        self.layout_a = layout_a or LayoutPolicy.row_major(len(shape))
        self.layout_b = layout_b or LayoutPolicy.transposed(len(shape))
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self._data_a = None    # host storage materialises on first host access
        sshape = list(self.layout_b.storage_shape(shape))
        if pad_last is not None:
            if self.layout_b.order[-1] != len(shape) - 1:
                raise ValueError("padding needs the last logical dim fastest in storage")
            sshape[-1] = pad_last
        if storage_b is not None:
            self.data_b = storage_b
        else:
            self.data_b = torch.zeros(sshape, dtype=_TORCH_DTYPE[self.dtype], device=self.device)
        self.modified_a = False
        self.modified_b = False
        self.transfer_count = 0

    @property
    def data_a(self) -> np.ndarray:
        if self._data_a is None:
            self._data_a = np.zeros(self.shape, dtype=self.dtype)
        return self._data_a

    @data_a.setter
    def data_a(self, value) -> None:
        self._data_a = value

    def _check(self, space):
        if space not in SPACES:
            raise ValueError(f"space must be one of {SPACES}, got {space!r}")
        return space

    def layout(self, space):
        return self.layout_a if self._check(space) == "a" else self.layout_b

    def view(self, space):
        """Logical-index view of the given space (numpy for 'a', torch for 'b')."""
        if self._check(space) == "a":
            return self.data_a
        v = self.data_b.permute(*self.layout_b.logical_axes())
        sl = tuple(slice(0, s) for s in self.shape)
        return v[sl]

    def storage(self, space):
        """The raw storage of a space (numpy for 'a', torch for 'b'), flattened."""
        return self.data_a.reshape(-1) if self._check(space) == "a" else self.data_b.reshape(-1)

    def modified(self, space):
        return self.modified_a if self._check(space) == "a" else self.modified_b

    def mark_modified(self, space):
        space = self._check(space)
        other = "b" if space == "a" else "a"
        if self.modified(other):
            raise MemspaceError(f"space {other!r} has unsynchronized modifications; "
                                f"sync before writing {space!r}")
        if space == "a":
            self.modified_a = True
        else:
            self.modified_b = True

    def sync(self, space):
        space = self._check(space)
        if space == "a" and self.modified_b:
            self.data_a[...] = download(self.view("b"))
            self.transfer_count += 1
            self.modified_b = False
        elif space == "b" and self.modified_a:
            self.view("b").copy_(torch.from_numpy(np.ascontiguousarray(self.data_a)).to(self.device))
            self.transfer_count += 1
            self.modified_a = False
        return self

    def read(self, space):
        self.sync(space)
        return self.view(space)

    def rebind(self, shape, storage_b) -> "DualArray":
        """Re-point this array at new device storage of a new leading extent (same
        dtype / layouts / padding): a fresh, clean mirror without re-running the
        constructor (the engine re-views its row buffers at every rebuild)."""
        self.shape = tuple(int(s) for s in shape)
        self.data_b = storage_b
        self._data_a = None
        self.modified_a = self.modified_b = False
        return self


def create_dual(shape, layout_a=None, layout_b=None, dtype=np.float64, device=None, **kw) -> DualArray:
    return DualArray(shape, layout_a=layout_a, layout_b=layout_b, dtype=dtype, device=device, **kw)


DEFAULT_WORKERS = 4


def worker_count(requested: int | None = None) -> int:
    """Logical worker count honouring the MDKK_THREADS cap (mdkk/parallel.py:15-26).

    On the GPU the workers are Duplicate's staging copies (one per worker)."""
    n = requested if requested is not None else DEFAULT_WORKERS
    cap = os.environ.get("MDKK_THREADS")
    if cap is not None:
        try:
            cap_n = int(cap)
        except ValueError as exc:
            raise ValueError(f"MDKK_THREADS must be an integer, got {cap!r}") from exc
        if cap_n < 1:
            raise ValueError(f"MDKK_THREADS must be >= 1, got {cap_n}")
        n = min(n, cap_n)
    return max(1, int(n))


class Serial:
    """Ordered sequential accumulation (mdkk/memspace.py:165-171): a deterministic
    segmented sum on the device, bit-identical to np.add.at in contribution order."""

    copies = 1

    def __repr__(self):
        return "Serial()"


class Duplicate:
    """Per-worker staging copies plus a fixed-order combine (mdkk/memspace.py:174-183)."""

    def __init__(self, copies: int | None = None):
        self.copies = worker_count(copies)
        if self.copies < 1:
            raise ValueError("Duplicate requires at least one copy")

    def __repr__(self):
        return f"Duplicate(copies={self.copies})"


class Atomic:
    """Concurrent FP64 RED adds on shared storage (mdkk/memspace.py:186-192)."""

    copies = 1

    def __repr__(self):
        return "Atomic()"


STRATEGIES = (Serial, Duplicate, Atomic)


def _lib():
    from . import _lib as lib_mod
    return lib_mod


def ordered_scatter(target: torch.Tensor, ld: int, width: int, idx: torch.Tensor, vals: torch.Tensor) -> None:
    """target[idx[e], :width] += vals[e] one contribution at a time in e order (Serial)."""
    n = int(idx.numel())
    if n == 0:
        return
    sorted_idx, perm = torch.sort(idx, stable=True)
    L = _lib()
    L.call("mdkk_scatter_ordered", target.data_ptr(), ld, width, sorted_idx.data_ptr(), perm.data_ptr(),
           vals.data_ptr(), n, L.stream(target.device))


def atomic_scatter(target: torch.Tensor, ld: int, width: int, idx: torch.Tensor, vals: torch.Tensor) -> None:
    n = int(idx.numel())
    if n:
        L = _lib()
        L.call("mdkk_scatter_atomic", target.data_ptr(), ld, width, idx.data_ptr(), vals.data_ptr(), n,
               L.stream(target.device))


def combine_copies(stage: torch.Tensor, out: torch.Tensor) -> None:
    """out += ((stage[0] + stage[1]) + ...) element-wise (Duplicate's finalize)."""
    copies = int(stage.shape[0])
    n = int(out.numel())
    if n:
        L = _lib()
        L.call("mdkk_scatter_combine", stage.data_ptr(), copies, int(stage[0].numel()), out.data_ptr(), n,
               L.stream(out.device))


class ScatterAccumulator:
    """Indexed accumulation into a dense device target (mdkk/memspace.py:198-254).

    Contributions index the first axis of ``target_shape``; values carry the
    remaining axes.  ``finalize`` is a barrier and returns the host array (the
    reference's return type); ``finalize_device`` returns the device tensor.
    FP64 only (the kernels accumulate in double).
    """

    def __init__(self, target_shape, strategy=None, dtype=np.float64, device=None):
        self.target_shape = tuple(int(s) for s in target_shape)
        if any(s < 0 for s in self.target_shape):
            raise ValueError(f"invalid target shape {self.target_shape}")
        self.strategy = strategy if strategy is not None else Serial()
        if not isinstance(self.strategy, STRATEGIES):
            raise TypeError(f"unknown scatter strategy {self.strategy!r}")
        if np.dtype(dtype) != np.float64:
            raise TypeError("ScatterAccumulator accumulates in float64 on the device")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._n = self.target_shape[0] if self.target_shape else 0
        self._width = int(np.prod(self.target_shape[1:])) if len(self.target_shape) > 1 else 1
        rows = max(self._n, 0)
        if isinstance(self.strategy, Duplicate):
            self._staging = torch.zeros((self.strategy.copies, rows * self._width), dtype=torch.float64,
                                        device=self.device)
            self._pending = [[] for _ in range(self.strategy.copies)]
        else:
            self._staging = None
            self._pending = [[]]
        self._data = torch.zeros(rows * self._width, dtype=torch.float64, device=self.device)
        self._bad = torch.empty(1, dtype=torch.int64, device=self.device)
        self._finalized = False

    def _check_indices(self, idx: torch.Tensor) -> None:
        if idx.numel() == 0:
            return
        self._bad.fill_(-1)   # all ones = no bad index
        L = _lib()
        L.call("mdkk_index_range", idx.data_ptr(), int(idx.numel()), self._n, self._bad.data_ptr(),
               L.stream(self.device))
        e = int(self._bad.item())
        if e != -1:
            raise IndexError(f"scatter index {int(idx[e].item())} out of range [0, {self._n})")

    def add(self, indices, values, worker: int = 0) -> None:
        """Accumulate ``values`` at first-axis ``indices`` on behalf of ``worker``."""
        if self._finalized:
            raise MemspaceError("accumulator already finalized")
        idx = torch.as_tensor(np.asarray(indices) if not torch.is_tensor(indices) else indices)
        idx = idx.to(device=self.device, dtype=torch.int64).reshape(-1).contiguous()
        vals = torch.as_tensor(np.asarray(values, dtype=np.float64) if not torch.is_tensor(values) else values)
        vals = vals.to(device=self.device, dtype=torch.float64).reshape(idx.numel(), self._width).contiguous()
        self._check_indices(idx)
        if isinstance(self.strategy, Atomic):
            atomic_scatter(self._data, self._width, self._width, idx, vals)
        elif isinstance(self.strategy, Serial):
            self._pending[0].append((idx, vals))
        else:
            self._pending[worker % self.strategy.copies].append((idx, vals))

    def finalize_device(self) -> torch.Tensor:
        """Barrier: combine staged contributions; the dense result stays on the device."""
        if self._finalized:
            raise MemspaceError("accumulator already finalized")
        self._finalized = True
        if isinstance(self.strategy, Serial):
            self._flush(self._data, self._pending[0])
        elif isinstance(self.strategy, Duplicate):
            for c, chunks in enumerate(self._pending):
                self._flush(self._staging[c], chunks)
            combine_copies(self._staging, self._data)
            self._staging = None
        self._pending = None
        return self._data.view(self.target_shape) if self.target_shape else self._data

    def finalize(self) -> np.ndarray:
        """Barrier: combine staged contributions and return the dense (host) result."""
        return self.finalize_device().cpu().numpy()

    def _flush(self, target, chunks):
        if not chunks:
            return
        idx = torch.cat([c[0] for c in chunks])
        vals = torch.cat([c[1] for c in chunks])
        ordered_scatter(target, self._width, self._width, idx, vals)


def scatter_accumulate(acc: ScatterAccumulator, contributions) -> np.ndarray:
    """Apply ``(index, value)`` contributions and finalize (mdkk/memspace.py:257-276):
    Duplicate splits the list into one contiguous chunk per copy; Serial and
    Atomic apply it in the given order."""
    contributions = list(contributions)
    if contributions:
        idx = np.asarray([c[0] for c in contributions])
        vals = np.asarray([c[1] for c in contributions])
        copies = acc.strategy.copies
        if copies <= 1 or len(contributions) < copies:
            acc.add(idx, vals, worker=0)
        else:
            bounds = np.linspace(0, len(contributions), copies + 1).astype(int)
            for w in range(copies):
                lo, hi = bounds[w], bounds[w + 1]
                if hi > lo:
                    acc.add(idx[lo:hi], vals[lo:hi], worker=w)
    return acc.finalize()
