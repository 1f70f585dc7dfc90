"""Dual-space arrays: space "a" = host numpy, space "b" = device (torch CUDA) storage.

Mirror of mdkk/memspace.py:26-162 with the reference's protocol unchanged
(single writer, copy only when stale, `transfer_count` counts physical
copies), but space "b" is real HBM.  Device rows may be padded: positions and
forces are stored as AoS double4 (x, y, z, pad) so one neighbour gather is one
32-byte sector, while the logical (n, 3) view is what both spaces expose.

Scatter strategies (Serial / Duplicate / Atomic, mdkk/memspace.py:165-254)
are accepted for signature compatibility; on the GPU the deconfliction is
fixed by the list style: full lists are owner-writes (no atomics), half lists
use FP64 atomics (`RED.E.ADD.F64`).
"""

from __future__ import annotations

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


def upload(a: np.ndarray, device) -> torch.Tensor:
    """Host array -> device tensor.  Large arrays are staged through pinned memory
    with torch's multi-threaded host copy, then DMA'd asynchronously (the caching
    host allocator keeps the staging block until the copy completes): ~2x the
    pageable path, whose single-threaded staging is the bottleneck."""
    src = torch.from_numpy(np.ascontiguousarray(a))
    if src.numel() * src.element_size() < _STAGE_MIN or torch.device(device).type != "cuda":
        return src.to(device)
    pin = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
    pin.copy_(src)
    return pin.to(device, non_blocking=True)


def download(t: torch.Tensor) -> np.ndarray:
    """Device tensor (any strides) -> fresh host array: one DMA into pinned staging,
    then torch's multi-threaded copy into new pageable memory (the page faults of a
    fresh 50 MB array are what bound a single-threaded copy: 11 ms -> 2 ms)."""
    if t.numel() * t.element_size() < _STAGE_MIN or not t.is_cuda:
        return t.cpu().numpy()
    pin = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    pin.copy_(t)
    out = np.empty(tuple(t.shape), dtype=pin.numpy().dtype)
    torch.from_numpy(out).copy_(pin)
    return out


_COPY_STREAMS: dict = {}


def download_async(t: torch.Tensor):
    """`download(t)` started now, finished by the returned callable: the DMA into pinned
    staging is queued on a copy stream behind the work already on the current stream, so
    kernels queued next overlap it; the host copy runs when the callable is invoked.
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
        out = np.empty(tuple(pin.shape), dtype=pin.numpy().dtype)
        torch.from_numpy(out).copy_(pin)
        return out
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


class Serial:
    copies = 1


class Duplicate:
    def __init__(self, copies: int | None = None):
        self.copies = int(copies or 1)


class Atomic:
    copies = 1
