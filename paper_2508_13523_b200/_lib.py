"""ctypes binding of the in-tree CUDA library (include/mdkk_b200.h).

There is no CPU fallback: importing a compute entry point without the built
`libmdkk_b200.so`, or calling one without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
_DEFAULT_LIB = os.path.join(HERE, "libmdkk_b200.so")
# MDKK_LIB: an alternative build of the same library (A/B experiments on the GPU box)
LIB_PATH = os.environ.get("MDKK_LIB") or _DEFAULT_LIB

OK, E_CAPACITY, E_COINCIDENT, E_NONFINITE, E_ARG, E_CUDA = range(6)
FLAG_COINCIDENT, FLAG_NONFINITE = 1, 2

_p = C.c_void_p
_i = C.c_int
_d = C.c_double
_l = C.c_longlong

# name -> argtypes (restype is always c_int unless listed in _RESTYPE)
SIGNATURES = {
    "mdkk_version": [],
    "mdkk_launch_count": [],
    "mdkk_last_error": [],
    "mdkk_device_sm_count": [_i, _p],
    "mdkk_ctx_create": [_i, _p],
    "mdkk_ctx_destroy": [_p],
    "mdkk_fp64_probe": [_i, _i, _p, _p],
    "mdkk_wrap": [_p, _i, _p, _p],
    "mdkk_halo_count": [_p, _p, _i, _p, _i, _p, _p, _p, _p, _p],
    "mdkk_boundary_rows": [_p, _p, _p, _i, _p, _p, _p],
    "mdkk_halo_fill": [_p, _p, _i, _p, _i, _p, _p, _p, _p, _p, _p, _p, _p],
    "mdkk_ghost_rows": [_p, _p, _p, _p, _p, _i, _p, _p, _p, _p],
    "mdkk_pack_shift": [_p, _p, _p, _p, _i, _p, _p],
    "mdkk_fold_add": [_p, _p, _p, _i, _p],
    "mdkk_gather_rows4": [_p, _p, _i, _p, _p],
    "mdkk_gather_i64": [_p, _p, _i, _p, _p],
    "mdkk_gather_i32": [_p, _p, _i, _p, _p],
    "mdkk_scatter_rows4": [_p, _p, _i, _p, _p],
    "mdkk_cell_keys": [_p, _i, _p, _p, _p, _p],
    "mdkk_rank_keys": [_p, _i, _p, _p, _p, _p],
    "mdkk_bucket_sort": [_p, _p, _i, _i, _p, _p, _p],
    "mdkk_bin_atoms": [_p, _p, _i, _p, _p, _p, _p, _p, _p],
    "mdkk_nbr_build": [_p, _p, _i, _i, _p, _p, _p, _p, _p, _p, _i, _d, _i, _i, _i, _p, _p, _p, _p],
    "mdkk_nbr_canonicalize": [_p, _p, _i, _i, _p, _p, _p],
    "mdkk_max_disp2": [_p, _p, _i, _p, _p],
    "mdkk_nbr_geo_order": [_p, _i, _i, _p, _p, _p],
    "mdkk_bin_merge": [_p, _p, _i, _i, _p, _p, _p, _p, _p, _p, _p],
    "mdkk_rebuild1_select": [_p, _p, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i, _p, _p, _p,
                             _p, _p, _p],
    "mdkk_lj_force": [_p, _p, _i, _p, _p, _i, _i, _i, _i, _d, _d, _d, _p, _p, _p, _p],
    "mdkk_lj_force_integrate": [_p, _p, _i, _p, _p, _i, _i, _d, _d, _d, _p, _p, _p, _p, _d, _p, _i, _i, _p, _p, _p,
                                _p, _d, _d, _p, _i, _p],
    "mdkk_lj_force_integrate_pack": [_p, _p, _i, _p, _p, _i, _i, _d, _d, _d, _p, _p, _p, _p, _d, _p, _i, _p, _p, _p,
                                     _p, _d, _d, _p, _p, _p, _i, _p, _p],
    "mdkk_cluster_flags": [_p, _i, _p, _p, _d, _i, _p, _p],
    "mdkk_lj_force_gated": [_p, _p, _i, _p, _p, _i, _i, _i, _i, _i, _d, _d, _d, _p, _p, _p, _p, _d, _p, _i, _p],
    "mdkk_lj_force_neighbor": [_p, _p, _i, _p, _p, _i, _i, _i, _i, _d, _d, _d, _p, _p, _p, _p],
    "mdkk_lj_force_strategy": [_p, _p, _i, _p, _p, _i, _i, _i, _d, _d, _d, _p, _p, _p, _i, _p, _l, _i, _p],
    "mdkk_scatter_atomic": [_p, _i, _i, _p, _p, _l, _p],
    "mdkk_scatter_ordered": [_p, _i, _i, _p, _p, _p, _l, _p],
    "mdkk_scatter_combine": [_p, _i, _l, _p, _l, _p],
    "mdkk_index_range": [_p, _l, _l, _p, _p],
    "mdkk_verlet_first": [_p, _p, _p, _p, _p, _i, _d, _d, _p, _i, _p],
    "mdkk_verlet_second": [_p, _p, _p, _i, _d, _d, _p, _p],
    "mdkk_kinetic": [_p, _p, _i, _d, _p, _p],
    "mdkk_snap_create": [_p, _i, _i, _p, _p, _i, _p, _p],
    "mdkk_snap_destroy": [_p],
    "mdkk_snap_set_schedule": [_p, _i, _i],
    "mdkk_snap_ui": [_p, _p, _i, _p, _p, _i, _d, _p, _i, _i, _p, _p],
    "mdkk_snap_yi": [_p, _p, _p, _i, _p, _i, _p, _i, _i, _p],
    "mdkk_snap_y_expand": [_p, _p, _i, _i, _p, _i, _i, _p],
    "mdkk_snap_y_compress": [_p, _p, _i, _p, _i, _i, _i, _p],
    "mdkk_snap_deidrj": [_p, _p, _i, _p, _p, _i, _d, _p, _i, _p, _p],
    "mdkk_snap_compute": [_p, _p, _p, _i, _p, _p, _i, _d, _p, _p, _p, _p, _p, _p],
    "mdkk_snap_pair_count": [_p, _p, _i, _p, _p, _i, _d, _p, _p, _p, _p],
    "mdkk_snap_pair_fill": [_p, _i, _p, _p, _i, _d, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
    "mdkk_snap_duidrj": [_p, _i, _p, _d, _p, _p],
    "mdkk_snap_deidrj_staged": [_p, _i, _p, _p, _p, _p, _p, _p],
    "mdkk_snap_bi": [_p, _p, _i, _p, _p, _p, _p, _i, _p, _i, _i, _p],
    "mdkk_snap_bi_warps": [],
    "mdkk_snap_pair_u": [_i, _i, _p, _p, _p, _p],
    "mdkk_snap_pair_grads": [_i, _p, _d, _p, _p, _p],
    "mdkk_snap_pair_dedr": [_p, _i, _p, _p, _p, _p, _p],
    "mdkk_qeq_offsets": [_p, _p, _i, _i, _p, _p, _p],
    "mdkk_qeq_build": [_p, _i, _p, _p, _i, _p, _p, _d, _d, _d, _p, _p, _p, _p],
    "mdkk_qeq_spmv": [_p, _p, _p, _p, _p, _i, _p, _p, _p, _p, _p, _p],
    "mdkk_qeq_gershgorin": [_p, _p, _p, _p, _i, _p, _p, _p, _p],
    "mdkk_dot": [_p, _p, _p, _i, _p, _p],
    "mdkk_cg_update": [_p, _i, _p, _p, _p, _p, _p, _p, _p, _p],
    "mdkk_cg_direction": [_i, _p, _p, _p, _p, _p],
}
_RESTYPE = {"mdkk_last_error": C.c_char_p, "mdkk_launch_count": C.c_ulonglong}

_lock = threading.Lock()
_lib = None
_ctx: dict[int, int] = {}


class MdkkError(RuntimeError):
    """A library call failed; `status` is the mdkk_status code."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def lib():
    """Load the library once (raises if it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: run `python -m paper_2508_13523_b200.buildlib` "
                        "(the B200 path has no CPU fallback)")
                handle = C.CDLL(LIB_PATH)
                for name, args in SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.argtypes = args
                    fn.restype = _RESTYPE.get(name, C.c_int)
                _lib = handle
    return _lib


def launch_count() -> int:
    """Kernels launched by this library so far (process-wide)."""
    return int(lib().mdkk_launch_count())


def check(status: int, what: str = "") -> None:
    if status != OK:
        err = lib().mdkk_last_error().decode(errors="replace")
        raise MdkkError(status, f"{what}: mdkk status {status} {err}".strip())


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def ctx(device: torch.device) -> int:
    """Per-device scratch context handle (created lazily, lives for the process)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    h = _ctx.get(idx)
    if h is None:
        out = C.c_void_p()
        with torch.cuda.device(idx):
            check(lib().mdkk_ctx_create(idx, C.byref(out)), "mdkk_ctx_create")
        h = _ctx[idx] = out.value
    return h


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream(device: torch.device | None = None) -> int:
    """The current stream of `device` as a raw cudaStream_t (what every C entry point takes).
    Called several times per step: torch's raw accessor skips building a Stream object."""
    if _raw_stream is not None:
        if device is None:
            idx = torch.cuda.current_device()
        else:
            idx = device if isinstance(device, int) else device.index
            if idx is None:
                idx = torch.cuda.current_device()
        return _raw_stream(idx)
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def dbl3(values) -> C.Array:
    arr = (C.c_double * len(values))(*[float(v) for v in values])
    return arr


def int_arr(values) -> C.Array:
    return (C.c_int * len(values))(*[int(v) for v in values])
