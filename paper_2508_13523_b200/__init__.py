"""B200-native force-and-neighbor hot path of arXiv 2508.13523 (LAMMPS-KOKKOS), as a drop-in for `mdkk`.

Modules mirror the reference package layout (mdkk/{domain,neighbor,pair_lj,
snap,driver}); every per-atom operation runs in hand-written sm_100a CUDA
(csrc/, exported through the C ABI in include/mdkk_b200.h).  There is no CPU
fallback: compute entry points raise if the library is not built.
"""

__version__ = "0.1.0"

from .domain import AtomStore, Box, DomainError, RankedSystem, RankSet, decompose  # noqa: E402
from .memspace import (Atomic, DualArray, Duplicate, LayoutPolicy, MemspaceError, ScatterAccumulator,  # noqa: E402
                       Serial, create_dual, scatter_accumulate)
from .neighbor import (NeighborError, NeighborList, StaleListError, any_needs_rebuild, brute_force_pairs,  # noqa: E402
                       build, build_all)
from .pair_lj import LJCut, PairError, PairParams, PairResult, compute_pair, u2_lj  # noqa: E402

__all__ = ["AtomStore", "Box", "DomainError", "RankedSystem", "RankSet", "decompose", "DualArray",
           "LayoutPolicy", "MemspaceError", "ScatterAccumulator", "Serial", "Duplicate", "Atomic", "create_dual",
           "scatter_accumulate", "NeighborError", "NeighborList", "StaleListError",
           "any_needs_rebuild", "brute_force_pairs", "build", "build_all", "LJCut", "PairError", "PairParams", "PairResult",
           "compute_pair", "u2_lj"]
