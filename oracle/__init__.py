"""CPU oracle for the force-and-neighbor hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the algorithms of the reference
`mdkk` engine (/root/reference/pkg/src/mdkk) that the B200 library replaces:
domain decomposition + ghosts (`domain.py`), cell-list neighbor builds
(`neighbor.py`), the truncated Lennard-Jones pair engine (`pair_lj.py`), the
velocity-Verlet driver (`driver/simulation.py`) and the SNAP descriptor
pipeline (`snap/*.py`).  Every function cites the reference file:line it
follows.

Parity status: PINNED.  The restatement is checked against golden vectors
produced by running the reference itself (tests/golden/make_golden.py, which
imports /root/reference in the build container) and against the reference's
own known-answer values (tests/test_oracle.py).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` legs may import this package, and only as the checker or
the timed CPU baseline.  The product path (`paper_2508_13523_b200`) never
imports it and has no CPU fallback.
"""

from . import md, snap  # noqa: F401
