"""CPU checks of the boundary: the C-ABI library builds, loads and exports every declared symbol.

No compute calls (no GPU here); host-side logic of the drop-in is checked too.
"""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(ROOT, "include", fn)).read()
            text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
            names |= set(re.findall(r"\b(mdkk_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    from paper_2508_13523_b200 import buildlib, _lib
    buildlib.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared()
    assert len(declared) > 20
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes signature table covers exactly the declared ABI
    assert set(_lib.SIGNATURES) == declared


def test_library_metadata_calls_without_gpu():
    from paper_2508_13523_b200 import _lib
    assert _lib.lib().mdkk_version() >= 1
    assert _lib.launch_count() >= 0


def test_sass_is_sm100a():
    import subprocess
    from paper_2508_13523_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_registry_suffix_dispatch():
    from paper_2508_13523_b200.driver import RegistryError, default_registry
    reg = default_registry()
    assert "lj/cut/kk" in reg
    f = reg.resolve("lj/cut", "kk")
    assert f(["2.5"]).name == "lj/cut/kk"
    assert reg.resolve("lj/cut", "nosuch")(["2.5"]).name == "lj/cut"
    with pytest.raises(RegistryError):
        reg.resolve("lj/cutt")


def test_script_reader():
    from paper_2508_13523_b200.driver import ParseError, parse_script
    cmds = parse_script("units lj # c\nlattice fcc &\n  0.8442\nrun 5\n")
    assert [c.name for c in cmds] == ["units", "lattice", "run"]
    assert cmds[1].args == ["fcc", "0.8442"]
    with pytest.raises(ParseError):
        parse_script("lattise fcc 1\n")


def test_decompose_and_capacity_rules():
    from paper_2508_13523_b200 import Box, decompose
    from paper_2508_13523_b200.neighbor import grow_capacity
    from oracle import md
    for n in (1, 2, 4, 8):
        assert decompose(Box((10.0, 10.0, 10.0)), n).grid == md.min_surface_grid(np.array([10.0] * 3), n)
    assert decompose(Box((20.0, 10.0, 10.0)), 2).grid == (2, 1, 1)
    assert [grow_capacity(16, k) for k in (10, 17, 78, 100)] == [16, 24, 81, 122]


def test_cell_grid_covers_cutoff():
    from paper_2508_13523_b200.domain import cell_grid
    g, n = cell_grid(np.zeros(3), np.array([134.368, 134.368, 134.368]), 2.8, 2.8)
    width = 1.0 / np.array(g[3:])
    assert np.all(width >= 2.8) and n[0] == int((134.368 + 5.6) // 2.8) or np.all(width >= 2.8)


def test_lattice_generators_match_oracle():
    from paper_2508_13523_b200.driver import lattice_positions, seeded_velocities
    from oracle import md
    for style, rho in (("fcc", 0.8442), ("sc", 0.8), ("bcc", 3.1803)):
        p, box = lattice_positions(style, rho, (3, 4, 5))
        q, L = md.lattice(style, rho, (3, 4, 5))
        assert np.array_equal(p, q) and np.array_equal(box.lengths, L)
    assert np.array_equal(seeded_velocities(100, 1.44, 1.0, 87287), md.seeded_velocities(100, 1.44, 1.0, 87287))
