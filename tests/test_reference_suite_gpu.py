"""The reference's own hot-path tests, run against the drop-ins.

The unmodified reference engine `mdkk` and its test modules are staged into
baseline/_ref by tools/stage_reference.py (run by `__graft_entry__.build()`;
git-ignored, shipped to the GPU box with the snapshot).  Test 1 runs
mdkk's tests/test_neighbor.py, test_pair_lj.py, test_snap.py, test_driver.py and
test_acceptance.py::test_01/02/03/06/09 in a subprocess with
tests/refsuite/kk_plugin.py, which rebinds mdkk's build / compute_pair / SNAP
stages to paper_2508_13523_b200.plugin before collection: the reference's
assertions, inputs and tolerances, the B200 kernels underneath.  Test 2 runs
the reference's own Simulation with `suffix kk` (the plug-in registry) and
compares its thermo log with the reference's CPU run.
"""

from __future__ import annotations

import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_PKG = os.path.join(REF, "pkg")

pytestmark = pytest.mark.gpu

SUITE = ["tests/test_neighbor.py", "tests/test_pair_lj.py", "tests/test_snap.py", "tests/test_driver.py",
         "tests/test_acceptance.py"]
ACCEPTANCE = "not test_04 and not test_05 and not test_07 and not test_08"   # QEq, torsion, memspace, throughput


def _staged():
    if not (os.path.isdir(os.path.join(REF, "mdkk")) and os.path.isdir(os.path.join(REF_PKG, "tests"))):
        pytest.skip("reference not staged in baseline/_ref (run tools/stage_reference.py)")


def test_reference_hot_path_suite_on_drop_ins(gpu):
    _staged()
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests", "refsuite")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "kk_plugin", "-p", "no:cacheprovider", "--rootdir", REF_PKG,
           "-o", "addopts=", *SUITE, "-k", ACCEPTANCE]
    out = subprocess.run(cmd, cwd=REF_PKG, env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                         timeout=1500)
    tail = "\n".join(out.stdout.splitlines()[-40:])
    assert out.returncode == 0, tail
    passed = int(re.search(r"(\d+) passed", out.stdout).group(1))
    launches = int(re.search(r"kk device launches: (\d+)", out.stdout).group(1))
    assert passed >= 110 and launches > 1000, tail   # every selected reference test
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "reference_suite.txt"), "w") as fh:
        fh.write(out.stdout)


def _ref_modules():
    _staged()
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import mdkk.driver.simulation as sim
    return sim


def _rows(sim_mod, text, registry=None, config=None):
    s = sim_mod.Simulation(config or sim_mod.RunConfig(), registry=registry, log=None)
    s.execute(sim_mod.parse_script(text))
    return s, np.array(s.results[-1].rows)


def test_reference_engine_runs_kk_styles(gpu):
    """`suffix kk` in the reference's own Simulation resolves lj/cut/kk and snap/kk (plug-in
    registry); their thermo logs equal the reference's CPU styles'."""
    from paper_2508_13523_b200 import plugin
    sim = _ref_modules()
    reg = sim.default_registry()
    plugin.register(reg)
    with open(os.path.join(REF_PKG, "scripts", "melt.in")) as fh:
        melt = fh.read().replace("run 1000", "run 200")
    for cfg in (dict(), dict(n_ranks=2), dict(list_style="full", newton=False), dict(strategy="atomic")):
        s_kk, rows_kk = _rows(sim, "suffix kk\n" + melt, reg, sim.RunConfig(**cfg))
        assert s_kk.style.name == "lj/cut/kk"
        _, rows_ref = _rows(sim, melt, None, sim.RunConfig(**cfg))
        assert rows_kk.shape == rows_ref.shape
        assert np.allclose(rows_kk[:, 1:], rows_ref[:, 1:], rtol=1e-10, atol=1e-12), cfg
    with open(os.path.join(REF_PKG, "scripts", "snap.in")) as fh:
        snap = fh.read()
    cwd = os.getcwd()
    os.chdir(REF_PKG)   # snap.in names its coefficient file relative to pkg/
    try:
        s_kk, rows_kk = _rows(sim, snap.replace("suffix opt", "suffix kk"), reg)
        assert s_kk.style.name == "snap/kk"
        _, rows_ref = _rows(sim, snap.replace("suffix opt", "suffix off"), None)
    finally:
        os.chdir(cwd)
    assert np.allclose(rows_kk[:, 1:], rows_ref[:, 1:], rtol=1e-10, atol=1e-12)
