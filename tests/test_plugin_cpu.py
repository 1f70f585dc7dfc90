"""Host-side checks of the drop-in plug-in (paper_2508_13523_b200/plugin.py); no kernels run here."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _run(code: str) -> str:
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]))
    out = subprocess.run([sys.executable, "-c", code], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stdout
    return out.stdout


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "mdkk")), reason="reference not staged")
def test_install_rebinds_every_hot_path_binding_and_registers_kk_styles():
    out = _run(
        "from paper_2508_13523_b200 import plugin\n"
        "names = plugin.install()\n"
        "import mdkk.driver.simulation as s, mdkk.neighbor as n, mdkk.pair_lj as p, mdkk.snap as sn\n"
        "assert n.build is plugin.build and p.compute_pair is plugin.compute_pair\n"
        "assert s.compute_pair is plugin.compute_pair and s.build is plugin.build\n"
        "assert sn.compute_ui is plugin.compute_ui and s.compute_fused_deidrj is plugin.compute_fused_deidrj\n"
        "reg = s.default_registry()\n"
        "assert reg.resolve('lj/cut', 'kk')(['2.5']).name == 'lj/cut/kk'\n"
        "assert reg.resolve('lj/cut/opt', 'kk')(['2.5']).default_mode == 'neighbor'\n"
        "assert reg.resolve('lj/cut', 'opt')(['2.5']).name == 'lj/cut/opt'\n"
        "plugin.uninstall()\n"
        "import mdkk.neighbor as n2\n"
        "assert n2.build is not plugin.build and s.default_registry().names() == "
        "['lj/cut', 'lj/cut/opt', 'snap', 'snap/opt']\n"
        "print(len(names))\n")
    assert int(out.strip().splitlines()[-1]) >= 20


def test_saturation_bench_validates_before_touching_the_device():
    """bench_saturation's argument checks (mdkk/driver/bench.py:105-115) and the CSV schema."""
    from paper_2508_13523_b200.driver.bench import BenchResult, bench_saturation
    from paper_2508_13523_b200.driver.simulation import RunError
    with pytest.raises(RunError):
        bench_saturation("eam", [1000])
    with pytest.raises(RunError):
        bench_saturation("lj", [1000], reps=0)
    r = BenchResult("lj", [(1000, 2.5e8), (8000, 1.5e9)])
    assert list(r.sizes) == [1000, 8000] and r.rates[1] == 1.5e9


def test_saturation_csv_schema(tmp_path):
    from paper_2508_13523_b200.driver.bench import BenchResult
    p = tmp_path / "s.csv"
    BenchResult("snap", [(64000, 1.25e8)]).write_csv(str(p))
    assert p.read_text().splitlines() == ["n_atoms,atom_steps_per_second", "64000,1.25e+08"]
