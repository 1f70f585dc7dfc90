"""Driver-level tests mirrored from mdkk tests/test_driver.py (registry, script reader,
lattices, velocities on CPU; runs, reproducibility and error paths on the GPU)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2508_13523_b200.driver import (RegistryError, RunConfig, RunError, StyleRegistry, default_registry,
                                          lattice_positions, parse_script, run_script, seeded_velocities)
from paper_2508_13523_b200.driver.script import ParseError

SILENT = None

MINI = """\
units lj
boundary p p p
lattice fcc 0.8
create_box 5 5 5
create_atoms
mass 1.0
velocity 0.1 1234
pair_style lj/cut 1.5
pair_coeff 1.0 1.0
timestep 0.004
thermo 10
run 20
"""


# ------------------------------------------------------------------ CPU part
def test_parse_basic_tokenization():
    text = "# leading comment\nunits lj\n\nlattice fcc 0.85   # trailing comment\ncreate_box 2 2 2\n"
    cmds = parse_script(text)
    assert [c.name for c in cmds] == ["units", "lattice", "create_box"]
    assert cmds[1].args == ["fcc", "0.85"] and cmds[1].line_no == 4


def test_parse_continuation_and_errors():
    cmds = parse_script("qeq on 0.8 &\n  # spacer\n\n  20.0 -0.35 &\n 2.0\nrun 0\n")
    assert cmds[0].name == "qeq" and cmds[0].args == ["on", "0.8", "20.0", "-0.35", "2.0"]
    assert cmds[0].line_no == 1 and cmds[1].line_no == 6
    with pytest.raises(ParseError, match="did you mean"):
        parse_script("lattise fcc 0.8\n")
    with pytest.raises(ParseError):
        parse_script("qeq on 1.0\n")
    with pytest.raises(ParseError):
        parse_script("qeq maybe\n")


def test_registry_resolution_order():
    reg = StyleRegistry()
    reg.register("alpha", "base")
    reg.register("alpha/opt", "fast")
    reg.register("beta", "beta-base")
    assert reg.resolve("alpha") == "base"
    assert reg.resolve("alpha", "opt") == "fast"
    assert reg.resolve("beta", "opt") == "beta-base"
    assert reg.resolve("alpha/opt", "opt") == "fast"
    assert "alpha" in reg and "gamma" not in reg
    assert reg.names() == ["alpha", "alpha/opt", "beta"]


def test_registry_errors():
    reg = StyleRegistry()
    reg.register("alpha", object())
    with pytest.raises(RegistryError, match="already registered"):
        reg.register("alpha", object())
    with pytest.raises(RegistryError) as exc:
        reg.resolve("alpah")
    assert "unknown style" in str(exc.value) and "alpha" in str(exc.value)


def test_default_registry_styles():
    reg = default_registry()
    assert set(reg.names()) >= {"lj/cut", "lj/cut/opt", "lj/cut/kk", "snap", "snap/opt", "snap/kk"}
    base = reg.resolve("lj/cut")(["1.5"])
    assert base.name == "lj/cut" and base.default_mode == "atom"
    opt = reg.resolve("lj/cut", "opt")(["1.5"])
    assert opt.name == "lj/cut/opt" and opt.default_mode == "neighbor"


def test_lattice_positions_fcc_and_sc():
    pos, box = lattice_positions("fcc", 0.8, (2, 3, 4))
    assert pos.shape == (4 * 24, 3)
    assert len(pos) / box.volume == pytest.approx(0.8, rel=1e-12)
    pos, box = lattice_positions("sc", 0.5, (3, 3, 3))
    assert pos.shape == (27, 3) and len(pos) / box.volume == pytest.approx(0.5, rel=1e-12)
    with pytest.raises(RunError):
        lattice_positions("hcp", 0.8, (2, 2, 2))


def test_seeded_velocities_momentum_and_temperature():
    v = seeded_velocities(50, 0.75, 2.0, seed=99)
    assert np.abs(v.mean(axis=0)).max() < 1e-13
    assert 2.0 * float(np.sum(v * v)) / (3.0 * 50) == pytest.approx(0.75, rel=1e-12)
    assert np.array_equal(v, seeded_velocities(50, 0.75, 2.0, seed=99))
    assert not np.allclose(v, seeded_velocities(50, 0.75, 2.0, seed=100))
    assert np.array_equal(seeded_velocities(10, 0.0, 1.0, 1), np.zeros((10, 3)))
    with pytest.raises(RunError):
        seeded_velocities(10, -0.5, 1.0, 1)


# ------------------------------------------------------------------ GPU part
@pytest.mark.gpu
def test_minimal_run_and_zero_steps(gpu):
    sim = run_script(MINI, RunConfig(), log=SILENT)
    res = sim.results[-1]
    assert [r[0] for r in res.rows] == [0, 10, 20]
    e0 = res.rows[0][3]
    assert abs(res.rows[-1][3] - e0) < 1e-3 * abs(e0)
    rows = run_script(MINI.replace("run 20", "run 0"), log=SILENT).results[-1].rows
    assert len(rows) == 1 and rows[0][0] == 0


@pytest.mark.gpu
def test_rank_count_does_not_change_physics(gpu):
    base = run_script(MINI, RunConfig(n_ranks=1), log=SILENT).results[-1]
    for n_ranks in (2, 4):
        other = run_script(MINI, RunConfig(n_ranks=n_ranks), log=SILENT).results[-1]
        for (s0, *r0), (s1, *r1) in zip(base.rows, other.rows):
            assert s0 == s1 and np.allclose(r0, r1, rtol=1e-12, atol=1e-12)
        for step, snap in base.snapshots.items():
            assert np.allclose(other.snapshots[step], snap, rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_same_config_is_exactly_reproducible_and_seed_override(gpu):
    a = run_script(MINI, RunConfig(n_ranks=2), log=SILENT)
    b = run_script(MINI, RunConfig(n_ranks=2), log=SILENT)
    assert a.results[-1].lines == b.results[-1].lines     # full lists: owner writes, fixed orders
    c = run_script(MINI, RunConfig(rng_seed=777), log=SILENT)
    assert not np.allclose(a._velocities, c._velocities)
    assert a.results[-1].rows[0][1] == pytest.approx(c.results[-1].rows[0][1], rel=1e-12)


@pytest.mark.gpu
def test_suffix_switches_style_variant(gpu):
    text = MINI.replace("pair_style lj/cut 1.5", "suffix opt\npair_style lj/cut 1.5")
    assert run_script(text, log=SILENT).style.name == "lj/cut/opt"
    off = MINI.replace("pair_style lj/cut 1.5", "suffix opt\nsuffix off\npair_style lj/cut 1.5")
    assert run_script(off, log=SILENT).style.name == "lj/cut"


@pytest.mark.gpu
def test_run_errors(gpu, tmp_path):
    with pytest.raises(RunError, match="lattice must be set"):
        run_script("units lj\ncreate_box 2 2 2\n", log=SILENT)
    with pytest.raises(RunError, match="create_atoms must run"):
        run_script("velocity 0.1 1\n", log=SILENT)
    with pytest.raises(RunError, match="pair_style must be set"):
        run_script("pair_coeff 1.0 1.0\n", log=SILENT)
    with pytest.raises(RunError, match="timestep must be positive"):
        run_script("timestep -0.1\n", log=SILENT)
    with pytest.raises(RegistryError, match="unknown style"):
        run_script("pair_style bogus 1.0\n", log=SILENT)
    coeff = tmp_path / "j1.coeff"
    coeff.write_text("1.0\n" + "\n".join(["0.1"] * 5) + "\n")
    snap = MINI.replace("pair_style lj/cut 1.5\npair_coeff 1.0 1.0", f"pair_style snap 1.6 {coeff}")
    with pytest.raises(RunError, match="requires full lists"):
        run_script(snap, RunConfig(list_style="half"), log=SILENT)
    with pytest.raises(RunError, match="pair_coeff does not apply"):
        run_script(MINI.replace("pair_style lj/cut 1.5", f"pair_style snap 1.6 {coeff}"), log=SILENT)


# ------------------------------------------ more of mdkk tests/test_driver.py
def test_parse_unknown_command_suggests_near_match():
    with pytest.raises(ParseError) as exc:
        parse_script("units lj\npair_stylee lj/cut 1.5\n")
    assert exc.value.line_no == 2
    assert "did you mean" in str(exc.value) and "pair_style" in str(exc.value)


def test_parse_arity_and_number_validation():
    with pytest.raises(ParseError, match="expects 2"):
        parse_script("velocity 0.1\n")
    with pytest.raises(ParseError, match="malformed number"):
        parse_script("timestep fast\n")
    with pytest.raises(ParseError, match="malformed integer"):
        parse_script("run 1.5\n")
    with pytest.raises(ParseError, match="expected one of"):
        parse_script("lattice bct 0.8\n")   # (bcc is accepted here: the SNAP tungsten lattice)
    with pytest.raises(ParseError, match="expected one of"):
        parse_script("boundary p p f\n")
    with pytest.raises(ParseError, match="expected one of"):
        parse_script("units si\n")


def test_parse_onoff_and_pair_style_shapes():
    assert parse_script("qeq off\n")[0].args == ["off"]
    with pytest.raises(ParseError, match="off takes no parameters"):
        parse_script("qeq off 1.0\n")
    with pytest.raises(ParseError, match="expects 4 parameter"):
        parse_script("qeq on 0.8 15.0 -0.3\n")
    assert parse_script("pair_style snap 1.6 w.coeff\n")[0].args[0] == "snap"
    with pytest.raises(ParseError, match="cutoff coeff_file"):
        parse_script("pair_style snap 1.6\n")
    with pytest.raises(ParseError, match="expects: cutoff"):
        parse_script("pair_style lj/cut 1.5 extra\n")
    with pytest.raises(ParseError, match="style name"):
        parse_script("pair_style\n")


def test_run_command_ordering_errors():
    """Raised before any device work (mdkk tests/test_driver.py:326-338)."""
    CPU = RunConfig(device="cpu")
    with pytest.raises(RunError, match="lattice must be set"):
        run_script("units lj\ncreate_box 2 2 2\n", CPU, log=SILENT)
    with pytest.raises(RunError, match="create_atoms must run"):
        run_script("velocity 0.1 1\n", CPU, log=SILENT)
    with pytest.raises(RunError, match="pair_style must be set"):
        run_script("pair_coeff 1.0 1.0\n", CPU, log=SILENT)
    with pytest.raises(RunError, match="timestep must be positive"):
        run_script("timestep -0.1\n", CPU, log=SILENT)
    with pytest.raises(RegistryError, match="unknown style"):
        run_script("pair_style bogus 1.0\n", CPU, log=SILENT)


def _coeff(tmp_path):
    from paper_2508_13523_b200.snap import QuantumIndex
    p = tmp_path / "snap_jmax1.coeff"
    p.write_text("1\n" + "\n".join(["0.1"] * len(QuantumIndex(1).triples())) + "\n")
    return str(p)


@pytest.mark.gpu
def test_more_run_errors_and_list_style_conflict(gpu, tmp_path):
    coeff = _coeff(tmp_path)
    with pytest.raises(RunError, match="pair_style must be set"):
        run_script(MINI.replace("pair_style lj/cut 1.5\n", "").replace("pair_coeff 1.0 1.0\n", ""), log=SILENT)
    with pytest.raises(RunError, match="pair_coeff does not apply"):
        run_script(MINI.replace("pair_style lj/cut 1.5", f"pair_style snap 1.6 {coeff}"), log=SILENT)
    with pytest.raises(RunError, match="requires full lists"):
        run_script(MINI.replace("pair_style lj/cut 1.5\npair_coeff 1.0 1.0", f"pair_style snap 1.6 {coeff}"),
                   RunConfig(list_style="half"), log=SILENT)


@pytest.mark.gpu
def test_strategy_and_mode_agree_through_driver(gpu):
    base = run_script(MINI, RunConfig(), log=SILENT).results[-1]
    for config in (RunConfig(strategy="duplicate", mode="neighbor", workers=3),
                   RunConfig(strategy="atomic", mode="neighbor", workers=2),
                   RunConfig(list_style="full", newton=False)):
        other = run_script(MINI, config, log=SILENT).results[-1]
        for (s0, *r0), (s1, *r1) in zip(base.rows, other.rows):
            assert s0 == s1 and np.allclose(r0, r1, rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_snap_script_runs_with_suffix(gpu, tmp_path):
    """A SNAP input through the driver, `suffix kk` resolving snap/kk (mdkk tests/test_driver.py:302-310)."""
    coeff = _coeff(tmp_path)
    text = (f"units lj\nboundary p p p\nlattice fcc 0.8\ncreate_box 3 3 3\ncreate_atoms\nmass 1.0\n"
            f"velocity 0.05 7\nsuffix kk\npair_style snap 1.6 {coeff}\ntimestep 0.002\nthermo 5\nrun 10\n")
    sim = run_script(text, log=SILENT)
    assert sim.style.name == "snap/kk"
    rows = np.array(sim.results[-1].rows)
    assert rows.shape[0] == 3 and np.isfinite(rows).all()
