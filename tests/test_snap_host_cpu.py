"""Host-side SNAP setup (indexing, Clebsch-Gordan, coefficient files) on CPU.

Mirrors mdkk tests/test_snap.py:125-245 and :534-565 against this package's own
host code (the oracle's copies are pinned in tests/test_oracle.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_2508_13523_b200.snap import (QuantumIndex, SnapError, SnapIndexError, clebsch_gordan,
                                        make_coupling_tables, read_coeff_file)


def test_quantum_index_counts():
    assert QuantumIndex(0).n_flat == 1
    assert QuantumIndex(0.5).n_flat == 5
    assert QuantumIndex(1).n_flat == 14
    assert QuantumIndex(4).n_flat == 285
    assert [len(QuantumIndex(j).triples()) for j in (0.5, 1, 2, 4)] == [2, 5, 14, 55]


def test_quantum_index_flat_roundtrip_and_blocks():
    qi = QuantumIndex(2)
    seen = []
    for tj in range(qi.twojmax + 1):
        blk = qi.block(tj)
        assert blk.stop - blk.start == (tj + 1) ** 2
        for p in range(tj + 1):
            for q in range(tj + 1):
                idx = qi.flat(tj, p, q)
                assert blk.start <= idx < blk.stop and qi.unflatten(idx) == (tj, p, q)
                seen.append(idx)
    assert sorted(seen) == list(range(qi.n_flat))


def test_quantum_index_triple_order_and_validation():
    qi = QuantumIndex(4)
    triples = qi.triples()
    assert triples == sorted(triples) and triples[:3] == [(0, 0, 0), (1, 1, 0), (2, 1, 1)]
    for tj, tj1, tj2 in triples:
        assert 0 <= tj2 <= tj1 <= tj <= qi.twojmax and tj <= tj1 + tj2 and (tj1 + tj2 - tj) % 2 == 0
    for bad in (0.3, -1):
        with pytest.raises(SnapIndexError):
            QuantumIndex(bad)
    q1 = QuantumIndex(1)
    for call in (lambda: q1.flat(3, 0, 0), lambda: q1.flat(1, 2, 0), lambda: q1.unflatten(q1.n_flat)):
        with pytest.raises(SnapIndexError):
            call()


def test_clebsch_gordan_frozen_values_and_orthogonality():
    assert clebsch_gordan(1, 1, 1, 1, 2, 2) == pytest.approx(1.0, abs=1e-15)
    assert clebsch_gordan(4, 4, 2, 2, 6, 6) == pytest.approx(1.0, abs=1e-15)
    assert clebsch_gordan(1, 1, 1, -1, 0, 0) == pytest.approx(np.sqrt(0.5), rel=1e-15)
    assert clebsch_gordan(1, -1, 1, 1, 0, 0) == pytest.approx(-np.sqrt(0.5), rel=1e-15)
    assert clebsch_gordan(1, 1, 1, -1, 2, 0) == pytest.approx(np.sqrt(0.5), rel=1e-15)
    assert clebsch_gordan(2, 2, 2, -2, 0, 0) == pytest.approx(1 / np.sqrt(3), rel=1e-15)
    assert clebsch_gordan(2, 2, 2, -2, 4, 0) == pytest.approx(1 / np.sqrt(6), rel=1e-15)
    assert clebsch_gordan(2, 2, 2, -2, 2, 0) == pytest.approx(1 / np.sqrt(2), rel=1e-15)
    assert clebsch_gordan(1, 1, 1, 1, 2, 0) == 0.0
    assert clebsch_gordan(1, 1, 1, 1, 4, 2) == 0.0
    assert clebsch_gordan(2, 0, 2, 0, 3, 0) == 0.0
    for tj1, tj2 in [(1, 1), (2, 1), (2, 2), (3, 2)]:
        jays = list(range(abs(tj1 - tj2), tj1 + tj2 + 1, 2))
        for tj in jays:
            for tjp in jays:
                for tm in range(-min(tj, tjp), min(tj, tjp) + 1, 2):
                    acc = sum(clebsch_gordan(tj1, tm1, tj2, tm - tm1, tj, tm)
                              * clebsch_gordan(tj1, tm1, tj2, tm - tm1, tjp, tm)
                              for tm1 in range(-tj1, tj1 + 1, 2) if abs(tm - tm1) <= tj2)
                    assert acc == pytest.approx(1.0 if tj == tjp else 0.0, abs=1e-13)


def test_coupling_tables_term_counts():
    assert len(make_coupling_tables(4).triples) == 55
    assert sum(len(t[3]) for t in make_coupling_tables(4).terms) == 32578


def test_coeff_file_parsing_and_errors(tmp_path):
    good = tmp_path / "good.coeff"
    good.write_text("# header comment\n1   # jmax\n0.1 0.2  # two on one line\n-0.3\n\n0.4 0.5\n")
    jmax, beta = read_coeff_file(good)
    assert jmax == 1.0 and np.array_equal(beta, [0.1, 0.2, -0.3, 0.4, 0.5])
    half = tmp_path / "half.coeff"
    half.write_text("0.5 1.0 2.0\n")
    jmax, beta = read_coeff_file(half)
    assert jmax == 0.5 and np.array_equal(beta, [1.0, 2.0])
    for name, text in (("empty", "# nothing but comments\n\n"), ("short", "1 0.1 0.2\n"),
                       ("bad", "1 0.1 0.2 x 0.4 0.5\n")):
        p = tmp_path / f"{name}.coeff"
        p.write_text(text)
        with pytest.raises(SnapError):
            read_coeff_file(p)


def test_run_config_knobs_override_style_knobs():
    """mdkk/driver/simulation.py:115-121: RunConfig batch_u / batch_y / tile_v / layout win over the style's."""
    from paper_2508_13523_b200.driver import RunConfig
    from paper_2508_13523_b200.snap.style import SnapStyle
    st = SnapStyle(4.73, 1, np.zeros(5), batch_u=8, tile_v=256)
    assert st._knobs(RunConfig()) == {"batch_u": 8, "batch_y": 2, "tile_v": 256, "layout": "a"}
    assert st._knobs(RunConfig(batch_u=2, batch_y=3, layout="b")) == {"batch_u": 2, "batch_y": 3, "tile_v": 256,
                                                                      "layout": "b"}
