"""MPS ingestion and reports (the reference's declared inc/hplp/mps_io.hpp,
SPEC.md [MODULE] mps_io): host-side, no GPU.  Fixtures are written here by
hand; round trips go through the product's own writer."""
from __future__ import annotations

import json
import math

import numpy as np
import pytest

from paper_2407_16144_b200 import abi, gen, hplp
from paper_2407_16144_b200.hplp import MpsParseError

TINY = """NAME          TINY
ROWS
 N  COST
 L  LIM1
 E  MYEQN
COLUMNS
    X1        COST         1.0   LIM1         1.0
    X1        MYEQN       -1.0
    X2        COST         2.0   LIM1         1.0
RHS
    RHS       LIM1         4.0   MYEQN        1.0
ENDATA
"""


def test_two_row_fixture():
    # SPEC.md mps_io example: one L row, one E row, RHS on both
    p = hplp.parse_mps(TINY)
    g = p.general()
    assert (p.m, p.n, p.nnz) == (2, 2, 3)
    assert p.name == "TINY" and p.objective_name == "COST"
    assert p.row_names == ["LIM1", "MYEQN"] and p.col_names == ["X1", "X2"]
    assert list(g.row_relation) == [abi.ROW_LE, abi.ROW_EQ]
    assert list(g.row_rhs) == [4.0, 1.0]
    assert list(g.objective) == [1.0, 2.0]
    assert list(g.row_ptr) == [0, 2, 3] and list(g.col_idx) == [0, 1, 0] and list(g.val) == [1.0, 1.0, -1.0]
    assert list(g.col_lower) == [0.0, 0.0] and list(g.col_upper) == [math.inf, math.inf]
    assert not g.maximize and g.objective_constant == 0.0 and np.isnan(g.row_range).all()


@pytest.mark.parametrize("text,line,needle", [
    (TINY.replace("COLUMNS", "COLUMNZ"), 6, "unknown section 'COLUMNZ'"),
    (TINY.replace("MYEQN       -1.0", "NOPE        -1.0"), 8, "undeclared row 'NOPE'"),
    (TINY.replace("X2        COST         2.0   LIM1         1.0", "X2        COST         2.0   LIM1         1.0x"),
     9, "malformed number"),
    (TINY.replace("    X1        MYEQN       -1.0", "    X1        LIM1        -1.0"), 8, "duplicate entry"),
    (TINY.replace("ENDATA\n", ""), 12, "missing ENDATA"),
    (TINY.replace(" E  MYEQN", " Q  MYEQN"), 5, "unknown row type"),
    (TINY.replace("ENDATA", "BOUNDS\n UP BND X9 1\nENDATA"), 13, "undeclared column 'X9'"),
    (TINY.replace("ENDATA", "BOUNDS\n XX BND X1 1\nENDATA"), 13, "unknown bound type"),
])
def test_parse_errors_carry_line_numbers(text, line, needle):
    with pytest.raises(MpsParseError) as e:
        hplp.parse_mps(text)
    assert e.value.line == line, str(e.value)
    assert needle in str(e.value)


def test_extra_objective_rows_dropped_with_warning():
    t = TINY.replace(" L  LIM1", " N  OTHER\n L  LIM1").replace("    X2        COST         2.0",
                                                               "    X2        OTHER        5.0\n    X2        COST         2.0")
    p = hplp.parse_mps(t)
    assert p.objective_name == "COST" and p.m == 2
    assert any("OTHER" in w for w in p.warnings)
    assert list(p.general().objective) == [1.0, 2.0]


def test_empty_columns_section():
    # SPEC.md: empty COLUMNS -> zero matrix
    p = hplp.parse_mps("NAME E\nROWS\n N obj\n E r\nCOLUMNS\nRHS\n    RHS r 0\nENDATA\n")
    assert (p.m, p.n, p.nnz) == (1, 0, 0)


def test_bound_types_objsense_constant_ranges_markers():
    t = """NAME B
OBJSENSE
    MAX
ROWS
 N obj
 L a
 G b
 E c
 E d
COLUMNS
    MARKER 'MARKER' 'INTORG'
    i1 obj 1 a 1
    MARKER 'MARKER' 'INTEND'
    u obj 1 b 1
    l obj 1 c 1
    f obj 1 d 1
    m obj 1 a 2
    p obj 1 b 2
    bv obj 1 c 2
    neg obj 1 d 2
RHS
    RHS obj 7.5 a 10
    RHS b 1 c 2
    RHS d 3
RANGES
    RNG a 4 b 5
    RNG c -2 d 2
BOUNDS
 UP BND u 3
 LO BND l -2
 FX BND f 1.25
 MI BND m
 UP BND m 9
 FR BND p
 BV BND bv
 UP BND neg -1
ENDATA
"""
    p = hplp.parse_mps(t)
    g = p.general()
    assert g.maximize and g.objective_constant == -7.5
    lo = dict(zip(p.col_names, g.col_lower))
    up = dict(zip(p.col_names, g.col_upper))
    assert (lo["i1"], up["i1"]) == (0.0, math.inf)
    assert (lo["u"], up["u"]) == (0.0, 3.0)
    assert (lo["l"], up["l"]) == (-2.0, math.inf)
    assert (lo["f"], up["f"]) == (1.25, 1.25)
    assert (lo["m"], up["m"]) == (-math.inf, 9.0)
    assert (lo["p"], up["p"]) == (-math.inf, math.inf)
    assert (lo["bv"], up["bv"]) == (0.0, 1.0)
    assert (lo["neg"], up["neg"]) == (-math.inf, -1.0)  # UP < 0 with no lower bound
    assert list(g.row_range) == [4.0, 5.0, -2.0, 2.0]
    assert any("integrality relaxed" in w for w in p.warnings)
    assert any("UP bound < 0" in w for w in p.warnings)
    # RANGES semantics through to_standard_form (src/lp_model.cpp:139-151):
    # L [rhs-|r|, rhs], G [rhs, rhs+|r|], E r<0 [rhs+r, rhs], E r>0 [rhs, rhs+r]
    # -> every ranged row gets a bounded slack: 4 rows + 4 bound rows after the
    #    column bounds' rows
    s = hplp.to_standard_form(g)
    assert s.m >= 4
    # the idempotent normalization of the writer
    p2 = hplp.parse_mps(p.write())
    _same_general(p.general(), p2.general())
    assert p2.write() == p.write()


def test_fixed_format_names_with_spaces():
    # fixed columns 5-12 / 15-22 / 25-36: a name with a space needs them
    def fixed(f1="", f2="", f3="", f4="", f5="", f6=""):  # 1-based columns 2, 5, 15, 25, 40, 50
        line = [" "] * 61
        for start, text in ((2, f1), (5, f2), (15, f3), (25, f4), (40, f5), (50, f6)):
            line[start - 1:start - 1 + len(text)] = list(text)
        return "".join(line).rstrip() + "\n"

    t = ("NAME          FIX\nROWS\n" + fixed("N", "COST") + fixed("E", "ROW A") + "COLUMNS\n"
         + fixed("", "COL 1", "COST", "1.0", "ROW A", "2.0") + "RHS\n" + fixed("", "RHS", "ROW A", "4.0") + "ENDATA\n")
    p = hplp.parse_mps(t)
    g = p.general()
    assert p.row_names == ["ROW A"] and p.col_names == ["COL 1"]
    assert list(g.val) == [2.0] and list(g.row_rhs) == [4.0]


def _same_general(a, b):
    assert (a.m, a.n) == (b.m, b.n)
    for f in ("row_ptr", "col_idx", "val", "row_relation", "row_rhs", "col_lower", "col_upper", "objective"):
        x, y = getattr(a, f), getattr(b, f)
        assert np.array_equal(x, y), f
    ra = np.nan_to_num(a.row_range, nan=1.5e300) if a.row_range is not None else np.full(a.m, 1.5e300)
    rb = np.nan_to_num(b.row_range, nan=1.5e300) if b.row_range is not None else np.full(b.m, 1.5e300)
    assert np.array_equal(ra, rb)
    assert a.maximize == b.maximize and a.objective_constant == b.objective_constant


@pytest.mark.parametrize("cfg", [0, "transport"])
def test_generated_lp_round_trip_bit_exact(cfg):
    g = gen.generate(0) if cfg == 0 else gen.generate(gen.scaled(3, sources=20, sinks=30))
    text = hplp.mps_from_general(g)
    p = hplp.parse_mps(text)
    back = p.general()
    _same_general(g, back)  # 17 significant digits: every double survives
    assert hplp.parse_mps(p.write()).write() == p.write()
    # the standard forms agree bit for bit
    s1, s2 = hplp.to_standard_form(g), hplp.to_standard_form(back)
    for f in ("row_ptr", "col_idx", "val", "b", "c"):
        assert np.array_equal(getattr(s1, f), getattr(s2, f)), f


REPORT = {
    "instance": "t", "status": "optimal", "primal_objective": 0.1 + 0.2, "dual_objective": None,
    "kkt": {"primal": 1e-300, "dual": 5e-324, "gap": 2.0 / 3.0, "max": "inf"},
    "iterations": 12, "epochs": 3, "spmv_count": 40, "eta": 0.123456789012345678, "sigma_estimate": 4.0,
    "primal_solution": [1.0 / 3.0, -0.0, 1e308], "dual_solution": {"elided": True, "length": 7},
    "primal_certificate": None,
    "dual_certificate": {"source": "normalized_iterate", "orientation": "negated", "at_iteration": 9,
                         "residual": 1e-7, "margin": -2.5, "vector": [0.6, 0.8]},
    "config": [["tolerance", "1e-8"]], "timing": {"solve_seconds": 0.25},
}


def test_solution_json_round_trip_bit_identical():
    text = json.dumps(REPORT)
    once = hplp.json_normalize(text)
    twice = hplp.json_normalize(once)
    assert once == twice  # deterministic key order, 17 digits
    d = json.loads(once)
    assert d["primal_objective"] == 0.1 + 0.2 and d["eta"] == REPORT["eta"]
    assert d["kkt"]["max"] == "inf" and d["dual_objective"] is None
    assert d["primal_solution"] == [1.0 / 3.0, -0.0, 1e308]
    assert d["dual_solution"] is None  # elided vectors parse to "absent"
    assert d["dual_certificate"]["vector"] == [0.6, 0.8] and d["dual_certificate"]["orientation"] == "negated"
    assert list(d)[:3] == ["instance", "status", "primal_objective"]
    no_t = json.loads(hplp.json_normalize(text, include_timing=False))
    assert "timing" not in no_t


def test_solution_json_rejects_unknown_status():
    with pytest.raises(ValueError):
        hplp.json_normalize(json.dumps(dict(REPORT, status="solved")))


# ---- fixture corpus (SPEC.md acceptance criterion 10) -----------------------
from pathlib import Path  # noqa: E402

CORPUS = Path(__file__).resolve().parent / "golden" / "mps"
GOOD = sorted(p for p in CORPUS.glob("[0-9]*.mps"))
BAD = {  # file: (line, message fragment)
    "bad_01_unknown_section.mps": (5, "unknown section 'COLUMNZ'"),
    "bad_02_undeclared_row.mps": (6, "undeclared row 'Q'"),
    "bad_03_duplicate_entry.mps": (7, "duplicate entry (R, X)"),
    "bad_04_malformed_number.mps": (8, "malformed number '1.2.3'"),
    "bad_05_unknown_bound.mps": (8, "unknown bound type 'XX'"),
    "bad_06_missing_endata.mps": (7, "missing ENDATA"),
}


def test_corpus_size():
    assert len(GOOD) >= 12 and len(BAD) >= 6


@pytest.mark.parametrize("path", GOOD, ids=lambda p: p.name)
def test_corpus_round_trip(path):
    """Every fixture parses; write -> parse reproduces it exactly, and the
    normalized text is a fixed point."""
    p = hplp.parse_mps(path.read_text())
    g = p.general()
    q = hplp.parse_mps(p.write())
    _same_general(g, q.general())
    assert q.row_names == p.row_names and q.col_names == p.col_names
    assert q.write() == p.write()
    if p.n:  # through to_standard_form as well
        s1, s2 = hplp.to_standard_form(g), hplp.to_standard_form(q.general())
        assert np.array_equal(s1.val, s2.val) and np.array_equal(s1.b, s2.b) and np.array_equal(s1.c, s2.c)


@pytest.mark.parametrize("name", sorted(BAD))
def test_corpus_corrupted(name):
    line, needle = BAD[name]
    with pytest.raises(MpsParseError) as e:
        hplp.parse_mps((CORPUS / name).read_text())
    assert e.value.line == line and needle in str(e.value), str(e.value)


def test_corpus_semantics():
    g = hplp.parse_mps((CORPUS / "04_all_bound_types.mps").read_text())
    lo = dict(zip(g.col_names, g.general().col_lower))
    up = dict(zip(g.col_names, g.general().col_upper))
    assert (lo["LIV"], up["LIV"]) == (1.0, math.inf) and (lo["UIV"], up["UIV"]) == (0.0, 9.0)
    assert (lo["PLV"], up["PLV"]) == (0.0, math.inf) and (lo["FRV"], up["FRV"]) == (-math.inf, math.inf)
    m = hplp.parse_mps((CORPUS / "05_objsense_max_constant.mps").read_text()).general()
    assert m.maximize and m.objective_constant == 12.5
    e = hplp.parse_mps((CORPUS / "12_rhs_without_set_name.mps").read_text()).general()
    assert list(e.row_rhs) == [2.0, 3.0] and e.row_range[0] == 1.0 and np.isnan(e.row_range[1])
    w = hplp.parse_mps((CORPUS / "09_extra_objective_rows.mps").read_text())
    assert w.objective_name == "FIRST" and any("SECOND" in x for x in w.warnings)
    assert list(w.general().objective) == [1.0, 0.0]
