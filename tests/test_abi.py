"""CPU-side checks of the C-ABI library (no device calls): it loads, exports every symbol the
header declares, and its host-side model layer (parser, validation, description) matches the
reference's behaviour."""
import ctypes as C
import os
import re

import pytest

from paper_1909_09213_b200 import _abi as A
from paper_1909_09213_b200 import models
from paper_1909_09213_b200 import solver as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "cubics.h")).read()
    declared = set(re.findall(r"\b(cubics_[a-z_]+)\s*\(", header)) - {"cubics_solution_cb", "cubics_keyed_solution_cb"}
    assert declared == set(A.EXPORTED)
    lib = S.lib()
    for name in declared:
        assert hasattr(lib, name), name


def test_config_init_matches_reference_defaults():
    c = A.SearchConfig()
    S.lib().cubics_search_config_init(C.byref(c))
    # fd::SearchConfig defaults (search.hpp:19-27)
    assert (c.var_heuristic, c.value_heuristic, c.max_solutions, c.thread_count, c.seed, c.alldiff,
            c.node_limit) == (A.FIRST_FAIL, 0, A.UINT64_MAX, 1, 0, A.ARC_CONSISTENT, 0)
    assert (c.engine, c.device, c.count_only) == (A.ENGINE_AUTO, -1, 0)


def test_build_info_and_no_cpu_fallback():
    assert "sm_100a" in S.build_info()


def test_parser_builds_reference_model_shapes():
    m = S.parse_model(models.gen_nqueens(4))
    assert (m.n_vars, m.n_cons) == (4, 13)
    assert m.con_kind == [A.ALLDIFF] + [A.RELBIN] * 12
    assert m.term_var[:4] == [0, 1, 2, 3]
    assert m.con_value[1:5] == [1, -1, 2, -2]
    # x > y + k normalises to y < x - k between variables (parser.cpp:380-385); literals keep >
    m = S.parse_model("var x in 1..5; var y in 1..5; constraint x > y + 2; constraint x >= 3; solve satisfy;")
    assert m.con_op == [A.LT, A.GE]
    assert m.term_var[:2] == [1, 0] and m.con_value[0] == -2
    m = S.parse_model("var a in 0..3; var b in 0..3; constraint 2*a - b + 3*a <= 7; solve maximize b;")
    assert m.con_kind == [A.LINEAR] and m.term_coeff == [2, -1, 3] and m.con_value == [7]
    assert (m.goal, m.goal_var) == (A.MAXIMIZE, 1)


@pytest.mark.parametrize("text,kind,line,col", [
    ("var x in 1..3;\nvar x in 1..2;\nsolve satisfy;", 2, 2, 5),
    ("var x in 3..1;\nsolve satisfy;", 3, 1, 10),
    ("var x in 0..1024;\nsolve satisfy;", 4, 1, 10),
    ("var x in 1..3;\nconstraint y < 2;\nsolve satisfy;", 1, 2, 12),
    ("var x in 1..3;\n", 5, 2, 1),
    ("var x in 1..3; constraint x == 2; solve satisfy;", 0, 1, 30),
    ("var x in 1..3; constraint 2 x <= 2; solve satisfy;", 0, 1, 29),
])
def test_parse_errors_like_reference(text, kind, line, col):
    with pytest.raises(ValueError) as ei:
        S.parse_model(text)
    assert (ei.value.kind, ei.value.line, ei.value.column) == (kind, line, col)


def test_model_validate_diagnostics():
    # model.cpp:39-80 : zero coefficient, alldifferent too small / duplicate member
    m = S.parse_model("var a in 1..3; var b in 1..3; constraint 0*a + b <= 2; solve satisfy;")
    assert m.validate() == [(5, 0)]
    arr = S.build_desc([1, 1], [3, 3], [S.Domain(1, 3), S.Domain(1, 3)], [A.ALLDIFF], [0], [0], [0, 2], [0, 0], [1, 1])
    m2 = S.model_from_desc(arr["desc"])
    assert sorted(m2.validate()) == [(6, 0), (7, 0)]


def test_desc_roundtrip_preserves_domains_with_holes():
    m = S.parse_model("var a in -3..70; var b in 5..5; solve satisfy;")
    d = [m.domains[0].copy(), m.domains[1].copy()]
    for v in (-3, 0, 64, 70):
        d[0].remove(v)
    m2 = m.with_domains(d)
    assert m2.domains[0].values() == d[0].values() and m2.domains[1].values() == [5]
