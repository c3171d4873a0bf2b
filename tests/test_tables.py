"""Positive table constraints (extension for BASELINE config 5; no reference counterpart):
grammar, model description and the oracle's propagator against brute force. CPU only."""
import itertools

import oracle_binding as O
from paper_1909_09213_b200 import _abi as A
from paper_1909_09213_b200 import models
from paper_1909_09213_b200 import solver as S


def test_table_grammar_and_description():
    m = S.parse_model("var x in 1..3; var y in 0..2; var z in 1..2;\n"
                      "constraint table(x, y : 1 0, 2 2, 3 -1);\n"
                      "constraint table(x, y, z : 1 0 1, 3 2 2);\n"
                      "constraint table < 3;\nsolve satisfy;".replace("table <", "x <"))
    assert m.con_kind == [A.TABLE, A.TABLE, A.RELBIN]
    assert m.con_value[:2] == [3, 2]
    assert m.table_data[:6] == [1, 0, 2, 2, 3, -1]
    assert m.table_data[6:12] == [1, 0, 1, 3, 2, 2]


def test_reference_models_with_a_var_named_table_still_parse():
    m = S.parse_model("var table in 1..3; constraint table < 3; solve satisfy;")
    assert m.con_kind == [A.RELBIN]


def test_oracle_tables_vs_brute_force():
    for seed in range(40):
        n, d = 4 + seed % 3, 3
        m = S.parse_model(models.random_binary_csp(n, d, n + seed % 3, 0.5, seed))
        tabs = []
        for c in range(m.n_cons):
            vs = m.term_var[m.con_start[c]:m.con_start[c + 1]]
            tu = {tuple(m.table_data[m.table_start[c] + 2 * i:m.table_start[c] + 2 * i + 2]) for i in range(m.con_value[c])}
            tabs.append((vs, tu))
        bf = sorted(list(a) for a in itertools.product(range(1, d + 1), repeat=n)
                    if all(tuple(a[v] for v in vs) in tu for vs, tu in tabs))
        assert sorted(s.values for s in O.enumerate_solutions(m)) == bf, seed


def test_phase_transition_formula():
    assert abs(models.phase_transition_tightness(1000, 10, 2000) - (1 - 10 ** -0.5)) < 1e-12
