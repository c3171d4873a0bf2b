"""Grid-wide root fixpoints (cubics_propagate / cubics_removals on models with many
alldifferents): the reference's bench_propagation instances (tools/bench_propagation.cpp:71-74)
and smaller random models, against the oracle's propagate_fixpoint / propagate_round / run_batch."""
import pytest

from paper_1909_09213_b200 import _abi as A
from paper_1909_09213_b200 import models
from paper_1909_09213_b200 import solver as S

import oracle_binding as O

pytestmark = pytest.mark.gpu

CASES = [(200, 48, 400, 7), (400, 64, 800, 11), (120, 30, 300, 3), (60, 12, 200, 5), (300, 40, 150, 9)]


def _bits(doms):
    return [(d.offset, d.width, d.bits) for d in doms]


@pytest.mark.parametrize("vars_,width,cons,seed", CASES)
@pytest.mark.parametrize("alldiff", [A.ARC_CONSISTENT, A.FORWARD_CHECKING])
def test_grid_fixpoint_matches_oracle(vars_, width, cons, seed, alldiff):
    m = S.parse_model(models.gen_random(vars_, width, cons, seed))
    got_d, got = S.propagate_fixpoint(m, alldiff=alldiff)
    ref_d, ref = O.propagate_fixpoint(m, alldiff=alldiff)
    assert (got.failed, got.failed_var, got.rounds, got.last_status) == \
        (ref.failed, ref.failed_var, ref.rounds, ref.last_status)
    if not ref.failed:
        assert _bits(got_d) == _bits(ref_d)


@pytest.mark.parametrize("vars_,width,cons,seed", CASES[:3])
def test_grid_round_and_removals_match_oracle(vars_, width, cons, seed):
    m = S.parse_model(models.gen_random(vars_, width, cons, seed))
    got_d, got = S.propagate_fixpoint(m, max_rounds=1)
    ref_d, ref = O.propagate_fixpoint(m, max_rounds=1)
    assert (got.failed, got.failed_var, got.rounds) == (ref.failed, ref.failed_var, ref.rounds)
    if not ref.failed:
        assert _bits(got_d) == _bits(ref_d)
    subset = list(range(0, m.n_cons, 3))
    assert S.removals(m, cons=subset) == O.removals(m, cons=subset)
    assert S.removals(m) == O.removals(m)
