"""The instance generators match the reference's own generators byte for byte.

Fixture: tests/golden/generators.json, the sha256 of every text the unmodified reference
generator emitted (tests/golden/make_generator_fixtures.py over oracle/_ref/fdref_driver):
fd::gen_nqueens (generators.cpp:13-33), fd::gen_random (generators.cpp:35-112) and the acceptance
corpus (acceptance.cpp:47-54). Where the reference rejects the parameters (null), the Python
generator must raise.
"""
import hashlib
import json
import os

import pytest

from paper_1909_09213_b200 import models

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "generators.json")))


def sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


def check(want, gen):
    if want is None:
        with pytest.raises(ValueError):
            gen()
    else:
        assert sha(gen()) == want


def test_gen_nqueens_matches_reference():
    for n, want in FIX["nqueens"].items():
        check(want, lambda: models.gen_nqueens(int(n)))


def test_gen_random_matches_reference():
    for key, want in FIX["random"].items():
        v, w, c, s = map(int, key.split(","))
        check(want, lambda: models.gen_random(v, w, c, s))


def test_corpus_instances_match_reference():
    for seed, want in FIX["corpus"].items():
        check(want, lambda: models.corpus_instance(int(seed)))
