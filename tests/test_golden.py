"""CPU: the oracle reproduces its frozen fixture digests bit for bit
(tests/golden/gen_golden.py wrote them; FNV-1a as include/splatsim/rng.hpp:60-69)."""
import json
import os

import pytest

from golden.gen_golden import FIXTURES, compute

HERE = os.path.dirname(os.path.abspath(__file__))


def test_golden_digests():
    with open(os.path.join(HERE, "golden", "digests.json")) as f:
        frozen = json.load(f)
    assert set(frozen) == set(FIXTURES)
    assert compute() == frozen
