"""Pins for the oracle's R29 trusted stub between layers (not gpu):
`relu_requant` and `avgpool` against hand-computed fixtures
(tests/golden/r29_stub.json) and ReLU against PAPER.md:86's own form
Y = (X + sign(X) X) / 2."""
import json
import os

import numpy as np
import pytest

from oracle import ref as R

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "r29_stub.json")))


@pytest.mark.parametrize("case", range(len(GOLD["relu_requant"])))
def test_relu_requant_golden(case):
    g = GOLD["relu_requant"][case]
    got = R.relu_requant(np.array(g["x"], np.int64), g["t"], g["shift"], g["qmax"])
    assert got.tolist() == g["expect"], g["why"]


@pytest.mark.parametrize("case", range(len(GOLD["avgpool"])))
def test_avgpool_golden(case):
    g = GOLD["avgpool"][case]
    assert R.avgpool(np.array(g["x"], np.int64)).tolist() == g["expect"], g["why"]


def test_relu_is_paper_form():
    # PAPER.md:86 (§II-B): ReLU(X) = (X + sign(X) X) / 2.  With shift 0, no
    # clamp and |X| < t/2 the stub is exactly that map.
    t = 65537
    X = np.arange(-32768, 32769, 7, dtype=np.int64)
    paper = (X + np.sign(X) * X) // 2
    assert np.array_equal(R.relu_requant(X, t, 0, 1 << 40), paper)
