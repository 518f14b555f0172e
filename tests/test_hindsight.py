"""NEXT-2 search (tests/tools/hindsight.c) is sound: on C1 (n = 8) its best schedule is
feasible under Eqs. 2-3 and never beats the brute-force hindsight optimum (itself pinned
against scipy's MILP in test_oracle_pins.py); it reaches OPT on most instances."""
import sys
from pathlib import Path

import numpy as np

import workloads as W

sys.path.insert(0, str(Path(__file__).resolve().parent / "tools"))


def test_hindsight_search_never_beats_opt(oracle_mod):
    import hindsight as H
    H.build()
    b = W.c1(120, 77, "b")
    hits = 0
    for k in range(b.n_inst):
        req, M = b.instance(k)
        mc, best, opt, _ = H.one((req, M, 3000, 5 + k, True))
        assert opt <= best <= mc
        hits += best == opt
    assert hits >= 0.8 * b.n_inst
