"""The bench's expected outputs (tests/golden/bench_golden.json, written by
tools/gen_bench_golden.py from oracle O2 alone) against the independent fingerprints of
SURVEY.md Appendix A.1 (tests/golden/survey_fingerprints.json) and the closed forms the
paper fixes: a plain check that the file bench.py gates on is the greedy's output."""
import json
import math
import os

import pytest

import workloads as WL

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
BENCH = {r["workload"]: r for r in json.load(open(os.path.join(GOLDEN, "bench_golden.json")))["rows"]}
SURVEY = {(r["n"], r["d"], r["order"]): r
          for r in json.load(open(os.path.join(GOLDEN, "survey_fingerprints.json")))["rows"]}


def test_every_bench_workload_has_a_golden_row():
    assert set(WL.BENCH_WORKLOADS) <= set(BENCH)


@pytest.mark.parametrize("wl", [w for w in WL.BENCH_WORKLOADS if len(w.split(",")) == 3])
def test_golden_matches_survey_fingerprints(wl):
    r = BENCH[wl]
    s = SURVEY[(r["n"], r["d"], r["order"])]
    assert r["M"] == s["M"]
    assert r["set_digest"] == s["set_digest"]
    assert r["seq_digest"] == s["seq_digest"]
    if "w_def" in r:
        # SURVEY A.1 prints W_def to 5 significant digits
        assert abs(r["w_def"] - s["w_def"]) <= 1e-4 * s["w_def"]


@pytest.mark.parametrize("wl", [w for w in WL.BENCH_WORKLOADS if len(w.split(",")) == 3])
def test_golden_sizes_closed_forms(wl):
    n, d, o, _ = WL.parse_workload(wl)
    M = BENCH[wl]["M"]
    if d == 3:      # shortened Hamming code size
        assert M == 1 << (n - math.ceil(math.log2(n + 1)))
    elif d == 4:    # extended: the d=3 size at n - 1
        assert M == 1 << (n - 1 - math.ceil(math.log2(n)))
    elif (n, d) == (24, 8):
        assert M == 4096      # extended Golay code (BASELINE configs[1])


def test_fingerprint_functions_match_oracle_module():
    import numpy as np
    import oracle as O
    w = np.array([0, 7, 25, 30, 42, 45, 51, 52, 76, 75, 85, 86, 97, 98, 112, 127], dtype=np.uint32)
    assert WL.seq_digest(w) == O.seq_digest(w)
    assert WL.set_digest(w) == O.set_digest(w)
