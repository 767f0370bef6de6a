"""Pins for the CPU oracle (oracle/): what the paper and the mathematics fix.

Every test here ties the oracle to something other than itself:
  * values printed in PAPER.md (Example 1, perfect/Golay claims) -- tests/golden/paper_pins.json
  * closed forms (shortened / extended Hamming sizes, sphere-packing equality)
  * special cases with a known answer (d=1, d=2, d=n)
  * the defining properties of the greedy output checked by brute force on tiny n
    (pairwise distance >= d; every rejected vector has an EARLIER accepted vector
    within distance d-1; acceptance order = rank order) -- these characterise the
    greedy output uniquely, so they pin the whole sequence
  * agreement of two different algorithms (O1 plain scan, O2 ball marking)
  * an independent implementation's fingerprints
No test here needs a GPU.
"""
import itertools
import json
import math
import os
import random

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
PINS = json.load(open(os.path.join(GOLDEN, "paper_pins.json")))
ORDERS = ["lex", "gray", "glex", "grlex"]


def bitcount(x: int) -> int:
    # independent of the oracle's popcount: Python's binary string
    return bin(x).count("1")


# ------------------------------------------------------------ bit primitives

def test_distance_matches_bit_by_bit_count():
    rng = random.Random(0)
    pairs = [(rng.getrandbits(32), rng.getrandbits(32)) for _ in range(20000)]
    pairs += [(u, v) for u in range(64) for v in range(64)]
    for u, v in pairs:
        assert O.distance(u, v) == bitcount(u ^ v)
        assert O.weight(u) == bitcount(u)


def test_distance_metric_axioms_exhaustive_n5():
    N = 1 << 5
    for u in range(N):
        assert O.distance(u, u) == 0
        for v in range(N):
            duv = O.distance(u, v)
            assert duv == O.distance(v, u)
            assert (duv == 0) == (u == v)
            for w in range(0, N, 3):
                assert O.distance(u, w) <= duv + O.distance(v, w)


# ------------------------------------------------------------------ orderings

def test_orderings_small_examples():
    p = PINS["orderings_n3"]
    assert O.order_table("lex", 3).tolist() == p["lex"]
    assert O.order_table("gray", 3).tolist() == p["gray"]
    assert O.order_table("glex", 3).tolist() == p["glex"]
    assert O.order_table("grlex", 2).tolist() == p["grlex_n2"]


@pytest.mark.parametrize("ordering", ORDERS)
@pytest.mark.parametrize("n", [1, 2, 5, 8, 12, 16])
def test_ordering_is_bijection_starting_at_zero(ordering, n):
    t = O.order_table(ordering, n)
    assert t[0] == 0  # PAPER.md:59 "starting from zero vector"
    assert np.array_equal(np.sort(t), np.arange(1 << n, dtype=np.uint32))


@pytest.mark.parametrize("n", [1, 2, 3, 8, 13, 16, 20])
def test_gray_is_reflected_binary(n):
    t = O.order_table("gray", n).astype(np.int64)
    # consecutive vectors differ in exactly one coordinate
    diff = t[1:] ^ t[:-1]
    assert np.all((diff & (diff - 1)) == 0) and np.all(diff != 0)
    # closed form of the reflected binary code (textbook): g(r) = r XOR (r >> 1)
    r = np.arange(1 << n, dtype=np.int64)
    assert np.array_equal(t, r ^ (r >> 1))


@pytest.mark.parametrize("ordering", ["glex", "grlex"])
@pytest.mark.parametrize("n", [2, 5, 9, 14])
def test_graded_orders(ordering, n):
    t = O.order_table(ordering, n).tolist()
    w = [bitcount(x) for x in t]
    assert all(a <= b for a, b in zip(w, w[1:]))  # weight classes ascending
    for a, b, wa, wb in zip(t, t[1:], w, w[1:]):
        if wa == wb:
            assert (a < b) if ordering == "glex" else (a > b)  # DESIGN.md reading R2
    # class sizes are binomial coefficients
    for k in range(n + 1):
        assert w.count(k) == math.comb(n, k)


# -------------------------------------------------------------- Example 1

def test_example1_output_and_steps():
    e = PINS["example1"]
    for fn in (lambda: O.greedy_plain(3, 2, "lex"), lambda: O.greedy_ball(3, 2, "lex")):
        assert fn().tolist() == e["output"]
    # "Output array size is checked ... (size = s)" before step k considers rank k-1
    for step, size in e["steps_sizes"].items():
        prefix = O.greedy_plain(3, 2, "lex", nranks=int(step) - 1)
        assert len(prefix) == size, (step, prefix)


# ----------------------------------------------------------- paper theorems

@pytest.mark.parametrize("case", PINS["perfect"]["cases"], ids=lambda c: f"n{c['n']}d{c['d']}")
def test_perfect_lexicodes(case):
    n, d = case["n"], case["d"]
    w = O.greedy_ball(n, d, "lex")
    assert len(w) == case["M"]
    assert O.gf2_rank(w) == case["k"] and O.is_linear(w)
    t = (d - 1) // 2
    assert len(w) * sum(math.comb(n, i) for i in range(t + 1)) == 1 << n  # perfect
    if "weights" in case:
        assert O.weight_distribution(w) == {int(k): v for k, v in case["weights"].items()}
        # linear code: min distance = min nonzero weight
        assert min(k for k in O.weight_distribution(w) if k) == d
    if len(w) <= 2048:
        assert O.min_distance_pairs(w) == d


@pytest.mark.slow
def test_extended_golay_lexicode():
    g = PINS["extended_golay"]
    w = O.greedy_ball(24, 8, "lex")
    assert len(w) == g["M"] and O.gf2_rank(w) == g["k"]
    assert O.weight_distribution(w) == {int(k): v for k, v in g["weights"].items()}


@pytest.mark.parametrize("n", range(3, 23))
def test_d3_lexicode_is_shortened_hamming(n):
    # M = 2^(n - ceil(log2(n+1)))  (BASELINE.json north_star; Hamming code theory)
    w = O.greedy_ball(n, 3, "lex")
    r = math.ceil(math.log2(n + 1))
    assert len(w) == 1 << (n - r)
    assert O.is_linear(w)


@pytest.mark.parametrize("n", range(4, 23))
def test_d4_lexicode_is_extended_hamming(n):
    # M = 2^(n - 1 - ceil(log2 n))  (extended / shortened-extended Hamming codes)
    w = O.greedy_ball(n, 4, "lex")
    assert len(w) == 1 << (n - 1 - math.ceil(math.log2(n)))


@pytest.mark.parametrize("ordering", ORDERS)
@pytest.mark.parametrize("n", [1, 2, 4, 7, 10])
def test_special_cases(ordering, n):
    t = O.order_table(ordering, n)
    # d = 1: every vector is at distance >= 1 from every other -> all 2^n, in order
    assert np.array_equal(O.greedy_ball(n, 1, ordering), t)
    assert np.array_equal(O.greedy_plain(n, 1, ordering), t)
    # d = n: only the all-ones vector is at distance n from 0
    assert O.greedy_ball(n, n, ordering).tolist() == ([0, (1 << n) - 1] if n >= 1 else [0])
    # d = 2: the even-weight code, as a set, for every ordering
    if n >= 2:
        w = O.greedy_ball(n, 2, ordering)
        assert sorted(w.tolist()) == [v for v in range(1 << n) if bitcount(v) % 2 == 0]


# ------------------------------------------- brute-force characterisation

def brute_force_is_greedy_output(n, d, table, words):
    """The greedy output is the unique list S with: ranks strictly increasing,
    pairwise distances >= d, and every non-member v has a member of smaller rank
    within distance < d.  Checked here by exhaustive loops with Python's own
    bit counting -- independent of the oracle's code."""
    rank = {int(v): r for r, v in enumerate(table.tolist())}
    S = [int(x) for x in words]
    if any(rank[a] >= rank[b] for a, b in zip(S, S[1:])):
        return False
    for a, b in itertools.combinations(S, 2):
        if bitcount(a ^ b) < d:
            return False
    members = set(S)
    for v in range(1 << n):
        if v in members:
            continue
        if not any(rank[s] < rank[v] and bitcount(s ^ v) < d for s in S):
            return False
    return True


@pytest.mark.parametrize("ordering", ORDERS)
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 9])
def test_oracles_satisfy_greedy_characterisation(ordering, n):
    t = O.order_table(ordering, n)
    for d in range(1, n + 1):
        w1 = O.greedy_plain(n, d, ordering, table=t)
        w2 = O.greedy_ball(n, d, ordering)
        assert np.array_equal(w1, w2), (n, d)
        assert brute_force_is_greedy_output(n, d, t, w1), (n, d)
        assert O.certify(n, d, ordering, w1, table=t) == (True, 0)


def test_certificate_rejects_wrong_lists():
    n, d = 8, 3
    t = O.order_table("lex", n)
    w = O.greedy_plain(n, d, "lex", table=t)
    assert O.certify(n, d, "lex", w, table=t) == (True, 0)
    assert O.certify(n, d, "lex", w[:-1], table=t)[1] == 3                    # not maximal
    swapped = w.copy(); swapped[[2, 3]] = swapped[[3, 2]]
    assert O.certify(n, d, "lex", swapped, table=t)[1] == 1                   # order
    extra = np.sort(np.append(w, np.uint32(1)))                               # 1 is within 1 of 0
    assert O.certify(n, d, "lex", extra, table=t)[0] is False
    other = O.greedy_plain(n, d, "glex")
    assert O.certify(n, d, "lex", other, table=t)[0] is False or np.array_equal(other, w)
    for bad in (w[:-1], swapped, extra):
        assert not brute_force_is_greedy_output(n, d, t, bad)


# ------------------------------------------------ O1 == O2 (two algorithms)

@pytest.mark.parametrize("ordering", ORDERS)
@pytest.mark.parametrize("n", [10, 13, 16])
def test_plain_equals_ball(ordering, n):
    t = O.order_table(ordering, n)
    for d in range(2, min(n, 8) + 1):
        w1 = O.greedy_plain(n, d, ordering, table=t)
        w2 = O.greedy_ball(n, d, ordering)
        assert np.array_equal(w1, w2), (n, d)
        assert O.certify(n, d, ordering, w2, table=t) == (True, 0)


@pytest.mark.slow
@pytest.mark.parametrize("ordering", ORDERS)
def test_plain_equals_ball_n18_d3(ordering):
    t = O.order_table(ordering, 18)
    assert np.array_equal(O.greedy_plain(18, 3, ordering, table=t), O.greedy_ball(18, 3, ordering))


# ------------------------------------------------------ paper invariants

@pytest.mark.parametrize("ordering", ["lex", "gray"])
@pytest.mark.parametrize("n", [6, 11, 16])
def test_lex_and_gray_codes_are_linear(ordering, n):
    # PAPER.md:175 (Fig. 5 caption) for lex; Gray is a B-ordering
    for d in range(1, n + 1):
        assert O.is_linear(O.greedy_ball(n, d, ordering)), (n, d)


@pytest.mark.parametrize("n", range(2, 17))
def test_power_of_two_d_lex_equals_graded_lex_as_sets(n):
    # d a power of 2 -> lex and graded-lex greedy codes contain the same words
    for d in (2, 4, 8):
        if d <= n:
            a = O.greedy_ball(n, d, "lex")
            b = O.greedy_ball(n, d, "glex")
            assert sorted(a.tolist()) == sorted(b.tolist()), (n, d)


# ---------------------------------------- independent implementation (survey)

SURVEY = json.load(open(os.path.join(GOLDEN, "survey_fingerprints.json")))["rows"]


def ranks_of(words, n, ordering):
    t = O.order_table(ordering, n)
    inv = np.empty(1 << n, dtype=np.int64)
    inv[t] = np.arange(1 << n)
    return inv[np.asarray(words, dtype=np.int64)]


@pytest.mark.parametrize(
    "row", [r for r in SURVEY if r["n"] <= 21 or (r["n"] == 23 and r["d"] == 7)],
    ids=lambda r: f"n{r['n']}d{r['d']}{r['order']}")
def test_oracle_matches_survey_fingerprints(row):
    n, d, o = row["n"], row["d"], row["order"]
    w = O.greedy_ball(n, d, o)
    assert len(w) == row["M"]
    assert w[:8].tolist() == row["first8"][: len(w[:8])]
    assert int(w[-1]) == row["last"]
    rk = ranks_of(w, n, o)
    assert int(rk[-1]) == row["last_rank"]
    assert O.is_linear(w) == row["linear"]
    assert format(O.set_digest(w), "016x") == row["set_digest"]
    assert format(O.seq_digest(w), "016x") == row["seq_digest"]
    wd = O.w_def(n, rk)
    assert abs(wd - row["w_def"]) <= 1e-4 * row["w_def"]


# ------------------------------- O1 with thread sections (Fig. 2(b))

def test_plain_mt_example1():
    # Example 1 with the inner loop split over 1..4 threads
    e = PINS["example1"]
    for T in (1, 2, 3, 4):
        assert O.greedy_plain_mt(3, 2, "lex", threads=T).tolist() == e["output"]
        for step, size in e["steps_sizes"].items():
            assert len(O.greedy_plain_mt(3, 2, "lex", threads=T, nranks=int(step) - 1)) == size


@pytest.mark.parametrize("ordering", ORDERS)
@pytest.mark.parametrize("n", [4, 7, 9])
def test_plain_mt_satisfies_greedy_characterisation(ordering, n):
    t = O.order_table(ordering, n)
    for d in range(1, n + 1):
        for T in (2, 5):
            w = O.greedy_plain_mt(n, d, ordering, threads=T, table=t)
            assert brute_force_is_greedy_output(n, d, t, w), (n, d, T)


@pytest.mark.parametrize("ordering", ORDERS)
def test_plain_mt_hamming_sizes(ordering):
    # d = 3 lexicode size = shortened Hamming code size 2^(n - ceil(log2(n+1))) (every ordering: P:231)
    for n in (11, 14):
        w = O.greedy_plain_mt(n, 3, ordering, threads=4)
        assert len(w) == 1 << (n - math.ceil(math.log2(n + 1)))
        assert np.array_equal(w, O.greedy_ball(n, 3, ordering))
