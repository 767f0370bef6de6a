"""Pins for the oracle's SURVEY 8(f) rows: B-ordering, self-orthogonal
greedy codes and constant-weight greedy codes.
Each is tied to the paper's values, to special cases that reduce to the base greedy,
or to a brute-force characterisation with Python's own bit counting."""
import itertools
import json
import math
import os
import random

import numpy as np
import pytest

import oracle as O

PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


def bitcount(x):
    return bin(x).count("1")


def random_basis(n, rng):
    """n random linearly independent vectors (independence checked with Python ints)."""
    while True:
        b = [rng.randrange(1, 1 << n) for _ in range(n)]
        red = {}
        ok = True
        for x in b:
            while x:
                h = x.bit_length() - 1
                if h in red:
                    x ^= red[h]
                else:
                    red[h] = x
                    break
            else:
                ok = False
        if ok:
            return b


# ------------------------------------------------------------------ B-ordering

def test_b_ordering_examples():
    p = PINS["b_ordering"]
    assert O.order_table_basis(3, p["standard_n3"]["basis"]).tolist() == p["standard_n3"]["table"]
    with pytest.raises(ValueError):
        O.order_table_basis(3, p["dependent_n3"])
    t = O.order_table_basis(3, p["independent_n3"])
    assert t.tolist() == [0, 3, 1, 2, 4, 7, 5, 6]        # {0, b1, b2, b2+b1, b3, ...} by hand


@pytest.mark.parametrize("n", [1, 4, 9, 14])
def test_standard_basis_is_lex_and_gray_basis_is_gray(n):
    assert np.array_equal(O.order_table_basis(n, [1 << j for j in range(n)]), O.order_table("lex", n))
    gray_basis = [1] + [3 << (j - 1) for j in range(1, n)]      # b_1 = 1, b_j = 3 * 2^(j-2)
    assert np.array_equal(O.order_table_basis(n, gray_basis), O.order_table("gray", n))


@pytest.mark.parametrize("n", [5, 8, 11])
def test_b_ordering_is_xor_of_basis_for_set_bits(n):
    rng = random.Random(n)
    b = random_basis(n, rng)
    t = O.order_table_basis(n, b).tolist()
    for r in range(1 << n):
        x = 0
        for j in range(n):
            if r >> j & 1:
                x ^= b[j]
        assert t[r] == x
    assert sorted(t) == list(range(1 << n))


@pytest.mark.parametrize("seed", range(6))
def test_b_greedy_codes_are_linear(seed):
    # Brualdi-Pless B-greedy theorem (PAPER.md:19 and :119 cite it): B-greedy codes are linear
    rng = random.Random(100 + seed)
    n = rng.randrange(6, 14)
    b = random_basis(n, rng)
    for d in (2, 3, 4, 5):
        w = O.greedy_ball_ex(n, d, basis=b)
        assert O.is_linear(w), (n, d, b)
        assert np.array_equal(w, O.greedy_plain_ex(n, d, basis=b))


# ------------------------------------------------------------ self-orthogonal

@pytest.mark.parametrize("case", PINS["self_orthogonal"]["cases"], ids=lambda c: f"n{c['n']}d{c['d']}")
def test_self_orthogonal_lexicodes(case):
    n, d = case["n"], case["d"]
    w = O.greedy_ball_ex(n, d, "lex", self_orthogonal=True)
    assert len(w) == case["M"]
    if "words" in case:
        assert w.tolist() == case["words"]
    assert O.is_linear(w) and O.gf2_rank(w) == n // 2          # self-dual: dimension n/2
    if len(w) <= 4096:
        assert O.is_self_orthogonal(w)
    if "weights" in case:
        assert O.weight_distribution(w) == {int(k): v for k, v in case["weights"].items()}
    if n <= 12:
        assert np.array_equal(w, O.greedy_plain_ex(n, d, "lex", self_orthogonal=True))


def brute_force_constrained(n, d, table, words, cw, so):
    """Greedy characterisation with the constraints, by exhaustive loops."""
    rank = {int(v): r for r, v in enumerate(table.tolist())}
    S = [int(x) for x in words]

    def allowed(v):
        return (cw < 0 or bitcount(v) == cw) and (not so or bitcount(v) % 2 == 0)

    def compatible(u, v):
        return bitcount(u ^ v) >= d and (not so or bitcount(u & v) % 2 == 0)

    if any(rank[a] >= rank[b] for a, b in zip(S, S[1:])) or not all(allowed(v) for v in S):
        return False
    if any(not compatible(a, b) for a, b in itertools.combinations(S, 2)):
        return False
    members = set(S)
    for v in range(1 << n):
        if v in members or not allowed(v):
            continue
        if all(rank[s] > rank[v] or compatible(s, v) for s in S):
            return False
    return True


@pytest.mark.parametrize("ordering", ["lex", "gray", "glex", "grlex"])
@pytest.mark.parametrize("n", [2, 4, 6, 8])
def test_self_orthogonal_brute_force(ordering, n):
    t = O.order_table(ordering, n)
    for d in range(1, n + 1):
        w1 = O.greedy_plain_ex(n, d, ordering, self_orthogonal=True, table=t)
        w2 = O.greedy_ball_ex(n, d, ordering, self_orthogonal=True, table=t)
        assert np.array_equal(w1, w2)
        assert brute_force_constrained(n, d, t, w1, -1, True), (n, d)


# -------------------------------------------------------------- constant weight

def test_constant_weight_example():
    p = PINS["constant_weight"]
    w = O.greedy_plain_ex(p["n"], p["d"], "lex", constant_weight=p["w"])
    assert w.tolist() == p["words"]


@pytest.mark.parametrize("ordering", ["lex", "gray", "glex", "grlex"])
@pytest.mark.parametrize("n", [3, 5, 7, 9])
def test_constant_weight_brute_force(ordering, n):
    t = O.order_table(ordering, n)
    for d in (1, 2, 3, 4):
        if d > n:
            continue
        for cw in range(0, n + 1, 2):
            w1 = O.greedy_plain_ex(n, d, ordering, constant_weight=cw, table=t)
            w2 = O.greedy_ball_ex(n, d, ordering, constant_weight=cw, table=t)
            assert np.array_equal(w1, w2)
            assert all(bitcount(int(x)) == cw for x in w1)
            if d == 1 or d == 2 and cw <= 1:
                assert len(w1) == math.comb(n, cw)           # every weight-w vector
            if n <= 7:
                assert brute_force_constrained(n, d, t, w1, cw, False), (n, d, cw)


def test_no_constraint_reduces_to_base_greedy():
    for o in ("lex", "gray", "glex", "grlex"):
        for n, d in ((10, 3), (12, 4), (11, 5)):
            assert np.array_equal(O.greedy_ball_ex(n, d, o), O.greedy_ball(n, d, o))


# ------------------------------------------- is_self_orthogonal: negative pins
# a self-orthogonal code has every codeword "orthogonal to themselves and
# to each other" (AND-parity even).  These fail a checker that returns 1 unconditionally,
# skips the diagonal (a word against itself) or skips the off-diagonal pairs.

def test_is_self_orthogonal_negative_golay23():
    # the (23,7) lexicode is the [23,12,7] Golay code: odd weights 7, 11, ...
    w = O.greedy_ball(23, 7, "lex")
    assert len(w) == 4096
    assert not O.is_self_orthogonal(w[:64])     # contains words of odd weight 7


def test_is_self_orthogonal_negative_pair():
    # 3 = 011, 5 = 101: both of even weight (each orthogonal to itself), 3 & 5 = 001 odd
    assert O.orthogonal(3, 3) and O.orthogonal(5, 5)
    assert not O.orthogonal(3, 5)
    assert not O.is_self_orthogonal([3, 5])
    assert not O.is_self_orthogonal([0, 3, 5])


def test_is_self_orthogonal_negative_single_odd_word():
    # a word of odd weight is not orthogonal to itself (the diagonal): 7 = 111
    assert not O.is_self_orthogonal([7])
    assert not O.is_self_orthogonal([0, 7])


def test_is_self_orthogonal_positive_small():
    assert O.is_self_orthogonal([])
    assert O.is_self_orthogonal([0])
    assert O.is_self_orthogonal([0, 3, 12, 15])     # [4,2] repetition pairs: 0011, 1100, 1111


# ------------------------- constant weight on 64-bit words ("up to 35")

@pytest.mark.parametrize("ordering", ["lex", "glex", "grlex"])
@pytest.mark.parametrize("n", [33, 35])
def test_cw64_closed_forms(ordering, n):
    from math import comb
    for w in (1, 2, 3):
        # d = 2: any two distinct weight-w words differ in >= 2 places, so every one is accepted
        w2 = O.greedy_cw64(n, 2, w, ordering)
        assert len(w2) == comb(n, w) and len(set(w2.tolist())) == comb(n, w)
        assert all(bin(int(x)).count("1") == w for x in w2)
        # d = 2w: supports must be disjoint; the greedy takes consecutive blocks of w coordinates
        wd = O.greedy_cw64(n, 2 * w, w, ordering)
        assert len(wd) == n // w
        acc = 0
        for x in wd.tolist():
            assert acc & x == 0
            acc |= x
        # d > 2w: no two weight-w words are that far apart
        if 2 * w + 1 <= n:
            assert len(O.greedy_cw64(n, 2 * w + 1, w, ordering)) == 1
    # the orders: ascending / descending values within the class
    w4 = O.greedy_cw64(n, 2, 4, ordering)
    assert list(w4) == sorted(w4.tolist(), reverse=(ordering == "grlex"))


@pytest.mark.parametrize("ordering", ["lex", "glex", "grlex"])
@pytest.mark.parametrize("n,d,w", [(12, 4, 5), (14, 4, 4), (16, 6, 6), (18, 4, 3), (20, 6, 5), (13, 3, 6)])
def test_cw64_matches_u32_oracle(ordering, n, d, w):
    # the 32-bit constant-weight oracles (pinned in this file) restricted to n <= 32
    ref = O.greedy_ball_ex(n, d, ordering, constant_weight=w)
    got = O.greedy_cw64(n, d, w, ordering)
    assert np.array_equal(got.astype(np.uint32), ref) and got.max(initial=0) < (1 << n)


@pytest.mark.parametrize("ordering", ["lex", "grlex"])
@pytest.mark.parametrize("n", [6, 8, 9])
def test_cw64_greedy_characterisation(ordering, n):
    # brute force: in the order of the weight class, a word is in the code iff it is at distance
    # >= d from every EARLIER code word (Python bit counting, independent of the oracle's code)
    from itertools import combinations
    for w in range(1, n):
        cls = sorted((sum(1 << b for b in c) for c in combinations(range(n), w)), reverse=(ordering == "grlex"))
        for d in range(1, n + 1):
            code = O.greedy_cw64(n, d, w, ordering).tolist()
            pos = {v: i for i, v in enumerate(cls)}
            for i, v in enumerate(cls):
                earlier = [c for c in code if pos[c] < i]
                ok = all(bin(v ^ c).count("1") >= d for c in earlier)
                assert (v in code) == ok, (n, d, w, v)
