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
