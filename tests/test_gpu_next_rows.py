"""GPU parity for the SURVEY 8(f) rows (B-ordering, self-orthogonal, constant weight):
the persistent sm_100a engine through gc_construct against the oracle, bit-exact."""
import json
import os
import random

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


@pytest.fixture(scope="module")
def gc(need_gpu):
    import paper_1507_05398_b200 as m
    return m


def random_basis(n, rng):
    while True:
        b = [rng.randrange(1, 1 << n) for _ in range(n)]
        red, ok = {}, True
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


def run(gc, n, d, **kw):
    w, st = gc.gc_construct(n, d, **kw)
    assert st["M"] == len(w)
    return w.astype(np.uint32)


@pytest.mark.parametrize("seed", range(8))
def test_b_ordering_random_bases(gc, seed):
    rng = random.Random(seed)
    n = rng.randrange(8, 21)
    b = random_basis(n, rng)
    for d in (2, 3, 4, 6):
        w = run(gc, n, d, basis=b)
        assert np.array_equal(w, O.greedy_ball_ex(n, d, basis=b)), (n, d)


@pytest.mark.parametrize("n", [10, 18])
def test_b_ordering_special_bases(gc, n):
    std = [1 << j for j in range(n)]
    gray = [1] + [3 << (j - 1) for j in range(1, n)]
    for d in (3, 5):
        assert np.array_equal(run(gc, n, d, basis=std), gc.gc_generate(n, d, "lex").astype(np.uint32))
        assert np.array_equal(run(gc, n, d, basis=gray), gc.gc_generate(n, d, "gray").astype(np.uint32))


@pytest.mark.parametrize("case", PINS["self_orthogonal"]["cases"], ids=lambda c: f"n{c['n']}d{c['d']}")
def test_self_orthogonal_paper_codes(gc, case):
    n, d = case["n"], case["d"]
    w = run(gc, n, d, self_orthogonal=True)
    assert len(w) == case["M"]
    assert O.is_linear(w) and O.gf2_rank(w) == n // 2
    if "weights" in case:
        assert O.weight_distribution(w) == {int(k): v for k, v in case["weights"].items()}
    assert np.array_equal(w, O.greedy_ball_ex(n, d, "lex", self_orthogonal=True))


@pytest.mark.parametrize("ordering", ["lex", "gray", "glex", "grlex"])
@pytest.mark.parametrize("n", [6, 11, 16])
def test_self_orthogonal_vs_oracle(gc, ordering, n):
    for d in (2, 3, 4, 6):
        if d <= n:
            w = run(gc, n, d, ordering=ordering, self_orthogonal=True)
            assert np.array_equal(w, O.greedy_ball_ex(n, d, ordering, self_orthogonal=True)), (n, d)


def test_constant_weight_example(gc):
    p = PINS["constant_weight"]
    assert run(gc, p["n"], p["d"], constant_weight=p["w"]).tolist() == p["words"]


@pytest.mark.parametrize("ordering", ["lex", "gray", "glex", "grlex"])
@pytest.mark.parametrize("n", [9, 14, 18])
def test_constant_weight_vs_oracle(gc, ordering, n):
    for d, cw in ((2, 3), (4, n // 2), (6, n // 2 + 1), (3, 1)):
        w = run(gc, n, d, ordering=ordering, constant_weight=cw)
        assert np.array_equal(w, O.greedy_ball_ex(n, d, ordering, constant_weight=cw)), (n, d, cw)


@pytest.mark.parametrize("sched", [{"tile_min": 32, "tile_max": 64, "window0": 32}, {"window_growth": 1},
                                   {"tile_min": 4096, "tile_max": 4096}, {"flags": 32}, {"emulate_ranks": 4}])
def test_combined_constraints_schedule_invariance(gc, sched):
    rng = random.Random(7)
    b = random_basis(14, rng)
    for kw in (dict(basis=b, self_orthogonal=True), dict(ordering="glex", constant_weight=7),
               dict(basis=b, constant_weight=5), dict(ordering="gray", self_orthogonal=True, constant_weight=6)):
        n, d = 14, 4
        w = run(gc, n, d, options=sched, **kw)
        ref = O.greedy_ball_ex(n, d, kw.get("ordering", "lex"), constant_weight=kw.get("constant_weight", -1),
                               self_orthogonal=kw.get("self_orthogonal", False), basis=kw.get("basis"))
        assert np.array_equal(w, ref), (kw, sched)


def test_extended_problems_need_persistent_engine(gc):
    with pytest.raises(gc.GCError) as e:
        gc.gc_construct(10, 3, self_orthogonal=True, options={"flags": 16})
    assert e.value.name == "GC_EUNSUPPORTED"


# ------------- constant weight on 64-bit words, n = 33..35 ("up-to 35")

@pytest.mark.parametrize("ordering", ["lex", "glex", "grlex"])
@pytest.mark.parametrize("n,d,w", [(33, 4, 4), (35, 4, 4), (35, 6, 5), (33, 2, 3), (35, 8, 4), (34, 6, 6),
                                   (35, 10, 5), (33, 4, 30)])
def test_cw64_matches_oracle(gc, ordering, n, d, w):
    got, st = gc.gc_construct(n, d, ordering=ordering, constant_weight=w)
    ref = O.greedy_cw64(n, d, w, ordering)
    assert st["M"] == len(ref)
    assert np.array_equal(got.astype(np.uint64), ref), (n, d, w, ordering)


def test_cw64_unsupported_combinations(gc):
    for kw in (dict(ordering="gray", constant_weight=4), dict(ordering="lex"),
               dict(ordering="lex", constant_weight=4, self_orthogonal=True)):
        with pytest.raises(gc.GCError) as e:
            gc.gc_construct(34, 4, **kw)
        assert e.value.name == "GC_EUNSUPPORTED"
