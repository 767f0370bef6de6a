"""GPU code analysis against the oracle's definitions."""
import random

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gc(need_gpu):
    import paper_1507_05398_b200 as m
    return m


def check(gc, words, pairwise=True, orthogonality=True):
    words = np.asarray(words, dtype=np.uint32)
    a = gc.gc_analyze(words.astype(np.uint64), pairwise=pairwise, orthogonality=orthogonality)
    assert a["M"] == len(words)
    assert a["weights"] == O.weight_distribution(words)
    assert a["gf2_rank"] == O.gf2_rank(words)
    assert a["is_linear"] == O.is_linear(words)
    if pairwise and len(words) <= 5000:
        assert a["min_distance"] == (O.min_distance_pairs(words) if len(words) > 1 else 0)
        assert a["pairs_checked"] == len(words) * (len(words) - 1) // 2
    if orthogonality and len(words) <= 5000:
        assert a["self_orthogonal"] == O.is_self_orthogonal(words)
    return a


def test_golay_codes(gc):
    g23 = O.greedy_ball(23, 7, "lex")
    a = check(gc, g23)
    assert a["min_distance"] == 7 and a["gf2_rank"] == 12 and a["is_linear"]
    g24 = O.greedy_ball(24, 8, "lex")
    a = check(gc, g24)
    assert a["min_distance"] == 8 and a["self_orthogonal"] is True
    # linear code: min distance from the weights without the pairwise pass
    a2 = gc.gc_analyze(g24.astype(np.uint64))
    assert a2["min_distance"] == 8 and a2["self_orthogonal"] is True and a2["pairs_checked"] == 0


def test_nonlinear_and_small(gc):
    check(gc, O.greedy_ball(23, 7, "glex"))           # 585 words, nonlinear
    check(gc, O.greedy_ball(16, 5, "grlex"))
    check(gc, [5])
    a = gc.gc_analyze(np.zeros(0, dtype=np.uint64))
    assert a["M"] == 0 and a["min_distance"] == 0
    a = gc.gc_analyze(np.array([3, 5], dtype=np.uint64))    # even weights, nonlinear, no pairwise: unknown
    assert a["self_orthogonal"] is None and a["min_distance"] == 0


@pytest.mark.parametrize("seed", range(4))
def test_random_sets(gc, seed):
    rng = random.Random(seed)
    M = rng.randrange(2, 3000)
    words = sorted(set(rng.getrandbits(rng.randrange(5, 33)) for _ in range(M)))
    check(gc, words)


def test_device_entry_on_a_gpu_code(gc):
    import torch
    n, d = 22, 6
    cap = gc.gc_capacity_bound(n, d)
    cb = torch.empty(cap, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    gc.gc_construct_device(n, d, cb, cnt, self_orthogonal=True)
    M = int(cnt.item())
    a = gc.gc_analyze_device(cb, M=M, pairwise=True, orthogonality=True)
    assert M == 2048 and a["gf2_rank"] == 11 and a["min_distance"] == 6 and a["self_orthogonal"] is True
