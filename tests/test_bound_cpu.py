"""CPU pins for the exact pruning bounds the GPU screen uses (host logic, no GPU).

The persistent engine skips a block of codewords when a LOWER BOUND on the distance between
every live candidate of a warp and every codeword of the block is already >= d.  Skipping is
exact only if the bound never exceeds a true distance; these tests pin that lemma by brute
force on random and adversarial sets, independently of the CUDA code (which the GPU parity
tests cover end to end, with and without GC_FLAG_NO_BLOCK_BOUND).

  block bound  (csrc/gc_persistent.cu p_lb):
      lb = popc(((AND_blk & ~OR_cand) | (AND_cand & ~OR_blk)) & (2^n - 1))
      -- positions where every codeword has bit x and every candidate has 1 - x.
  weight bound (graded orders, p_base):  |wt(u) - wt(v)| <= dist(u, v).
"""
import random

import pytest


def popc(x):
    return bin(x).count("1")


def block_bound(block, cands, n):
    band, bor, cand, cor = (1 << n) - 1, 0, (1 << n) - 1, 0
    for w in block:
        band &= w
        bor |= w
    for v in cands:
        cand &= v
        cor |= v
    return popc(((band & ~cor) | (cand & ~bor)) & ((1 << n) - 1))


@pytest.mark.parametrize("seed", range(40))
def test_block_bound_never_exceeds_min_distance(seed):
    rng = random.Random(seed)
    n = rng.choice([3, 7, 12, 20, 28, 32])
    for _ in range(50):
        # mixes of random words and near-identical clusters (where the bound is tight)
        base_b, base_c = rng.getrandbits(n), rng.getrandbits(n)
        flip = rng.randrange(0, n + 1)
        block = [(base_b ^ (rng.getrandbits(n) & rng.getrandbits(n) & rng.getrandbits(n)))
                 if rng.random() < 0.8 else rng.getrandbits(n) for _ in range(rng.randrange(1, 33))]
        cands = [(base_c ^ (rng.getrandbits(n) & rng.getrandbits(n) & rng.getrandbits(n)))
                 for _ in range(rng.randrange(1, 65))]
        if flip:
            cands = [v ^ ((1 << flip) - 1) for v in cands]
        lb = block_bound(block, cands, n)
        dmin = min(popc(u ^ v) for u in block for v in cands)
        assert lb <= dmin


def test_block_bound_is_tight_for_single_words():
    # one codeword, one candidate: AND = OR = the word, so the bound is the distance itself
    rng = random.Random(7)
    for _ in range(2000):
        n = rng.randrange(1, 33)
        u, v = rng.getrandbits(n), rng.getrandbits(n)
        assert block_bound([u], [v], n) == popc(u ^ v)


def test_block_bound_ignores_bits_above_n():
    # bits >= n are masked: an empty high part never contributes
    assert block_bound([0b101], [0b010], 3) == 3
    assert block_bound([0b0], [0b0], 1) == 0


def test_block_bound_weak_for_mixed_sets():
    # a block containing a word and its complement agrees on no position: bound 0
    n = 16
    assert block_bound([0x1234, 0x1234 ^ 0xFFFF], [0x0F0F], n) == 0


@pytest.mark.parametrize("seed", range(10))
def test_weight_bound(seed):
    rng = random.Random(100 + seed)
    for _ in range(2000):
        n = rng.randrange(1, 33)
        u, v = rng.getrandbits(n), rng.getrandbits(n)
        assert abs(popc(u) - popc(v)) <= popc(u ^ v)


# ------------------------------------------------ parity refinement (a.par, n <= 30)

def tagged(words):
    # bit 31 = weight parity, as the parity-tagged summaries hold it (csrc/gc_screen.cuh p_ptag)
    return [w | ((popc(w) & 1) << 31) for w in words]


def parity_bound(block, cands, n):
    """p_lbs: the block bound rounded up to the parity every distance must have when both sides
    have a single weight parity (AND and OR agree in bit 31)."""
    tb, tc = tagged(block), tagged(cands)
    band, bor, cand, cor = 0xFFFFFFFF, 0, 0xFFFFFFFF, 0
    for w in tb:
        band &= w
        bor |= w
    for v in tc:
        cand &= v
        cor |= v
    lb = popc(((band & ~cor) | (cand & ~bor)) & ((1 << n) - 1))
    uniform = not (((band ^ bor) | (cand ^ cor)) >> 31) & 1
    if uniform and (lb ^ ((bor ^ cor) >> 31)) & 1:
        lb += 1
    return lb


@pytest.mark.parametrize("seed", range(40))
def test_parity_bound_never_exceeds_min_distance(seed):
    rng = random.Random(1000 + seed)
    n = rng.choice([4, 7, 12, 20, 26, 30])
    for _ in range(60):
        # single-weight-class blocks and candidate batches (graded orders) and mixtures
        wb, wc = rng.randrange(0, n + 1), rng.randrange(0, n + 1)

        def word(weight):
            if rng.random() < 0.7:
                bits = rng.sample(range(n), weight)
                return sum(1 << b for b in bits)
            return rng.getrandbits(n)
        block = [word(wb) for _ in range(rng.randrange(1, 33))]
        cands = [word(wc) for _ in range(rng.randrange(1, 65))]
        lb = parity_bound(block, cands, n)
        dmin = min(popc(u ^ v) for u in block for v in cands)
        assert lb <= dmin
        assert lb >= block_bound(block, cands, n)


def test_parity_bound_rounds_up():
    # one weight class on each side: equal parities -> every distance even
    n = 8
    block = [0b00000111]                        # weight 3
    cands = [0b01101000]                        # weight 3: distance 6
    lb0 = block_bound(block, cands, n)
    assert lb0 == 6 and parity_bound(block, cands, n) == 6
    block = [0b00000111, 0b00001011]            # weight 3 (AND = 0b11)
    cands = [0b00110001]                        # weight 3; plain bound 3 (odd) -> parity even -> 4
    assert block_bound(block, cands, n) == 3
    assert parity_bound(block, cands, n) == 4 == min(popc(b ^ cands[0]) for b in block)
