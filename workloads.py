"""workloads.py -- the bench / test workload strings and their seeded inputs.

Shared by bench.py (the B200 arm), tools/gen_bench_golden.py (which writes the expected
values with oracle/ only) and the tests.  It holds NONE of the method's arithmetic: it
turns "n,d,ordering[,so][,cw=W][,basis=gray|std|seed:S]" into the problem's parameters,
and draws the seeded random basis of a B-ordering -- an input of the
problem, passed to both sides.
"""
from __future__ import annotations

import random

# The bench's workloads: BASELINE.json configs (cfg1 (7,3,lex), cfg2 (24,8,lex), cfg3 d=3
# n=16..24 x 4 orderings, cfg4 (26,4) Gray/graded-lex, cfg5 (28,3,lex)), the other orderings
# of the north_star's "all four orderings up to n=28", and the SURVEY 8(f) rows.
BENCH_WORKLOADS = [
    "7,3,lex",
    "24,8,lex", "24,8,gray", "24,8,glex", "24,8,grlex",
    "24,3,lex", "24,3,gray", "24,3,glex", "24,3,grlex",
    "26,4,lex", "26,4,gray", "26,4,glex", "26,4,grlex",
    "28,3,lex", "28,3,gray", "28,3,glex", "28,3,grlex",
    "22,6,lex,so", "24,6,glex,cw=12", "24,8,lex,basis=seed:1",
]


def random_basis(n: int, seed: int) -> list[int]:
    """n random vectors of F_2^n that are linearly independent (rejection sampling, seeded)."""
    rng = random.Random(seed)
    while True:
        b = [rng.randrange(1, 1 << n) for _ in range(n)]
        red = {}
        for x in b:
            while x:
                h = x.bit_length() - 1
                if h in red:
                    x ^= red[h]
                else:
                    red[h] = x
                    break
        if len(red) == n:
            return b


def parse_workload(s: str):
    """n,d,ordering[,so][,cw=W][,basis=gray|std|seed:S] -> (n, d, ordering, extras)."""
    parts = s.split(",")
    n, d, o = int(parts[0]), int(parts[1]), parts[2]
    ex = {}
    for p in parts[3:]:
        if p == "so":
            ex["self_orthogonal"] = True
        elif p.startswith("cw="):
            ex["constant_weight"] = int(p[3:])
        elif p.startswith("basis="):
            kind = p[6:]
            if kind == "gray":
                ex["basis"] = [1] + [3 << (j - 1) for j in range(1, n)]
            elif kind == "std":
                ex["basis"] = [1 << j for j in range(n)]
            elif kind.startswith("seed:"):
                ex["basis"] = random_basis(n, int(kind[5:]))
            else:
                raise ValueError(f"unknown basis {kind}")
        else:
            raise ValueError(f"unknown workload option {p}")
    return n, d, o, ex


# Output fingerprints: a way to compare two codeword sequences without
# storing them.  Not the method's arithmetic.
_SM1, _SM2, _SM3 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB
SEQ_DIGEST_H0 = 1469598103934665603
_M64 = (1 << 64) - 1


def set_digest(words) -> int:
    """sum of splitmix64(v) mod 2^64 (order-independent)."""
    import numpy as np
    v = np.asarray(words, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = v + np.uint64(_SM1)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_SM2)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_SM3)
        z = z ^ (z >> np.uint64(31))
        return int(z.sum(dtype=np.uint64))


def seq_digest(words, h0: int = SEQ_DIGEST_H0) -> int:
    """FNV-style multiply over whole words (order-dependent)."""
    import numpy as np
    h = h0
    for v in np.asarray(words, dtype=np.uint64).tolist():
        h = ((h ^ v) * 0x100000001B3) & _M64
    return h
