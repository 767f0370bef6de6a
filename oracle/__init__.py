"""CPU oracle for the greedy binary-code construction -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1507_05398_b200``) never imports it, and it imports nothing from the
product path: the two share no code (the only common module is
``tests/inputs.py``-style parameter generation, which holds no arithmetic of the
method -- here the "input" is just (n, d, ordering)).

The arithmetic lives in ``greedy_oracle.c`` (plain C, compiled by
``__graft_entry__.build()`` into ``oracle/liboracle.so``).  This module is
argument marshalling plus a few analysis helpers written in numpy.

Functions follow PAPER.md (``/root/reference/PAPER.md``):
  order_table      -- Sec. 4.2 orderings
  greedy_plain     -- O1, Fig. 2(a) serial greedy
  greedy_ball      -- O2, exact ball-marking restatement of the same greedy
  certify          -- O3, certificate that a list IS the greedy output
  gf2_rank, weight_distribution, min_distance_pairs -- analysis
  seq_digest, set_digest -- fingerprints (SURVEY.md Appendix A.3 definitions)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

LEX, GRAY, GRADED_LEX, GRADED_REVLEX = 0, 1, 2, 3
ORDER_NAMES = {"lex": LEX, "gray": GRAY, "glex": GRADED_LEX, "grlex": GRADED_REVLEX}

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "greedy_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile greedy_oracle.c with plain gcc -O2 (no tuning flags)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-mpopcnt", "-Wall", "-pthread", "-shared", "-fPIC", "-o", _SO, _SRC]
        )
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        L.or_order_table.argtypes = [ctypes.c_int, ctypes.c_int, u32p]
        L.or_order_table.restype = ctypes.c_int
        L.or_greedy_plain.argtypes = [ctypes.c_int, ctypes.c_int, u32p, ctypes.c_uint64, u32p,
                                      ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
        L.or_greedy_plain.restype = ctypes.c_int64
        L.or_greedy_plain_mt.argtypes = [ctypes.c_int, ctypes.c_int, u32p, ctypes.c_uint64, ctypes.c_int, u32p,
                                         ctypes.c_uint64]
        L.or_greedy_plain_mt.restype = ctypes.c_int64
        L.or_greedy_ball.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, u32p, ctypes.c_uint64]
        L.or_greedy_ball.restype = ctypes.c_int64
        L.or_certify.argtypes = [ctypes.c_int, ctypes.c_int, u32p, u32p, ctypes.c_uint64,
                                 ctypes.POINTER(ctypes.c_int)]
        L.or_certify.restype = ctypes.c_int
        L.or_gf2_rank.argtypes = [u32p, ctypes.c_uint64]
        L.or_gf2_rank.restype = ctypes.c_int
        L.or_weight_distribution.argtypes = [u32p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
        L.or_min_distance_pairs.argtypes = [u32p, ctypes.c_uint64]
        L.or_min_distance_pairs.restype = ctypes.c_int
        L.or_distance.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.or_distance.restype = ctypes.c_int
        L.or_weight.argtypes = [ctypes.c_uint32]
        L.or_weight.restype = ctypes.c_int
        L.or_order_table_basis.argtypes = [ctypes.c_int, u32p, u32p]
        L.or_order_table_basis.restype = ctypes.c_int
        L.or_greedy_plain_ex.argtypes = [ctypes.c_int, ctypes.c_int, u32p, ctypes.c_uint64, ctypes.c_int,
                                         ctypes.c_int, u32p, ctypes.c_uint64]
        L.or_greedy_plain_ex.restype = ctypes.c_int64
        L.or_greedy_ball_ex.argtypes = [ctypes.c_int, ctypes.c_int, u32p, ctypes.c_int, ctypes.c_int, u32p,
                                        ctypes.c_uint64]
        L.or_greedy_ball_ex.restype = ctypes.c_int64
        L.or_is_self_orthogonal.argtypes = [u32p, ctypes.c_uint64]
        L.or_is_self_orthogonal.restype = ctypes.c_int
        L.or_greedy_cw64.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_uint64), ctypes.c_uint64]
        L.or_greedy_cw64.restype = ctypes.c_int64
        L.or_orthogonal.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.or_orthogonal.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _ord(o) -> int:
    return ORDER_NAMES[o] if isinstance(o, str) else int(o)


def distance(u: int, v: int) -> int:
    return lib().or_distance(u, v)


def weight(v: int) -> int:
    return lib().or_weight(v)


def order_table(ordering, n: int) -> np.ndarray:
    """table[r] = r-th vector of F_2^n in the ordering."""
    t = np.empty(1 << n, dtype=np.uint32)
    rc = lib().or_order_table(_ord(ordering), n, _p(t))
    if rc != 0:
        raise ValueError(f"or_order_table({ordering}, {n}) -> {rc}")
    return t


def hamming_bound(n: int, d: int) -> int:
    """Upper bound on M used to size output buffers (sphere packing; for even d
    the bound of (n-1, d-1)).  Exact integer arithmetic."""
    from math import comb
    if d % 2 == 0:
        n, d = n - 1, d - 1
    t = (d - 1) // 2
    vol = sum(comb(n, i) for i in range(t + 1))
    return max(1, (1 << n) // vol) if n >= 0 else 1


def greedy_plain(n: int, d: int, ordering="lex", nranks: int | None = None, table=None,
                 return_checks: bool = False):
    """O1: plain serial greedy, oldest-first, break on violation."""
    if table is None:
        table = order_table(ordering, n)
    N = 1 << n
    nranks = N if nranks is None else nranks
    cap = min(N, max(hamming_bound(n, d), 1)) if nranks == N else nranks
    out = np.empty(max(cap, 1), dtype=np.uint32)
    checks = ctypes.c_uint64(0)
    M = lib().or_greedy_plain(n, d, _p(table), nranks, _p(out), cap, ctypes.byref(checks))
    if M < 0:
        raise RuntimeError(f"or_greedy_plain -> {M}")
    res = out[:M].copy()
    return (res, checks.value) if return_checks else res


def greedy_plain_mt(n: int, d: int, ordering="lex", threads: int = 2, nranks: int | None = None,
                    table=None) -> np.ndarray:
    """O1 with the inner loop in `threads` sections (Fig. 2(b))."""
    if table is None:
        table = order_table(ordering, n)
    N = 1 << n
    nranks = N if nranks is None else nranks
    cap = min(N, max(hamming_bound(n, d), 1)) if nranks == N else nranks
    out = np.empty(max(cap, 1), dtype=np.uint32)
    M = lib().or_greedy_plain_mt(n, d, _p(table), nranks, int(threads), _p(out), cap)
    if M < 0:
        raise RuntimeError(f"or_greedy_plain_mt -> {M}")
    return out[:M].copy()


def greedy_ball(n: int, d: int, ordering="lex") -> np.ndarray:
    """O2: exact ball-marking restatement of the greedy (same output as O1)."""
    cap = min(1 << n, hamming_bound(n, d))
    out = np.empty(max(cap, 1), dtype=np.uint32)
    M = lib().or_greedy_ball(n, d, _ord(ordering), _p(out), cap)
    if M < 0:
        raise RuntimeError(f"or_greedy_ball -> {M}")
    return out[:M].copy()


def certify(n: int, d: int, ordering, words, table=None) -> tuple[bool, int]:
    """O3: True iff `words` is exactly the greedy output for (n, d, ordering).
    Returns (ok, why) with why in {0 ok, 1 rank order/distinct, 2 distance, 3 maximality}."""
    if table is None:
        table = order_table(ordering, n)
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32))
    why = ctypes.c_int(0)
    rc = lib().or_certify(n, d, _p(table), _p(w) if len(w) else None, len(w), ctypes.byref(why))
    if rc < 0:
        raise RuntimeError(f"or_certify -> {rc}")
    return bool(rc), why.value


def gf2_rank(words) -> int:
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32))
    return lib().or_gf2_rank(_p(w), len(w))


def is_linear(words) -> bool:
    """Linear <=> the (distinct) words fill the span: M == 2^rank."""
    return len(words) == (1 << gf2_rank(words))


def weight_distribution(words) -> dict:
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32))
    hist = (ctypes.c_uint64 * 33)()
    lib().or_weight_distribution(_p(w), len(w), hist)
    return {i: int(hist[i]) for i in range(33) if hist[i]}


def min_distance_pairs(words) -> int:
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32))
    return lib().or_min_distance_pairs(_p(w), len(w))


_SM1 = 0x9E3779B97F4A7C15
_SM2 = 0xBF58476D1CE4E5B9
_SM3 = 0x94D049BB133111EB
_M64 = (1 << 64) - 1


def set_digest(words) -> int:
    """Order-independent fingerprint: sum of splitmix64(v) mod 2^64."""
    v = np.asarray(words, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = v + np.uint64(_SM1)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_SM2)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_SM3)
        z = z ^ (z >> np.uint64(31))
        return int(z.sum(dtype=np.uint64))


SEQ_DIGEST_H0 = 1469598103934665603  # SURVEY A.3's decimal start value (0x14650fb0739d0383)


def seq_digest(words, h0: int = SEQ_DIGEST_H0) -> int:
    """Order-dependent fingerprint: FNV-style multiply over whole words, with the
    start value SURVEY A.3 used, so its Appendix A.1 table can be compared."""
    h = h0
    for v in np.asarray(words, dtype=np.uint64).tolist():
        h = ((h ^ v) * 0x100000001B3) & _M64
    return h


def w_def(n: int, ranks_of_accepted) -> int:
    """Definitional work of the paper's kernel: every candidate is compared
    with every codeword accepted before it (one thread per
    codeword).  = sum_j (2^n - 1 - p_j) over accepted ranks p_j."""
    p = np.asarray(ranks_of_accepted, dtype=np.int64)
    return int(((1 << n) - 1 - p).sum())


# ------------------------------------------------ SURVEY 8(f) extension rows

def order_table_basis(n: int, basis) -> np.ndarray:
    """B-ordering of PAPER.md:119-120 built by its recursive definition."""
    b = np.ascontiguousarray(np.asarray(basis, dtype=np.uint32))
    if len(b) != n:
        raise ValueError("basis must have n vectors")
    t = np.empty(1 << n, dtype=np.uint32)
    if lib().or_order_table_basis(n, _p(b), _p(t)) != 0:
        raise ValueError("basis is not linearly independent over F_2 (or out of range)")
    return t


def orthogonal(u: int, v: int) -> bool:
    return bool(lib().or_orthogonal(u, v))


def is_self_orthogonal(words) -> bool:
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32))
    return bool(lib().or_is_self_orthogonal(_p(w), len(w)))


def greedy_plain_ex(n, d, ordering="lex", constant_weight=-1, self_orthogonal=False, table=None, basis=None):
    """O1 with the constant-weight / self-orthogonal (:122-123) constraints,
    over any ordering (a name, a B-ordering basis, or a table)."""
    if table is None:
        table = order_table_basis(n, basis) if basis is not None else order_table(ordering, n)
    cap = min(1 << n, hamming_bound(n, d))
    out = np.empty(max(cap, 1), dtype=np.uint32)
    M = lib().or_greedy_plain_ex(n, d, _p(table), 1 << n, int(constant_weight), int(bool(self_orthogonal)),
                                 _p(out), cap)
    if M < 0:
        raise RuntimeError(f"or_greedy_plain_ex -> {M}")
    return out[:M].copy()


def greedy_ball_ex(n, d, ordering="lex", constant_weight=-1, self_orthogonal=False, table=None, basis=None):
    """O2 with the same constraints (ball map for distance, span basis for orthogonality)."""
    if table is None:
        table = order_table_basis(n, basis) if basis is not None else order_table(ordering, n)
    cap = min(1 << n, hamming_bound(n, d))
    out = np.empty(max(cap, 1), dtype=np.uint32)
    M = lib().or_greedy_ball_ex(n, d, _p(table), int(constant_weight), int(bool(self_orthogonal)), _p(out), cap)
    if M < 0:
        raise RuntimeError(f"or_greedy_ball_ex -> {M}")
    return out[:M].copy()


def greedy_cw64(n: int, d: int, w: int, ordering="lex", cap: int | None = None) -> np.ndarray:
    """Constant-weight greedy on 64-bit words, n <= 63: uint64 words in
    acceptance order.  Orderings: lex / glex (ascending value within the weight class), grlex."""
    from math import comb
    cap = comb(n, w) if cap is None else cap
    out = np.empty(max(cap, 1), dtype=np.uint64)
    M = lib().or_greedy_cw64(n, d, w, _ord(ordering), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), cap)
    if M < 0:
        raise RuntimeError(f"or_greedy_cw64 -> {M}")
    return out[:M].copy()
