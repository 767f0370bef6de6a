"""Small constructions for compute-sanitizer (memcheck / racecheck / synccheck): every engine
and the schedule corners that exercise the hand-rolled memory protocol (commit token, tile-slot
phases, fire-and-forget summary atomics, multi-chunk resolves).  Each result is compared with the
oracle so a sanitizer run is also a parity run.  Run under gpurun:
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
import paper_1507_05398_b200 as gc

CASES = [
    ((10, 3, "lex"), {}),                                       # pipelined engine (default)
    ((12, 4, "glex"), {}),
    ((12, 3, "gray"), {"grid_ctas": 3}),                        # resolver + preparing CTA + screening CTA
    ((12, 3, "lex"), {"pipeline_depth": 1}),
    ((12, 3, "lex"), {"pipeline_depth": 16, "tile_min": 32, "tile_max": 64}),   # ring reuse
    ((11, 3, "grlex"), {"tile_min": 32, "tile_max": 32, "window0": 32}),
    ((12, 2, "lex"), {"tile_min": 4096, "tile_max": 4096}),     # multi-chunk resolve and preparation
    ((12, 3, "lex"), {"flags": 0x800}),                         # no preparing CTAs
    ((12, 3, "gray"), {"emulate_ranks": 2}),                    # multi-rank pipeline: peer stores + flags
    ((12, 4, "glex"), {"emulate_ranks": 4, "tile_min": 32, "tile_max": 256}),
    ((10, 3, "lex"), {"flags": 0x100}),                         # tile-barrier engine (k_construct)
    ((12, 2, "lex"), {"flags": 0x100, "partial_s": 32}),        # partial tiles
    ((12, 3, "gray"), {"flags": 0x100, "emulate_ranks": 2}),    # tile-barrier partitioned path + k_resolve_tile
    ((12, 4, "glex"), {"flags": 0x10}),                         # launched engine
]
bad = 0
for (n, d, o), opts in CASES:
    w, st = gc.gc_generate_ex(n, d, o, options=opts)
    ok = np.array_equal(w.astype(np.uint32), O.greedy_plain(n, d, o))
    bad += not ok
    print(f"{n},{d},{o} {opts}: M={st['M']} {'ok' if ok else 'MISMATCH'}", flush=True)
for kw in (dict(ordering="lex", self_orthogonal=True), dict(ordering="glex", constant_weight=5)):
    w, st = gc.gc_construct(12, 4, **kw)
    ok = np.array_equal(w.astype(np.uint32), O.greedy_plain_ex(12, 4, **kw))
    bad += not ok
    print(f"12,4 {kw}: M={st['M']} {'ok' if ok else 'MISMATCH'}", flush=True)
# 64-bit constant-weight engine (n > 32)
for n, d, w, o in ((33, 4, 3, "lex"), (34, 6, 4, "grlex")):
    got, st = gc.gc_construct(n, d, ordering=o, constant_weight=w)
    ok = np.array_equal(got.astype(np.uint64), O.greedy_cw64(n, d, w, o))
    bad += not ok
    print(f"cw64 {n},{d},{w},{o}: M={st['M']} {'ok' if ok else 'MISMATCH'}", flush=True)
print("SANITIZE_CASES", "FAIL" if bad else "OK")
sys.exit(1 if bad else 0)
