"""Write tests/golden/bench_golden.json: the expected output of every bench workload, computed
by the oracle alone (O2, oracle/greedy_oracle.c `or_greedy_ball[_ex]`, the exact ball-marking
restatement of the greedy of PAPER.md:59).  bench.py's parity gate and the GPU tests read the
file; nothing here touches the CUDA path.

    python tools/gen_bench_golden.py [-j 8]
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as WL  # noqa: E402


def one(wl):
    import numpy as np
    import oracle as O
    n, d, o, ex = WL.parse_workload(wl)
    t = time.time()
    if ex:
        w = O.greedy_ball_ex(n, d, o, **ex)
    else:
        w = O.greedy_ball(n, d, o)
    dt = time.time() - t
    row = {"workload": wl, "n": n, "d": d, "order": o, "M": int(len(w)),
           "set_digest": format(WL.set_digest(w), "016x"), "seq_digest": format(WL.seq_digest(w), "016x"),
           "last": int(w[-1]) if len(w) else None, "oracle": "O2" + ("_ex" if ex else ""),
           "oracle_s": round(dt, 2)}
    if not ex:
        # W_def = sum_j (2^n - 1 - rank_j); ranks from the oracle's own
        # order table (PAPER.md:116 orderings by their definitions), inverted by a scatter
        table = O.order_table(o, n)
        inv = np.empty(1 << n, dtype=np.uint32)
        inv[table] = np.arange(1 << n, dtype=np.uint32)
        ranks = inv[w].astype(np.int64)
        del table, inv
        row["w_def"] = int(((1 << n) - 1 - ranks).sum())
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=os.cpu_count())
    args = ap.parse_args()
    with ProcessPoolExecutor(args.j) as ex:
        rows = list(ex.map(one, WL.BENCH_WORKLOADS))
    out = {"source": "tools/gen_bench_golden.py: oracle O2 (oracle/greedy_oracle.c) only; digests as in "
                     "workloads.py (SURVEY.md A.3)", "rows": rows}
    p = os.path.join(ROOT, "tests", "golden", "bench_golden.json")
    json.dump(out, open(p, "w"), indent=1)
    for r in rows:
        print(r)


if __name__ == "__main__":
    main()
