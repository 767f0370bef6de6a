"""Development check of the default (pipelined) engine on small problems against the oracle O2,
then per-config timings of both persistent engines.  Run under gpurun; not the bench contract."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import oracle as O
import paper_1507_05398_b200 as gc

bad = 0
for n, d, o in [(3, 2, "lex"), (7, 3, "lex"), (10, 3, "gray"), (12, 4, "glex"), (14, 3, "grlex"), (16, 3, "lex"),
                (18, 5, "glex"), (20, 3, "gray"), (20, 4, "grlex"), (22, 3, "lex"), (24, 8, "lex")]:
    t = time.time()
    w, st = gc.gc_generate_ex(n, d, o)
    dt = time.time() - t
    ref = O.greedy_ball(n, d, o)
    ok = np.array_equal(w.astype(np.uint32), ref)
    bad += not ok
    print(json.dumps({"cfg": f"{n},{d},{o}", "ok": ok, "M": int(st["M"]), "ref_M": len(ref), "wall_s": round(dt, 4),
                      "dev_ms": round(st["device_ms"], 3), "tiles": st["tiles"], "wait_ms": round(st["resolve_wait_ms"], 3),
                      "busy_ms": round(st["resolve_busy_ms"], 3)}), flush=True)
print("PIPE_CHECK", "FAIL" if bad else "OK", flush=True)
if bad:
    sys.exit(1)
cfgs = [(24, 8, "lex"), (24, 3, "lex"), (24, 3, "gray"), (24, 3, "glex"), (24, 3, "grlex"), (26, 4, "gray"),
        (26, 4, "glex"), (28, 3, "lex")]
if len(sys.argv) > 1:
    cfgs = [tuple(int(x) if x.isdigit() else x for x in a.split(",")) for a in sys.argv[1:]]
opts_list = json.loads(os.environ.get("PIPE_OPTS", '[{}, {"flags": 256}]'))
for n, d, o in cfgs:
    for opts in opts_list:
        gc.gc_generate_ex(n, d, o, options=opts)
        best = None
        for _ in range(2):
            w, st = gc.gc_generate_ex(n, d, o, options=opts)
            if best is None or st["device_ms"] < best["device_ms"]:
                best = st
        st = best
        print(json.dumps({"cfg": f"{n},{d},{o}", "opts": opts, "M": st["M"], "dev_ms": round(st["device_ms"], 3),
                          "tiles": st["tiles"], "levels": st["phases"], "W_exec": f"{st['checks_exec']:.3e}",
                          "tests": f"{st['bound_tests']:.3e}", "surv/M": round(st["survivors"] / max(1, st["M"]), 3),
                          "res_chk": f"{st['resolve_checks']:.2e}", "wait_ms": round(st["resolve_wait_ms"], 2),
                          "busy_ms": round(st["resolve_busy_ms"], 2),
                          "us_per_tile": round(1e3 * st["device_ms"] / max(1, st["tiles"]), 2)}), flush=True)
