"""Knob sweep with a parity gate: every (workload, options) run is compared with the O2 golden
digests (tests/golden/bench_golden.json: M, set and sequence digests) before its time is printed.
Development aid, run under gpurun; not the bench contract.
    KNOB_OPTS='[{}, {"flags": 16384}]' python tools/knob_check.py 28,3,lex 26,4,glex ..."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_1507_05398_b200 as gc
from workloads import parse_workload, seq_digest, set_digest

rows = {r["workload"]: r for r in json.load(open(os.path.join(ROOT, "tests", "golden", "bench_golden.json")))["rows"]}
opts_list = json.loads(os.environ.get("KNOB_OPTS", "[{}]"))
reps = int(os.environ.get("KNOB_REPS", "2"))
bad = 0
for wl in sys.argv[1:]:
    n, d, o = wl.split(",")[:3]
    n, d = int(n), int(d)
    g = rows[wl]
    for opts in opts_list:
        best = None
        for _ in range(reps + 1):
            w, st = gc.gc_generate_ex(n, d, o, options=opts)
            if best is None or st["device_ms"] < best[1]["device_ms"]:
                best = (w, st)
        w, st = best
        w = np.asarray(w, dtype=np.uint64)
        ok = (len(w) == g["M"] and f"{set_digest(w):016x}" == g["set_digest"] and f"{seq_digest(w):016x}" == g["seq_digest"])
        bad += not ok
        print(json.dumps({"cfg": wl, "opts": opts, "parity": ok, "dev_ms": round(st["device_ms"], 2),
                          "tiles": st["tiles"], "wait_ms": round(st["resolve_wait_ms"], 1),
                          "busy_ms": round(st["resolve_busy_ms"], 1), "prep_used": st.get("prep_used"),
                          "us_per_tile": round(1e3 * st["device_ms"] / max(1, st["tiles"]), 2)}), flush=True)
print("KNOB_CHECK", "FAIL" if bad else "OK", flush=True)
sys.exit(1 if bad else 0)
