"""Development check of the multi-rank pipelined engine with emulated ranks (one launch, one CTA
group per rank, peer stores between the groups' buffers) against the oracle, then timings per
rank count.  Run under gpurun with a timeout; not the bench contract."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
import paper_1507_05398_b200 as gc

bad = 0
for n, d, o in [(7, 3, "lex"), (10, 3, "gray"), (12, 4, "glex"), (14, 3, "grlex"), (16, 3, "lex"), (18, 5, "glex"),
                (20, 3, "gray"), (22, 3, "lex"), (24, 8, "lex")]:
    ref = O.greedy_ball(n, d, o)
    for G in (2, 4, 8):
        w, st = gc.gc_generate_ex(n, d, o, options={"emulate_ranks": G})
        ok = np.array_equal(w.astype(np.uint32), ref)
        bad += not ok
        print(json.dumps({"cfg": f"{n},{d},{o}", "G": G, "ok": ok, "M": int(st["M"]), "ref_M": len(ref),
                          "dev_ms": round(st["device_ms"], 3), "tiles": st["tiles"], "n_ranks": st["n_ranks"]}),
              flush=True)
print("RANKS_CHECK", "FAIL" if bad else "OK", flush=True)
if bad:
    sys.exit(1)
for n, d, o in [(24, 8, "lex"), (24, 3, "glex"), (26, 4, "glex"), (28, 3, "lex")]:
    for G in (1, 2, 4, 8):
        gc.gc_generate_ex(n, d, o, options={"emulate_ranks": G})
        w, st = gc.gc_generate_ex(n, d, o, options={"emulate_ranks": G})
        print(json.dumps({"cfg": f"{n},{d},{o}", "G": G, "M": st["M"], "dev_ms": round(st["device_ms"], 3),
                          "tiles": st["tiles"], "W_exec": f"{st['checks_exec']:.3e}",
                          "wait_ms": round(st["resolve_wait_ms"], 2), "busy_ms": round(st["resolve_busy_ms"], 2)}),
              flush=True)
