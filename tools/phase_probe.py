"""Per-tile phase breakdown of both persistent engines (GC_FLAG_DEBUG_PHASES on stderr) for a
few configs (development aid, run under gpurun; not the bench contract).
    python tools/phase_probe.py [n,d,ord ...]   env PROBE_OPTS='[{}, {"flags": 256}]'"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_05398_b200 as gc

cfgs = [(28, 3, "lex"), (24, 3, "lex"), (26, 4, "glex"), (24, 8, "lex")]
if len(sys.argv) > 1:
    cfgs = [tuple(int(x) if x.isdigit() else x for x in a.split(",")) for a in sys.argv[1:]]
opts_list = json.loads(os.environ.get("PROBE_OPTS", '[{}, {"flags": 256}]'))
for n, d, o in cfgs:
    for opts in opts_list:
        gc.gc_generate_ex(n, d, o, options=opts)                       # warm
        _, st = gc.gc_generate_ex(n, d, o, options=opts)
        o2 = dict(opts)
        o2["flags"] = o2.get("flags", 0) | gc.GC_FLAG_DEBUG_PHASES
        print(f"=== {n},{d},{o} {opts}: {st['device_ms']:.2f} ms, {st['tiles']} tiles (untimed run); debug run:",
              file=sys.stderr, flush=True)
        gc.gc_generate_ex(n, d, o, options=o2)
        sys.stderr.flush()
