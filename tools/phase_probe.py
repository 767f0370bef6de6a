"""Per-phase screen work for a few (config, tile_max, window0) settings (development aid)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GC_DEBUG_PHASES"] = "1"
import paper_1507_05398_b200 as gc
runs = [((28, 3, "lex"), 65536, 1024), ((28, 3, "lex"), 16384, 1024), ((28, 3, "lex"), 4096, 1024),
        ((28, 3, "lex"), 65536, 256), ((26, 4, "glex"), 65536, 1024), ((26, 4, "glex"), 8192, 1024),
        ((24, 8, "lex"), 65536, 1024), ((24, 8, "lex"), 4096, 4096)]
for (n, d, o), tmax, w0 in runs:
    print(f"=== {n},{d},{o} tile_max={tmax} window0={w0}", flush=True)
    w, st = gc.gc_generate_ex(n, d, o, options={"tile_max": tmax, "window0": w0})
    floor = st["M"] * (st["M"] - 1) / 2
    print(json.dumps({"dev_ms": round(st["device_ms"], 1), "W_exec/floor": round(st["checks_exec"] / floor, 3),
                      "surv/M": round(st["survivors"] / st["M"], 3), "tiles": st["tiles"], "launches": st["launches"],
                      "conflicts": st["conflicts"], "res_chk": st["resolve_checks"]}), flush=True)
