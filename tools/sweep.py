"""Schedule sweep: device time, executed work and launches per (config, options) (development aid)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_05398_b200 as gc

def run(n, d, o, **opts):
    gc.gc_generate_ex(n, d, o, options=opts or None)
    w, st = gc.gc_generate_ex(n, d, o, options=opts or None)
    floor = st["M"] * (st["M"] - 1) / 2
    R = 148 * 16 * 1.965e9
    print(json.dumps({"cfg": f"{n},{d},{o}", "opts": opts, "dev_ms": round(st["device_ms"], 2),
                      "Wdef/s": f"{st['w_def'] / (st['device_ms'] * 1e-3):.3e}",
                      "Wexec/floor": round(st["checks_exec"] / max(floor, 1), 3),
                      "Wexec/s/R": round(st["checks_exec"] / (st["device_ms"] * 1e-3) / R, 3),
                      "surv/M": round(st["survivors"] / max(1, st["M"]), 3), "tiles": st["tiles"],
                      "levels": st["phases"], "launches": st["launches"]}), flush=True)

if __name__ == "__main__":
    spec = json.loads(sys.argv[1])
    for item in spec:
        n, d, o = item["cfg"]
        run(n, d, o, **item.get("opts", {}))
