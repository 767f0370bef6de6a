"""Quick per-config timing through gc_generate_ex (development aid, not the bench contract)."""
import sys, time, json
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1507_05398_b200 as gc

cfgs = [(7, 3, "lex"), (24, 8, "lex"), (20, 3, "lex"), (22, 3, "glex"), (24, 3, "lex"), (24, 3, "grlex"),
        (26, 4, "gray"), (26, 4, "glex"), (28, 3, "lex")]
if len(sys.argv) > 1:
    cfgs = [tuple(int(x) if x.isdigit() else x for x in a.split(",")) for a in sys.argv[1:]]
for n, d, o in cfgs:
    gc.gc_generate_ex(n, d, o)  # warm
    t = time.time()
    w, st = gc.gc_generate_ex(n, d, o)
    wall = time.time() - t
    R = 148 * 16 * 1.965e9
    print(json.dumps({"cfg": f"{n},{d},{o}", "M": st["M"], "wall_s": round(wall, 4), "dev_ms": round(st["device_ms"], 3),
                      "tiles": st["tiles"], "phases": st["phases"], "W_def/s": f"{st['w_def']/(st['device_ms']*1e-3):.3e}",
                      "W_exec": f"{st['checks_exec']:.3e}", "W_exec/s": f"{st['checks_exec']/(st['device_ms']*1e-3):.3e}",
                      "frac_popc": round(st['checks_exec']/(st['device_ms']*1e-3)/R, 3),
                      "surv/M": round(st["survivors"]/max(1,st["M"]), 2), "conf": st["conflicts"],
                      "res_chk": f"{st['resolve_checks']:.2e}"}), flush=True)
