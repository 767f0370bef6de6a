"""One construction with the given options (development aid for cuda-gdb runs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_05398_b200 as gc
n, d, o = sys.argv[1].split(",")
opts = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
w, st = gc.gc_generate_ex(int(n), int(d), o, options=opts)
print("ok", st["M"], st["tiles"])
