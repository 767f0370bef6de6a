"""Top source lines by warp-stall samples (development aid).

  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = None, None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        hdr = None
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:          # CUDA line rows (SASS rows have no line no)
        d = dict(zip(hdr, r))
        d["Source"] = r[1]
        try:
            smp = int(d["Warp Stall Sampling (All Samples)"])
        except ValueError:
            continue
        if smp:
            stalls = {k: int(v) for k, v in d.items()
                      if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
            top3 = sorted(stalls.items(), key=lambda x: -x[1])[:3]
            out.append((smp, fname, d["Line No"], d["Source"].strip()[:70], top3))
tot = sum(o[0] for o in out)
print("total samples", tot)
for smp, f, ln, src, t3 in sorted(out, reverse=True)[:top]:
    print(f"{100 * smp / tot:5.1f}% {f}:{ln:5s} {src:70s} {' '.join(f'{k[6:]}={v}' for k, v in t3)}")
