"""Summarise ncu output into profiles/ (run here, on the CPU box, after a gpurun).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
      per-kernel share of the device time from an `ncu --metrics gpu__time_duration.sum --csv` log
  python tools/ncu_summary.py full <prof.ncu-rep> <out.md> [<out.json>]
      key metrics of a `--set full` capture (time, dram bytes, pipe utilisation, stall reasons)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def read_csv_text(text):
    lines = [l for l in text.splitlines() if l.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def launches(path, out):
    rows = read_csv_text(open(path).read())
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
        per[name][0] += 1
        per[name][1] += val * scale
    tot = sum(v[1] for v in per.values()) or 1.0
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary ({path})\n\n")
        f.write("Cold-cache, serialised per-launch times (ncu); compare SHARES with bench.py, not absolutes.\n\n")
        f.write("| kernel | launches | total us | share |\n|---|---|---|---|\n")
        for k, (n, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {k} | {n} | {us:.1f} | {100 * us / tot:.2f}% |\n")
    print(open(out).read())


METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
]


def full(rep, out, out_json=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = read_csv_text(txt)
    units = rows[0] if rows else {}
    res = []
    for r in rows[1:]:
        d = {"kernel": r.get("Kernel Name", "?").split("(")[0]}
        for m in METRICS:
            if m in r:
                d[m] = f"{r[m]} {units.get(m, '')}".strip()
        # every pipe-utilisation metric present
        for k, v in r.items():
            if k.startswith("sm__inst_executed_pipe_") and k.endswith("avg.pct_of_peak_sustained_active"):
                d[k] = f"{v} %"
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    if float(v.replace(",", "")) > 0:
                        d[k] = v
                except ValueError:
                    pass
        res.append(d)
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary ({rep})\n\n")
        for d in res:
            f.write(f"## {d['kernel']}\n\n| metric | value |\n|---|---|\n")
            for k, v in d.items():
                if k != "kernel":
                    f.write(f"| {k} | {v} |\n")
            f.write("\n")
    if out_json:
        json.dump(res, open(out_json, "w"), indent=1)
    print(open(out).read()[:6000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
