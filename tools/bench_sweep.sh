#!/bin/bash
# One bench.py line per workload (short runs) -> gpurun_out/workloads.jsonl
mkdir -p gpurun_out
out=gpurun_out/workloads.jsonl
: > $out
for w in "7,3,lex" "24,8,lex" "24,8,gray" "24,8,glex" "24,8,grlex" "16,3,lex" "20,3,gray" "22,3,glex" "24,3,lex" "24,3,gray" "24,3,glex" "24,3,grlex" \
         "26,4,gray" "26,4,glex" "23,7,lex" "22,6,lex,so" "24,8,lex,so" "24,8,lex,basis=seed:1" "26,4,lex,basis=gray" "24,6,glex,cw=12" "26,4,lex,cw=13"; do
  timeout 300 python bench.py --workload "$w" --steps 3 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 >> $out
done
cat $out | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(f\"{d['config']['workload']:>24s}  {d['ms_per_step']:10.3f} ms  value {d['value']:.3e}  M={d['config']['M']}  roofline {d['roofline']['frac']:.3f}\")
"
