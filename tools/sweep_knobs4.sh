# follow-up: window sub-range knobs for Gray and graded orders at the r01l defaults (run under gpurun)
mkdir -p gpurun_out
G='[{"cfg":[26,4,"glex"]},{"cfg":[24,3,"grlex"]},{"cfg":[26,4,"gray"]},{"cfg":[24,3,"gray"]}]'
{
for kv in X=0 GC_SUB_MAX=131072 GC_SUB_MAX=524288 GC_GEO_HEAD=4096 GC_GEO_HEAD=16384 GC_GEO_HEAD=0 GC_SPLIT_BITS=16; do echo "== $kv"; env $kv timeout 120 python tools/sweep.py "$G"; done
} > gpurun_out/sweep_knobs4.log 2>&1
