# follow-up: lex window sub-range knobs, repeated (run under gpurun)
mkdir -p gpurun_out
L='[{"cfg":[28,3,"lex"]},{"cfg":[28,3,"lex"]},{"cfg":[26,4,"lex"]},{"cfg":[24,3,"lex"]}]'
{
for kv in X=0 GC_SUB_MAX=262144 GC_SUB_MAX=524288 GC_GEO_HEAD=8192 "GC_SUB_MAX=262144 GC_GEO_HEAD=8192" X=1 GC_TARGET_ACCEPTED=320 GC_TARGET_ACCEPTED=448; do echo "== $kv"; env $kv timeout 120 python tools/sweep.py "$L"; done
} > gpurun_out/sweep_knobs3.log 2>&1
