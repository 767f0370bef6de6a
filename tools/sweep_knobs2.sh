# follow-up: tile-size target for graded and Gray orders (run under gpurun)
mkdir -p gpurun_out
G='[{"cfg":[26,4,"glex"]},{"cfg":[24,3,"grlex"]},{"cfg":[24,3,"glex"]},{"cfg":[20,3,"glex"]},{"cfg":[16,3,"grlex"]},{"cfg":[24,8,"glex"]}]'
Y='[{"cfg":[26,4,"gray"]},{"cfg":[24,3,"gray"]},{"cfg":[20,3,"gray"]},{"cfg":[26,4,"lex"]},{"cfg":[24,3,"lex"]},{"cfg":[24,8,"lex"]}]'
{
for t in 0 1536 2048 3072; do echo "== G $t"; if [ $t = 0 ]; then timeout 120 python tools/sweep.py "$G"; else GC_TARGET_ACCEPTED=$t timeout 120 python tools/sweep.py "$G"; fi; done
for t in 0 768 1024; do echo "== Y $t"; if [ $t = 0 ]; then timeout 120 python tools/sweep.py "$Y"; else GC_TARGET_ACCEPTED=$t timeout 120 python tools/sweep.py "$Y"; fi; done
} > gpurun_out/sweep_knobs2.log 2>&1
