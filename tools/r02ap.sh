# round-2 pass ap: tile-barrier engine vs pipelined on the n <= 26 lex / Gray rows; constant weight
# after excluding it from the graded defaults (run under gpurun)
mkdir -p gpurun_out
export KNOB_OPTS='[{}, {"flags": 256}]'
timeout 1500 python tools/knob_check.py 24,3,lex 24,3,gray 26,4,lex 26,4,gray 24,8,lex 28,3,lex 28,3,gray 24,3,glex 24,3,grlex 26,4,glex > gpurun_out/knob_r02ap.log 2>&1
timeout 300 python bench.py --workload 24,6,glex,cw=12 --no-cpu-baseline > gpurun_out/bench_cw_r02ap.log 2>&1
