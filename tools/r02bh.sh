# round-2 pass bh: one dedicated preparing CTA (the other screens) (run under gpurun)
mkdir -p gpurun_out
export KNOB_OPTS='[{}, {"prep_ctas": 1}]' KNOB_REPS=3
timeout 1200 python tools/knob_check.py 28,3,lex 28,3,gray 26,4,lex 26,4,glex 24,8,lex > gpurun_out/knob_r02bh.log 2>&1
