# round-2 pass bg: preparation lead / two-stage preparation re-check on the final code (run under gpurun)
mkdir -p gpurun_out
export KNOB_OPTS='[{}, {"prep_lead": 2}, {"flags": 262144, "prep_lead": 2}, {"flags": 262144}, {"prep_ctas": 3}]' KNOB_REPS=2
timeout 1500 python tools/knob_check.py 28,3,lex 28,3,gray 26,4,lex 26,4,gray > gpurun_out/knob_r02bg.log 2>&1
