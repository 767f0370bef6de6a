# round-2 pass an: confirm graded defaults (sub-range 32768; depth 8 vs 10), 5 repetitions each (run under gpurun)
mkdir -p gpurun_out
export KNOB_REPS=5
export KNOB_OPTS='[{"sub_max": 32768}, {"sub_max": 32768, "pipeline_depth": 10}, {"sub_max": 32768, "pipeline_depth": 9}]'
timeout 1800 python tools/knob_check.py 26,4,glex 26,4,grlex 24,3,glex 24,3,grlex 28,3,glex 28,3,grlex > gpurun_out/knob_r02an.log 2>&1
