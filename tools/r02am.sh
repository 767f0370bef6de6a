# round-2 pass am: graded-order screen knobs (sub-range length, depth) (run under gpurun)
mkdir -p gpurun_out
export KNOB_OPTS='[{}, {"sub_max": 32768}, {"sub_max": 16384}, {"sub_max": 32768, "pipeline_depth": 10}, {"sub_max": 16384, "pipeline_depth": 12}, {"sub_max": 8192}]'
timeout 1800 python tools/knob_check.py 26,4,glex 26,4,grlex 24,3,glex 24,3,grlex 28,3,glex > gpurun_out/knob_r02am.log 2>&1
