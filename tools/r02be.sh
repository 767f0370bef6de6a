# round-2 pass be: graded-order tile target re-sweep on the final engine (run under gpurun)
mkdir -p gpurun_out
export KNOB_OPTS='[{}, {"target_accepted": 768}, {"target_accepted": 1024}, {"target_accepted": 2048}, {"target_accepted": 3072}]' KNOB_REPS=2
timeout 2000 python tools/knob_check.py 26,4,glex 26,4,grlex 24,3,glex 24,3,grlex 28,3,glex > gpurun_out/knob_r02be.log 2>&1
