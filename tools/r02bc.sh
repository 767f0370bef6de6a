# round-2 pass bc: tile-size target re-sweep on the final engine (run under gpurun)
mkdir -p gpurun_out
export KNOB_OPTS='[{}, {"target_accepted": 256}, {"target_accepted": 320}, {"target_accepted": 448}, {"target_accepted": 512}, {"target_accepted": 640}]' KNOB_REPS=2
timeout 1500 python tools/knob_check.py 28,3,lex 28,3,gray 26,4,lex 26,4,gray > gpurun_out/knob_r02bc.log 2>&1
