# round-2 pass ar: fence.acq_rel.gpu instead of fence.sc.gpu in the pipelined engine (run under gpurun)
mkdir -p gpurun_out
PIPE_OPTS='[{}]' timeout 600 python tools/pipe_check.py 7,3,lex > gpurun_out/pipe_check_r02ar.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02ar.log
grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02ar.log || exit 1
export KNOB_OPTS='[{}]' KNOB_REPS=3
timeout 1500 python tools/knob_check.py 28,3,lex 24,8,lex 26,4,glex 26,4,gray 26,4,lex 28,3,gray 24,3,glex > gpurun_out/knob_r02ar.log 2>&1
PROBE_OPTS='[{}]' timeout 600 python tools/phase_probe.py 28,3,lex > gpurun_out/phase_probe_r02ar.log 2>&1
