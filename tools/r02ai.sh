# round-2 pass ai: deferred resolver counters, commit published at once again (run under gpurun)
# cross lists opt-in, catch-up default for graded orders (run under gpurun)
mkdir -p gpurun_out
timeout 120 python tools/dbg_case.py 20,3,lex '{"flags": 512}' > gpurun_out/dbg_r02ai.log 2>&1; echo "exit $?" >> gpurun_out/dbg_r02ai.log
PIPE_OPTS='[{}]' timeout 600 python tools/pipe_check.py 7,3,lex > gpurun_out/pipe_check_r02ai.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02ai.log
grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02ai.log || exit 1
export KNOB_OPTS='[{}, {"flags": 16384}, {"flags": 32768}]'
timeout 1500 python tools/knob_check.py 28,3,lex 24,3,lex 26,4,gray 26,4,lex 26,4,glex 24,8,lex 24,3,glex 28,3,gray > gpurun_out/knob_r02ai.log 2>&1
PROBE_OPTS='[{}, {"flags": 16384}]' timeout 600 python tools/phase_probe.py 28,3,lex > gpurun_out/phase_probe_r02ai.log 2>&1
