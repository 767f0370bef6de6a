# round-2 pass ah: deferred resolver counters + commit published under the next tile's loads;
# cross lists opt-in, catch-up default for graded orders (run under gpurun)
mkdir -p gpurun_out
timeout 120 python tools/dbg_case.py 20,3,lex '{"flags": 512}' > gpurun_out/dbg_r02ah.log 2>&1; echo "exit $?" >> gpurun_out/dbg_r02ah.log
PIPE_OPTS='[{}]' timeout 600 python tools/pipe_check.py 7,3,lex > gpurun_out/pipe_check_r02ah.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02ah.log
grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02ah.log || exit 1
export KNOB_OPTS='[{}, {"flags": 16384}, {"prep_lead": 2}]'
timeout 1500 python tools/knob_check.py 28,3,lex 24,3,lex 26,4,gray 26,4,lex 26,4,glex 24,8,lex 24,3,glex 28,3,gray > gpurun_out/knob_r02ah.log 2>&1
PROBE_OPTS='[{}, {"flags": 16384}]' timeout 600 python tools/phase_probe.py 28,3,lex > gpurun_out/phase_probe_r02ah.log 2>&1
