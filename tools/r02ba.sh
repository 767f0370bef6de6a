# round-2 pass au: preparation stages its newest words during the gather (run under gpurun)
mkdir -p gpurun_out
timeout 120 python tools/dbg_case.py 26,3,lex '{"flags": 512}' > gpurun_out/dbg_r02ba.log 2>&1; echo "exit $?" >> gpurun_out/dbg_r02ba.log
PIPE_OPTS='[{}]' timeout 600 python tools/pipe_check.py 7,3,lex > gpurun_out/pipe_check_r02ba.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02ba.log
grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02ba.log || exit 1
export KNOB_OPTS='[{}]' KNOB_REPS=3
timeout 1500 python tools/knob_check.py 28,3,lex 24,8,lex 26,4,glex 26,4,gray 26,4,lex 28,3,gray 24,3,glex 28,3,glex > gpurun_out/knob_r02ba.log 2>&1
PROBE_OPTS='[{}]' timeout 600 python tools/phase_probe.py 28,3,lex 24,8,lex > gpurun_out/phase_probe_r02ba.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -k "parity or knobs or next_rows or schedule" > gpurun_out/pytest_r02ba.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r02ba.log
