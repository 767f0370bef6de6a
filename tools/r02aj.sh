# round-2 pass aj: GPU tests (cross lists / catch-up level schedules added), default vs knobs (run under gpurun)
mkdir -p gpurun_out
timeout 120 python tools/dbg_case.py 20,3,lex '{"flags": 512}' > gpurun_out/dbg_r02aj.log 2>&1; echo "exit $?" >> gpurun_out/dbg_r02aj.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02aj.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02aj.log
export KNOB_OPTS='[{}, {"flags": 32768}, {"flags": 65536}]'
timeout 1500 python tools/knob_check.py 28,3,lex 24,3,lex 26,4,gray 26,4,lex 26,4,glex 26,4,grlex 24,8,lex 24,3,glex 24,3,grlex 28,3,glex > gpurun_out/knob_r02aj.log 2>&1
