# round-2 pass m: ballot-driven per-node tail; racecheck; GPU tests (run under gpurun)
mkdir -p gpurun_out
export PIPE_OPTS='[{}]'
timeout 1500 python tools/pipe_check.py 24,8,lex 24,3,lex 24,3,gray 24,3,glex 24,3,grlex 26,4,gray 26,4,lex 26,4,glex 28,3,lex 28,3,gray > gpurun_out/pipe_check_r02p.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02p.log
PROBE_OPTS='[{}]' timeout 600 python tools/phase_probe.py 28,3,lex 24,3,lex > gpurun_out/phase_probe_r02p.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck_r02p.log 2>&1; echo "exit $?" >> gpurun_out/sanitize_racecheck_r02p.log
if grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02p.log; then
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02p.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02p.log
fi
