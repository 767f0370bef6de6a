# round-2 pass l: small-tail fallback, parity-refined block bound (run under gpurun)
mkdir -p gpurun_out
export PIPE_OPTS='[{}, {"flags": 8192}]'
timeout 1500 python tools/pipe_check.py 24,8,lex 24,3,lex 24,3,gray 24,3,glex 24,3,grlex 26,4,gray 26,4,lex 26,4,glex 28,3,lex 28,3,gray > gpurun_out/pipe_check_r02l.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02l.log
PROBE_OPTS='[{}]' timeout 600 python tools/phase_probe.py 28,3,lex 24,3,lex > gpurun_out/phase_probe_r02l.log 2>&1
if grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02l.log; then
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02l.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02l.log
fi
