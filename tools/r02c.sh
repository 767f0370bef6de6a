# round-2 pass c: the prep stage of the pipelined engine -- parity first, then phase breakdown (run under gpurun)
mkdir -p gpurun_out
export PIPE_OPTS='[{}, {"pipeline_depth": 6}, {"pipeline_depth": 8}, {"pipeline_depth": 12}]'
timeout 900 python tools/pipe_check.py 24,8,lex 24,3,lex 24,3,glex 26,4,glex 28,3,lex > gpurun_out/pipe_check_r02c.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02c.log
if grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02c.log; then
PROBE_OPTS='[{}, {"pipeline_depth": 8}]' timeout 600 python tools/phase_probe.py > gpurun_out/phase_probe_r02c.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02c.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02c.log
fi
