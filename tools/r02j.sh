# round-2 pass j: burst sub-chunks, adaptive rounds, read-ahead of the next prep word (run under gpurun)
mkdir -p gpurun_out
export PIPE_OPTS='[{}, {"burst_chunk": 256}, {"burst_chunk": 1024}, {"burst_chunk": 2048}]'
timeout 1200 python tools/pipe_check.py 24,3,lex 24,3,gray 26,4,gray 26,4,lex 26,4,glex 28,3,lex 28,3,gray > gpurun_out/pipe_check_r02j.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02j.log
if grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02j.log; then
PROBE_OPTS='[{}]' timeout 600 python tools/phase_probe.py 28,3,lex 24,3,lex 26,4,gray > gpurun_out/phase_probe_r02j.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02j.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02j.log
fi
