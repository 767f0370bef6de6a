# round-2 pass d: pipelined engine with emulated ranks (peer stores), then parity + GPU tests (run under gpurun)
mkdir -p gpurun_out
timeout 600 python tools/ranks_check.py > gpurun_out/ranks_check_r02d.log 2>&1; echo "exit $?" >> gpurun_out/ranks_check_r02d.log
export PIPE_OPTS='[{}]'
timeout 600 python tools/pipe_check.py 24,8,lex 24,3,lex 24,3,gray 24,3,glex 24,3,grlex 26,4,gray 26,4,glex 28,3,lex > gpurun_out/pipe_check_r02d.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02d.log
if grep -q "RANKS_CHECK OK" gpurun_out/ranks_check_r02d.log; then
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02d.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02d.log
fi
