# round-2 pass f: GPU tests (64-bit constant-weight engine, race-free rounds), compute-sanitizer (run under gpurun)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02f.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02f.log
bash tools/r02_sanitize.sh
export PIPE_OPTS='[{}]'
timeout 600 python tools/pipe_check.py 24,8,lex 24,3,lex 26,4,glex 28,3,lex > gpurun_out/pipe_check_r02f.log 2>&1
