# round-2 first GPU pass: pipelined engine check, GPU tests, smoke, bench (run under gpurun)
mkdir -p gpurun_out
timeout 600 python tools/pipe_check.py > gpurun_out/pipe_check_r02a.log 2>&1; echo "pipe_check exit $?" >> gpurun_out/pipe_check_r02a.log
if grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02a.log; then
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02a.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02a.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_r02a.log 2>&1
fi
