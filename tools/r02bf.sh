# round-2 pass bf: full GPU test suite + smoke on the final code (run under gpurun)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02bf.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02bf.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02bf.log
timeout 600 python bench.py > gpurun_out/bench_r02bf.log 2>&1
