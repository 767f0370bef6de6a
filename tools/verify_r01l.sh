# verification after the tile-target change (run under gpurun)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01l.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r01l.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r01l.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_r01l.log 2>&1
for w in 24,8,lex 26,4,glex 26,4,gray 26,4,lex 24,3,lex 24,3,gray 24,3,glex 24,3,grlex 22,6,lex,so 24,6,glex,cw=12 24,8,lex,basis=seed:1 7,3,lex; do timeout 200 python bench.py --workload $w --no-cpu-baseline >> gpurun_out/bench_r01l_others.log 2>&1; done
