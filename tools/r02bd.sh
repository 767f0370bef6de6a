# round-2 pass bd: Gray tile target 448 on the pipelined engine; bench lines for the Gray rows (run under gpurun)
mkdir -p gpurun_out
export KNOB_OPTS='[{}]' KNOB_REPS=2
timeout 900 python tools/knob_check.py 28,3,gray 26,4,gray 24,3,gray > gpurun_out/knob_r02bd.log 2>&1
for w in 28,3,gray 26,4,gray; do timeout 300 python bench.py --workload $w --no-cpu-baseline >> gpurun_out/bench_r02bd_gray.log 2>&1; done
timeout 1200 python -m pytest tests -m gpu -q -x -k "gray" > gpurun_out/pytest_r02bd.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r02bd.log
