# round-1 profile pass (run under gpurun): launch list, full capture of k_construct, bench line, sweep
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG:-r01j}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG:-r01j}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke_${TAG:-r01j}.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG:-r01j}.csv python bench.py --warmup 1 --steps 2 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_construct -c 1 -o gpurun_out/prof_28_3_full_${TAG:-r01j} python tools/quick_bench.py 28,3,lex > gpurun_out/ncu_full.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_${TAG:-r01j}.log 2>&1
for w in 24,8,lex 26,4,glex 26,4,gray 26,4,lex 24,3,lex 24,3,gray 24,3,glex 24,3,grlex 22,6,lex,so 24,6,glex,cw=12 24,8,lex,basis=seed:1 7,3,lex; do timeout 200 python bench.py --workload $w --no-cpu-baseline >> gpurun_out/bench_${TAG:-r01j}_others.log 2>&1; done
GC_DEBUG_PHASES=1 timeout 100 python tools/sweep.py '[{"cfg":[28,3,"lex"]}]' > gpurun_out/phases_${TAG:-r01j}.log 2>&1
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref_${TAG:-r01j}.log 2>&1
