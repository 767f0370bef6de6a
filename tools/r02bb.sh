# round-2 measurement pass bb (final code of round 2): GPU tests, smoke, bench lines, reference arm,
# ncu launch list + full capture of k_pipeline, compute-sanitizer (run under gpurun)
mkdir -p gpurun_out
T=r02bb
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$T.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$T.log 2>&1
for w in 24,8,lex 26,4,glex 26,4,gray 26,4,lex 26,4,grlex 28,3,gray 28,3,glex 28,3,grlex 24,3,lex 24,3,gray 24,3,glex 24,3,grlex 22,6,lex,so 24,6,glex,cw=12 24,8,lex,basis=seed:1 7,3,lex; do timeout 300 python bench.py --workload $w --no-cpu-baseline >> gpurun_out/bench_${T}_others.log 2>&1; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$T.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --warmup 1 --steps 2 --no-cpu-baseline > gpurun_out/launches_bench_$T.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pipeline -c 1 -o gpurun_out/prof_28_3_full_$T python tools/quick_bench.py 28,3,lex > gpurun_out/ncu_full_$T.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$T.log
PROBE_OPTS="[{}]" timeout 900 python tools/phase_probe.py 28,3,lex 26,4,glex 24,8,lex > gpurun_out/phase_probe_$T.log 2>&1
