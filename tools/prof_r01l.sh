# ncu launch list + full capture of k_construct for the r01l build (run under gpurun)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01l.csv python bench.py --warmup 1 --steps 2 --no-cpu-baseline > gpurun_out/launches_bench_r01l.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_construct -c 1 -o gpurun_out/prof_28_3_full_r01l python tools/quick_bench.py 28,3,lex > gpurun_out/ncu_full_r01l.log 2>&1
