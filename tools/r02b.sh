# round-2 pass b: phase breakdown of both engines, GPU tests, bench with the parity gate (run under gpurun)
mkdir -p gpurun_out
timeout 600 python tools/phase_probe.py > gpurun_out/phase_probe_r02b.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02b.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02b.log
timeout 600 python bench.py > gpurun_out/bench_r02b.log 2>&1
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_r02b.log 2>&1
