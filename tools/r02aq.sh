# round-2 pass aq: default engine choice (tile-barrier for d = 3 lex / Gray, n <= 25): GPU tests, timings (run under gpurun)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02aq.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_r02aq.log
export KNOB_OPTS='[{}, {"flags": 131072}]'
timeout 900 python tools/knob_check.py 24,3,lex 24,3,gray 28,3,lex 26,4,lex > gpurun_out/knob_r02aq.log 2>&1
timeout 600 python tools/sweep.py '[{"cfg": [16,3,"lex"]}, {"cfg": [16,3,"lex"], "opts": {"flags": 131072}}, {"cfg": [20,3,"lex"]}, {"cfg": [20,3,"lex"], "opts": {"flags": 131072}}, {"cfg": [22,3,"gray"]}, {"cfg": [22,3,"gray"], "opts": {"flags": 131072}}, {"cfg": [25,3,"lex"]}, {"cfg": [25,3,"lex"], "opts": {"flags": 131072}}, {"cfg": [26,3,"lex"]}, {"cfg": [26,3,"lex"], "opts": {"flags": 256}}]' > gpurun_out/sweep_r02aq.log 2>&1
