mkdir -p gpurun_out
PROBE_OPTS='[{}]' timeout 600 python tools/phase_probe.py 28,3,lex 24,3,lex > gpurun_out/phase_probe_r02n.log 2>&1
