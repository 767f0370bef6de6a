# round-2 pass af: stage-A breakdown, catch-up on / off (run under gpurun)
mkdir -p gpurun_out
PROBE_OPTS='[{"flags": 16384}, {"flags": 49152}]' timeout 600 python tools/phase_probe.py 28,3,lex 24,3,lex > gpurun_out/phase_probe_r02af.log 2>&1
