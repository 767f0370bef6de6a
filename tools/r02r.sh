# round-2 pass r: per-tile phase breakdown of the current pipelined engine (run under gpurun)
mkdir -p gpurun_out
PROBE_OPTS='[{}]' timeout 900 python tools/phase_probe.py 28,3,lex 26,4,glex 24,3,lex 28,3,glex 24,8,lex > gpurun_out/phase_probe_r02r.log 2>&1
