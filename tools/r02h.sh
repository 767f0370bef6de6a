# round-2 pass h: resolver breakdown on prepared tiles (run under gpurun)
mkdir -p gpurun_out
PROBE_OPTS='[{}]' timeout 600 python tools/phase_probe.py 28,3,lex 24,3,lex 26,4,gray 24,8,lex > gpurun_out/phase_probe_r02h.log 2>&1
