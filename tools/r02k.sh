# round-2 pass k: early round break only for many undecided (run under gpurun)
mkdir -p gpurun_out
export PIPE_OPTS='[{}]'
timeout 1200 python tools/pipe_check.py 24,8,lex 24,3,lex 24,3,gray 24,3,glex 26,4,gray 26,4,lex 26,4,glex 28,3,lex 28,3,gray > gpurun_out/pipe_check_r02k.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02k.log
PROBE_OPTS='[{}]' timeout 600 python tools/phase_probe.py 28,3,lex 24,3,lex > gpurun_out/phase_probe_r02k.log 2>&1
