# round-2 pass s: cross lists (prepared tiles record conflicts with the previous tiles' prepared
# lists): small-problem parity, then a parity-gated knob sweep (run under gpurun)
mkdir -p gpurun_out
PIPE_OPTS='[{}]' timeout 600 python tools/pipe_check.py 7,3,lex > gpurun_out/pipe_check_r02s.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02s.log
grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02s.log || exit 1
export KNOB_OPTS='[{"flags": 16384}, {}, {"prep_lead": 2}, {"prep_lead": 3}, {"prep_lead": 2, "prep_ctas": 3}, {"prep_lead": 3, "prep_ctas": 4}, {"prep_lead": 4, "prep_ctas": 4}]'
timeout 1500 python tools/knob_check.py 28,3,lex 24,3,lex 26,4,lex 26,4,glex 24,8,lex > gpurun_out/knob_r02s.log 2>&1
PROBE_OPTS='[{"prep_lead": 2}, {"prep_lead": 3, "prep_ctas": 4}]' timeout 600 python tools/phase_probe.py 28,3,lex > gpurun_out/phase_probe_r02s.log 2>&1
