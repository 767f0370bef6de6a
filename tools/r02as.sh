# round-2 pass as: two-stage preparation without cross lists (GC_FLAG_STAGE_B): parity + lead sweep (run under gpurun)
mkdir -p gpurun_out
timeout 120 python tools/dbg_case.py 26,3,lex '{"flags": 262656}' > gpurun_out/dbg_r02as.log 2>&1; echo "exit $?" >> gpurun_out/dbg_r02as.log
PIPE_OPTS='[{}]' timeout 600 python tools/pipe_check.py 7,3,lex > gpurun_out/pipe_check_r02as.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02as.log
grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02as.log || exit 1
export KNOB_OPTS='[{}, {"flags": 262144}, {"flags": 262144, "prep_lead": 2}, {"flags": 262144, "prep_lead": 4}, {"flags": 262144, "prep_lead": 6, "prep_ctas": 4}]'
timeout 1500 python tools/knob_check.py 28,3,lex 28,3,gray 26,4,lex 26,4,gray 26,4,glex 24,8,lex > gpurun_out/knob_r02as.log 2>&1
PROBE_OPTS='[{"flags": 262144}, {"flags": 262144, "prep_lead": 4}]' timeout 600 python tools/phase_probe.py 28,3,lex > gpurun_out/phase_probe_r02as.log 2>&1
