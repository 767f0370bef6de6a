# round-2 pass ab: early preparations (lists published before the cross step, tiles picked in order,
# cross lists against up to 7 earlier lists): parity-gated lead sweep + phase probes (run under gpurun)
mkdir -p gpurun_out
timeout 120 python tools/dbg_case.py 20,3,lex '{"flags": 512}' > gpurun_out/dbg_r02ab.log 2>&1; echo "exit $?" >> gpurun_out/dbg_r02ab.log
PIPE_OPTS='[{}]' timeout 600 python tools/pipe_check.py 7,3,lex > gpurun_out/pipe_check_r02ab.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02ab.log
grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02ab.log || exit 1
export KNOB_OPTS='[{}, {"prep_lead": 2}, {"prep_lead": 3, "prep_ctas": 3}, {"prep_lead": 4, "prep_ctas": 4}, {"prep_lead": 6, "prep_ctas": 4}, {"prep_lead": 6, "prep_ctas": 8}]'
timeout 1500 python tools/knob_check.py 28,3,lex 24,3,lex 26,4,lex 26,4,glex > gpurun_out/knob_r02ab.log 2>&1
PROBE_OPTS='[{"prep_lead": 4, "prep_ctas": 4}, {"prep_lead": 6, "prep_ctas": 8}]' timeout 600 python tools/phase_probe.py 28,3,lex > gpurun_out/phase_probe_r02ab.log 2>&1
