# round-2 pass ak: prepared bursts decided in sub-chunks; (24,8) tile-size knobs (run under gpurun)
mkdir -p gpurun_out
timeout 120 python tools/dbg_case.py 20,3,lex '{"flags": 512}' > gpurun_out/dbg_r02ak.log 2>&1; echo "exit $?" >> gpurun_out/dbg_r02ak.log
PIPE_OPTS='[{}]' timeout 600 python tools/pipe_check.py 7,3,lex > gpurun_out/pipe_check_r02ak.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02ak.log
grep -q "PIPE_CHECK OK" gpurun_out/pipe_check_r02ak.log || exit 1
export KNOB_OPTS='[{}, {"burst_chunk": 256}, {"burst_chunk": 1024}, {"burst_chunk": 128}]'
timeout 1500 python tools/knob_check.py 28,3,lex 24,3,lex 24,3,gray 26,4,gray 26,4,lex 26,4,glex 28,3,gray > gpurun_out/knob_r02ak.log 2>&1
export KNOB_OPTS='[{}, {"target_accepted": 2048}, {"target_accepted": 8192}, {"tile_min": 2048}, {"pipeline_depth": 4}, {"prep_lead": 2}]'
timeout 600 python tools/knob_check.py 24,8,lex > gpurun_out/knob24_r02ak.log 2>&1
PROBE_OPTS='[{}]' timeout 600 python tools/phase_probe.py 28,3,lex 24,3,lex > gpurun_out/phase_probe_r02ak.log 2>&1
