# round-2 pass at: (24,8,lex) latency knobs (run under gpurun)
mkdir -p gpurun_out
export KNOB_OPTS='[{}, {"flags": 2048}, {"pipeline_depth": 12}, {"pipeline_depth": 16}, {"prep_ctas": 1}, {"tile_min": 1024}, {"flags": 1024}, {"window0": 4096, "window_growth": 12}]' KNOB_REPS=4
timeout 600 python tools/knob_check.py 24,8,lex > gpurun_out/knob_r02at.log 2>&1
PROBE_OPTS='[{}]' timeout 300 python tools/phase_probe.py 24,8,lex > gpurun_out/phase_probe_r02at.log 2>&1
