# round-2 pass ac: what the resolver finds on arrival (screen latency vs preparation) (run under gpurun)
mkdir -p gpurun_out
PROBE_OPTS='[{"prep_lead": 1}, {"prep_lead": 4, "prep_ctas": 4}, {"prep_lead": 6, "prep_ctas": 4, "pipeline_depth": 12}, {"flags": 16384}]' timeout 900 python tools/phase_probe.py 28,3,lex 26,4,glex > gpurun_out/phase_probe_r02ac.log 2>&1
