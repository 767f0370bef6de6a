# round-2 pass al: screen-latency knobs for the pipelined engine (run under gpurun)
mkdir -p gpurun_out
export KNOB_OPTS='[{}, {"sub_max": 131072}, {"sub_max": 65536}, {"sub_max": 32768}, {"items_per_warp": 2}, {"geo_head": 4096}, {"geo_head": 16384}, {"pipeline_depth": 10}, {"pipeline_depth": 6}]'
timeout 1500 python tools/knob_check.py 28,3,lex 24,3,lex 26,4,glex > gpurun_out/knob_r02al.log 2>&1
