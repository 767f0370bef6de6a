# round-2 pass g: racecheck after the warp-tail fix; tile-size / preparation knob sweep (run under gpurun)
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck_r02g.log 2>&1; echo "exit $?" >> gpurun_out/sanitize_racecheck_r02g.log
export PIPE_OPTS='[{}, {"target_accepted": 768}, {"target_accepted": 1536}, {"target_accepted": 192}, {"prep_lead": 1}, {"prep_ctas": 4}, {"prep_ctas": 4, "prep_lead": 3}]'
timeout 1200 python tools/pipe_check.py 28,3,lex 24,3,lex 26,4,gray 26,4,glex 24,8,lex > gpurun_out/pipe_check_r02g.log 2>&1
