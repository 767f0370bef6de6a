# round-2 pass w: r_decide counts undecided survivors without BAR.RED; debug-mode probes (run under gpurun)
mkdir -p gpurun_out
PIPE_OPTS='[{}]' timeout 600 python tools/pipe_check.py 7,3,lex > gpurun_out/pipe_check_r02w.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02w.log
for o in '{}' '{"prep_lead": 2}' '{"prep_lead": 3, "prep_ctas": 4}' '{"flags": 16384}'; do
  for w in 24,3,lex 28,3,lex; do
    PROBE_OPTS="[$o]" timeout 300 python tools/phase_probe.py $w >> gpurun_out/phase_probe_r02w.log 2>&1
    echo "exit $? $w $o" >> gpurun_out/phase_probe_r02w.log
  done
done
