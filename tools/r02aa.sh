# round-2 pass aa: one r_decide call site for prepared tiles; debug probes + parity-gated sweep (run under gpurun)
mkdir -p gpurun_out
for w in 24,3,lex 20,3,lex; do
  timeout 120 python tools/dbg_case.py $w '{"flags": 512}' >> gpurun_out/dbg_r02aa.log 2>&1
  echo "exit $? $w" >> gpurun_out/dbg_r02aa.log
done
PIPE_OPTS='[{}]' timeout 600 python tools/pipe_check.py 7,3,lex > gpurun_out/pipe_check_r02aa.log 2>&1; echo "exit $?" >> gpurun_out/pipe_check_r02aa.log
for o in '{}' '{"prep_lead": 2}' '{"prep_lead": 3, "prep_ctas": 4}'; do
  PROBE_OPTS="[$o]" timeout 300 python tools/phase_probe.py 28,3,lex 24,3,lex >> gpurun_out/phase_probe_r02aa.log 2>&1
done
