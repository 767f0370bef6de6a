GC_DEBUG_PHASES=1 timeout 100 python tools/sweep.py '[{"cfg":[24,3,"lex"]},{"cfg":[28,3,"lex"]}]' 2>&1 | awk '!seen[$0]++' | grep -v level
