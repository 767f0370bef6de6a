GC_DEBUG_PHASES=1 timeout 100 python tools/sweep.py '[{"cfg":[28,3,"lex"]}]' 2>&1 | awk '!seen[$0]++' | grep "per tile"
