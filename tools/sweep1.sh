C='[{"cfg":[28,3,"lex"]},{"cfg":[26,4,"glex"]},{"cfg":[26,4,"gray"]},{"cfg":[24,3,"lex"]},{"cfg":[24,3,"grlex"]},{"cfg":[24,8,"lex"]}]'
for I in 1 2 4 8; do echo "== items $I"; GC_ITEMS_PER_WARP=$I timeout 100 python tools/sweep.py "$C"; done
echo "== phases"; GC_ITEMS_PER_WARP=4 GC_DEBUG_PHASES=1 timeout 100 python tools/sweep.py '[{"cfg":[28,3,"lex"]},{"cfg":[26,4,"glex"]}]' 2>&1 | awk '!seen[$0]++'
