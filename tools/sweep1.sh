C='[{"cfg":[28,3,"lex"]},{"cfg":[26,4,"glex"]},{"cfg":[26,4,"gray"]},{"cfg":[24,3,"lex"]},{"cfg":[24,3,"grlex"]},{"cfg":[24,8,"lex"]}]'
for SM in 32768 4096 131072; do for I in 1 2; do echo "== sub_max $SM items $I"; GC_SUB_MAX=$SM GC_ITEMS_PER_WARP=$I timeout 100 python tools/sweep.py "$C"; done; done
echo "== phases"; GC_DEBUG_PHASES=1 timeout 100 python tools/sweep.py '[{"cfg":[28,3,"lex"]},{"cfg":[26,4,"glex"]}]'
