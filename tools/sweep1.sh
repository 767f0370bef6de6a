C='[{"cfg":[28,3,"lex"]},{"cfg":[26,4,"glex"]},{"cfg":[26,4,"gray"]},{"cfg":[24,3,"lex"]},{"cfg":[24,3,"grlex"]},{"cfg":[24,8,"lex"]},{"cfg":[24,3,"gray"]},{"cfg":[24,3,"glex"]}]'
timeout 100 python tools/sweep.py "$C"
for T in 320 448; do echo "== target $T"; GC_TARGET_ACCEPTED=$T timeout 100 python tools/sweep.py '[{"cfg":[28,3,"lex"]},{"cfg":[26,4,"gray"]},{"cfg":[24,3,"lex"]}]'; done
