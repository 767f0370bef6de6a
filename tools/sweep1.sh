C='[{"cfg":[28,3,"lex"]},{"cfg":[26,4,"gray"]},{"cfg":[24,3,"lex"]}]'
for S in 65536 262144 524288 1048576; do echo "== submax $S"; GC_SUB_MAX=$S timeout 100 python tools/sweep.py "$C"; done
