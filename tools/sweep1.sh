C='[{"cfg":[28,3,"lex"]},{"cfg":[26,4,"glex"]},{"cfg":[26,4,"gray"]},{"cfg":[26,4,"lex"]},{"cfg":[24,3,"lex"]},{"cfg":[24,3,"grlex"]},{"cfg":[24,3,"gray"]},{"cfg":[24,3,"glex"]},{"cfg":[24,8,"lex"]}]'
timeout 100 python tools/sweep.py "$C"
