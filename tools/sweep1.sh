timeout 100 python tools/sweep.py '[{"cfg":[26,4,"lex"]},{"cfg":[24,5,"lex"]},{"cfg":[28,3,"lex"]},{"cfg":[24,2,"lex"]},{"cfg":[24,2,"lex"],"opts":{"window0":4096}}]'
