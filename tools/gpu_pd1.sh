timeout 300 python tools/prof_dense.py 1 3 2>&1 | grep -v Warn | grep -v "return torch"
