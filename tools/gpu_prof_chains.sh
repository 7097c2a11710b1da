timeout 600 python tools/prof_chains.py 3 16 8 37 2>&1 | grep -v Warn
