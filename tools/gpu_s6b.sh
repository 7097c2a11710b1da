timeout 900 python -m pytest tests/test_precond.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/prof_pc_apply.py 1 2>&1 | grep apply
timeout 300 python tools/prof_pc_apply.py 3 2>&1 | grep apply
timeout 900 python tools/prof_precond.py 1 3 2>&1 | grep -v Warn
timeout 900 python tools/prof_precond.py 3 2 2>&1 | grep -v Warn
timeout 900 python tools/pc_chains_probe.py 3 ilu0 16 8 37 2>&1 | grep -v Warn | tail -1 | cut -c1-140
