timeout 900 python tools/pc_chains_probe.py 3 ilu0 16 8 37 2>&1 | grep -v Warn | tail -3
timeout 900 python tools/pc_chains_probe.py 1 ilu0 32 8 64 2>&1 | grep -v Warn | tail -3
timeout 900 python tools/pc_chains_probe.py 1 sor 32 8 64 2>&1 | grep -v Warn | tail -3
