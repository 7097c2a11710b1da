# apply time per level: grid size of the standalone apply kernel
for g in 148 8 1; do SKR_PC_GRID=$g timeout 300 python tools/prof_pc_apply.py 1 2>&1 | grep apply; done
for g in 148 37 16; do SKR_PC_GRID=$g timeout 300 python tools/prof_pc_apply.py 3 2>&1 | grep apply; done
