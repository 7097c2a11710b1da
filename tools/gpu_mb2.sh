timeout 120 ./tools/mb_fp64
