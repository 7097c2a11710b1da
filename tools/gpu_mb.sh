timeout 300 ./tools/mb_dots
